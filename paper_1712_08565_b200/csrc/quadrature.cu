// Tensor-Gauss quadrature on the device: the load vector and the L2 / H1 error integrals
// (SURVEY 8(f) rank 4).
//
//   assemble_rhs      f_i = int det J  b_i  (f o F) dxi                   assembly.py:201-230
//   _error_integrals  err2 = int det J (|u - u_h|^2 [+ |grad u - grad u_h|^2]),
//                     ref2 = int det J (|u|^2 [+ |grad u|^2])              problems.py:97-150
//
// Both are sum-factorised over blocks of EB x EB x 1 elements (one CTA each): the Gauss values of a
// block live in shared memory and are contracted direction by direction with the element-blocked
// collocation tables  Bt[d][q][k] = D^d b_{first(e(q)) + k}(x_q),  k = 0..p.
//   RHS:   point values -> z (p+1 planes) -> y (DoF rows) -> x (DoF columns) -> fp64 atomics into f
//   error: DoF window of u -> x -> y -> z -> per-point error terms -> per-CTA partial sums, reduced
//          in a fixed order (deterministic)
// The integrand is either a built-in manufactured case evaluated in the kernel (cube sine,
// quarter-ring oscillating; problems.py:77-94) or caller-provided values at every Gauss point
// (any host callable, evaluated by the Python layer at the mapped points).
#include <algorithm>
#include <cmath>

#include "ops.h"

namespace mfwq {

struct QuadDirDev {
  int n_el, nfull, n;  // elements, full basis functions, interior DoFs (= nfull - 2)
  const double* x;     // [n_el*g] Gauss points
  const double* w;     // [n_el*g] weights
  const double* B;     // [2][n_el*g][p+1]  (value, derivative)
  const int* first;    // [n_el] first full basis index of each element
};

struct QuadParams {
  QuadDirDev d[3];
  int p, g, EB;
  int wmax;  // max DoF window width of a block (x and y)
  int kind;  // geometry (GeomKind)
  double A[9], b[3];
  const double* J;      // GEOM_JACOBIAN: [Ng][9]
  int case_id;          // 0 = values from arrays, 1 = cube sine, 2 = quarter-ring oscillating
  const double* fvals;  // [Ng] values of f (rhs) / u (error)
  const double* gvals;  // [Ng][3] grad u (error, H1)
  int ng1, ng2;         // Gauss points per direction (x, y)
};

enum QuadCase { QCASE_VALUES = 0, QCASE_CUBE_SINE = 1, QCASE_RING_OSC = 2 };

// ---- manufactured solutions (problems.py:77-94), closed form of the sympy derivation --------
__device__ __forceinline__ void case_eval(int id, const double* x, double& u, double g[3], double& f) {
  if (id == QCASE_CUBE_SINE) {  // u = sin(pi x) sin(pi y) sin(pi z), f = -lap u = 3 pi^2 u
    double s[3], c[3];
    for (int l = 0; l < 3; ++l) sincospi(x[l], &s[l], &c[l]);
    u = s[0] * s[1] * s[2];
    g[0] = M_PI * c[0] * s[1] * s[2];
    g[1] = M_PI * s[0] * c[1] * s[2];
    g[2] = M_PI * s[0] * s[1] * c[2];
    f = 3.0 * M_PI * M_PI * u;
  } else {  // u = S h,  S = prod sin(5 pi x_l),  h = (r^2 - 1)(r^2 - 4),  r^2 = x^2 + y^2
    double s[3], c[3];
    for (int l = 0; l < 3; ++l) sincospi(5.0 * x[l], &s[l], &c[l]);
    const double k = 5.0 * M_PI;
    const double S = s[0] * s[1] * s[2];
    const double dS[3] = {k * c[0] * s[1] * s[2], k * s[0] * c[1] * s[2], k * s[0] * s[1] * c[2]};
    const double r2 = x[0] * x[0] + x[1] * x[1];
    const double h = (r2 - 1.0) * (r2 - 4.0);
    const double dh[3] = {(4.0 * r2 - 10.0) * x[0], (4.0 * r2 - 10.0) * x[1], 0.0};
    u = S * h;
    for (int l = 0; l < 3; ++l) g[l] = h * dS[l] + S * dh[l];
    const double lapS = -3.0 * k * k * S, laph = 16.0 * r2 - 20.0;
    f = -(h * lapS + 2.0 * (dS[0] * dh[0] + dS[1] * dh[1]) + S * laph);
  }
}

// geometry at a parametric point: physical point X, Jacobian J (geometry.py:47-96)
__device__ __forceinline__ void geom_eval(const QuadParams& P, const double* xi, long long q, double X[3],
                                          double J[3][3]) {
  if (P.kind == GEOM_IDENTITY) {
    for (int i = 0; i < 3; ++i) {
      X[i] = xi[i];
      for (int j = 0; j < 3; ++j) J[i][j] = i == j ? 1.0 : 0.0;
    }
  } else if (P.kind == GEOM_AFFINE) {
    for (int i = 0; i < 3; ++i) {
      X[i] = P.b[i];
      for (int j = 0; j < 3; ++j) {
        J[i][j] = P.A[3 * i + j];
        X[i] += P.A[3 * i + j] * xi[j];
      }
    }
  } else if (P.kind == GEOM_RING) {
    const double r = 1.0 + xi[0];
    double s, c;
    sincospi(0.5 * xi[1], &s, &c);
    X[0] = r * c;
    X[1] = r * s;
    X[2] = xi[2];
    J[0][0] = c; J[0][1] = -M_PI / 2 * r * s; J[0][2] = 0.0;
    J[1][0] = s; J[1][1] = M_PI / 2 * r * c; J[1][2] = 0.0;
    J[2][0] = 0.0; J[2][1] = 0.0; J[2][2] = 1.0;
  } else {
    const double* Jq = P.J + 9 * q;
    for (int i = 0; i < 3; ++i) {
      X[i] = 0.0;  // values come from the caller's arrays
      for (int j = 0; j < 3; ++j) J[i][j] = Jq[3 * i + j];
    }
  }
}

__device__ __forceinline__ double det3(const double J[3][3]) {
  return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

// DoF window of a block along one direction: full indices [w0, w0 + width)
__device__ __forceinline__ void window(const QuadDirDev& D, int e0, int ne, int p, int& w0, int& width) {
  w0 = D.first[e0];
  width = D.first[e0 + ne - 1] + p + 1 - w0;
}

// ---- load vector ------------------------------------------------------------------------
__global__ void rhs_kernel(QuadParams P, double* __restrict__ rhs) {
  extern __shared__ double sq[];
  const int p = P.p, g = P.g, EB = P.EB, NB = p + 1;
  const int e1a = blockIdx.x * EB, e2a = blockIdx.y * EB, e3 = blockIdx.z;
  const int ne1 = min(EB, P.d[0].n_el - e1a), ne2 = min(EB, P.d[1].n_el - e2a);
  const int n1g = ne1 * g, n2g = ne2 * g, EG = EB * g;
  double* vals = sq;                   // [g][EG][EG]
  double* tz = vals + g * EG * EG;     // [NB][EG][EG]
  double* ty = tz + NB * EG * EG;      // [NB][wmax][EG]
  int w10, w1n, w20, w2n;
  window(P.d[0], e1a, ne1, p, w10, w1n);
  window(P.d[1], e2a, ne2, p, w20, w2n);
  const int w30 = P.d[2].first[e3];
  // 1. integrand at the block's Gauss points: w1 w2 w3 det J f(F(xi))
  for (int i = threadIdx.x; i < g * n2g * n1g; i += blockDim.x) {
    const int gx = i % n1g, gy = (i / n1g) % n2g, gz = i / (n1g * n2g);
    const int q1 = e1a * g + gx, q2 = e2a * g + gy, q3 = e3 * g + gz;
    const long long q = ((long long)q3 * P.ng2 + q2) * P.ng1 + q1;
    const double xi[3] = {P.d[0].x[q1], P.d[1].x[q2], P.d[2].x[q3]};
    double X[3], J[3][3];
    geom_eval(P, xi, q, X, J);
    double f;
    if (P.case_id == QCASE_VALUES) {
      f = P.fvals[q];
    } else {
      double u, gr[3];
      case_eval(P.case_id, X, u, gr, f);
    }
    vals[(gz * EG + gy) * EG + gx] = P.d[0].w[q1] * P.d[1].w[q2] * P.d[2].w[q3] * det3(J) * f;
  }
  __syncthreads();
  // 2. z: the p+1 DoF planes of element e3
  const double* B3 = P.d[2].B + (size_t)e3 * g * NB;
  for (int i = threadIdx.x; i < NB * n2g * n1g; i += blockDim.x) {
    const int gx = i % n1g, gy = (i / n1g) % n2g, k = i / (n1g * n2g);
    double a = 0.0;
    for (int gz = 0; gz < g; ++gz) a += B3[gz * NB + k] * vals[(gz * EG + gy) * EG + gx];
    tz[(k * EG + gy) * EG + gx] = a;
  }
  __syncthreads();
  // 3. y: DoF rows of the window (gather over the points whose element reaches the row)
  for (int i = threadIdx.x; i < NB * w2n * n1g; i += blockDim.x) {
    const int gx = i % n1g, j2 = (i / n1g) % w2n, k3 = i / (n1g * w2n);
    double a = 0.0;
    for (int ey = 0; ey < ne2; ++ey) {
      const int k = j2 + w20 - P.d[1].first[e2a + ey];
      if (k < 0 || k > p) continue;
      const double* B2 = P.d[1].B + (size_t)(e2a + ey) * g * NB;
      for (int gl = 0; gl < g; ++gl) a += B2[gl * NB + k] * tz[(k3 * EG + ey * g + gl) * EG + gx];
    }
    ty[(k3 * P.wmax + j2) * EG + gx] = a;
  }
  __syncthreads();
  // 4. x, then add the interior entries into f
  const int n1 = P.d[0].n, n2 = P.d[1].n, n3 = P.d[2].n;
  for (int i = threadIdx.x; i < NB * w2n * w1n; i += blockDim.x) {
    const int j1 = i % w1n, j2 = (i / w1n) % w2n, k3 = i / (w1n * w2n);
    const int i1 = w10 + j1 - 1, i2 = w20 + j2 - 1, i3 = w30 + k3 - 1;  // interior indices
    if (i1 < 0 || i1 >= n1 || i2 < 0 || i2 >= n2 || i3 < 0 || i3 >= n3) continue;
    double a = 0.0;
    for (int ex = 0; ex < ne1; ++ex) {
      const int k = j1 + w10 - P.d[0].first[e1a + ex];
      if (k < 0 || k > p) continue;
      const double* B1 = P.d[0].B + (size_t)(e1a + ex) * g * NB;
      for (int gl = 0; gl < g; ++gl) a += B1[gl * NB + k] * ty[(k3 * P.wmax + j2) * EG + ex * g + gl];
    }
    atomicAdd(&rhs[((size_t)i3 * n2 + i2) * n1 + i1], a);
  }
}

// ---- error integrals ----------------------------------------------------------------------
__global__ void err_kernel(QuadParams P, const double* __restrict__ u, int with_grad, double* __restrict__ part) {
  extern __shared__ double sq[];
  const int p = P.p, g = P.g, EB = P.EB, NB = p + 1, W = P.wmax;
  const int e1a = blockIdx.x * EB, e2a = blockIdx.y * EB, e3 = blockIdx.z;
  const int ne1 = min(EB, P.d[0].n_el - e1a), ne2 = min(EB, P.d[1].n_el - e2a);
  const int n1g = ne1 * g, n2g = ne2 * g, EG = EB * g;
  int w10, w1n, w20, w2n;
  window(P.d[0], e1a, ne1, p, w10, w1n);
  window(P.d[1], e2a, ne2, p, w20, w2n);
  const int w30 = P.d[2].first[e3];
  const int nd = with_grad ? 2 : 1;
  double* uw = sq;                   // [NB][W][W]        DoF window (zero outside the interior)
  double* ax = uw + NB * W * W;      // [2][NB][W][EG]    x-contracted (B0, B1)
  double* ay = ax + 2 * NB * W * EG; // [3][NB][EG][EG]   y-contracted: B0B0, B0B1(x-deriv), B1B0(y-deriv)
  __shared__ double red[2][32];
  const int n1 = P.d[0].n, n2 = P.d[1].n, n3 = P.d[2].n;
  for (int i = threadIdx.x; i < NB * w2n * w1n; i += blockDim.x) {
    const int j1 = i % w1n, j2 = (i / w1n) % w2n, k3 = i / (w1n * w2n);
    const int i1 = w10 + j1 - 1, i2 = w20 + j2 - 1, i3 = w30 + k3 - 1;
    const bool in = i1 >= 0 && i1 < n1 && i2 >= 0 && i2 < n2 && i3 >= 0 && i3 < n3;
    uw[(k3 * W + j2) * W + j1] = in ? u[((size_t)i3 * n2 + i2) * n1 + i1] : 0.0;
  }
  __syncthreads();
  // x: for each Gauss x point, B0 / B1 combinations of the window columns
  for (int i = threadIdx.x; i < nd * NB * w2n * n1g; i += blockDim.x) {
    const int gx = i % n1g, j2 = (i / n1g) % w2n, k3 = (i / (n1g * w2n)) % NB, d = i / (n1g * w2n * NB);
    const int ex = gx / g, q1 = e1a * g + gx;
    const int c0 = P.d[0].first[e1a + ex] - w10;
    const double* B1 = P.d[0].B + ((size_t)d * P.d[0].n_el * g + q1) * NB;
    double a = 0.0;
    for (int k = 0; k < NB; ++k) a += B1[k] * uw[(k3 * W + j2) * W + c0 + k];
    ax[((d * NB + k3) * W + j2) * EG + gx] = a;
  }
  __syncthreads();
  // y: combos (y-deriv, x-deriv) = (0,0) -> 0, (0,1) -> 1, (1,0) -> 2
  const int ncomb = with_grad ? 3 : 1;
  for (int i = threadIdx.x; i < ncomb * NB * n2g * n1g; i += blockDim.x) {
    const int gx = i % n1g, gy = (i / n1g) % n2g, k3 = (i / (n1g * n2g)) % NB, cb = i / (n1g * n2g * NB);
    const int dy = cb == 2 ? 1 : 0, dx = cb == 1 ? 1 : 0;
    const int ey = gy / g, q2 = e2a * g + gy;
    const int r0 = P.d[1].first[e2a + ey] - w20;
    const double* B2 = P.d[1].B + ((size_t)dy * P.d[1].n_el * g + q2) * NB;
    double a = 0.0;
    for (int k = 0; k < NB; ++k) a += B2[k] * ax[((dx * NB + k3) * W + r0 + k) * EG + gx];
    ay[((cb * NB + k3) * EG + gy) * EG + gx] = a;
  }
  __syncthreads();
  // z + point terms
  double e2 = 0.0, r2 = 0.0;
  const double* B3v = P.d[2].B + (size_t)e3 * g * NB;
  const double* B3d = P.d[2].B + ((size_t)P.d[2].n_el * g + (size_t)e3 * g) * NB;
  for (int i = threadIdx.x; i < g * n2g * n1g; i += blockDim.x) {
    const int gx = i % n1g, gy = (i / n1g) % n2g, gz = i / (n1g * n2g);
    const int q1 = e1a * g + gx, q2 = e2a * g + gy, q3 = e3 * g + gz;
    const long long q = ((long long)q3 * P.ng2 + q2) * P.ng1 + q1;
    double uh = 0.0, gp[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < NB; ++k) {
      const double b0 = B3v[gz * NB + k];
      uh += b0 * ay[((0 * NB + k) * EG + gy) * EG + gx];
      if (with_grad) {
        gp[0] += b0 * ay[((1 * NB + k) * EG + gy) * EG + gx];
        gp[1] += b0 * ay[((2 * NB + k) * EG + gy) * EG + gx];
        gp[2] += B3d[gz * NB + k] * ay[((0 * NB + k) * EG + gy) * EG + gx];
      }
    }
    const double xi[3] = {P.d[0].x[q1], P.d[1].x[q2], P.d[2].x[q3]};
    double X[3], J[3][3];
    geom_eval(P, xi, q, X, J);
    const double det = det3(J);
    const double meas = P.d[0].w[q1] * P.d[1].w[q2] * P.d[2].w[q3] * det;
    double ue, ge[3], fdummy;
    if (P.case_id == QCASE_VALUES) {
      ue = P.fvals[q];
      if (with_grad)
        for (int l = 0; l < 3; ++l) ge[l] = P.gvals[3 * q + l];
    } else {
      case_eval(P.case_id, X, ue, ge, fdummy);
    }
    e2 += meas * (ue - uh) * (ue - uh);
    r2 += meas * ue * ue;
    if (with_grad) {
      // grad u_h = J^{-T} grad_xi u_h  (problems.py:141-142)
      const double id = 1.0 / det;
      double Ji[3][3];
      Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * id;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
      Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * id;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
      Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * id;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
      for (int l = 0; l < 3; ++l) {
        const double gh = Ji[0][l] * gp[0] + Ji[1][l] * gp[1] + Ji[2][l] * gp[2];
        e2 += meas * (ge[l] - gh) * (ge[l] - gh);
        r2 += meas * ge[l] * ge[l];
      }
    }
  }
  // fixed-order block reduction -> one partial pair per CTA
  for (int o = 16; o > 0; o >>= 1) {
    e2 += __shfl_down_sync(0xffffffffu, e2, o);
    r2 += __shfl_down_sync(0xffffffffu, r2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = e2;
    red[1][threadIdx.x >> 5] = r2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    const size_t blk = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    part[2 * blk] = a;
    part[2 * blk + 1] = b;
  }
}

__global__ void sum_pairs_kernel(const double* __restrict__ part, long long n, double* __restrict__ out) {
  __shared__ double s[2][256];
  double a = 0.0, b = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  s[0][threadIdx.x] = a;
  s[1][threadIdx.x] = b;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s[0][threadIdx.x] += s[0][threadIdx.x + o];
      s[1][threadIdx.x] += s[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s[0][0];
    out[1] = s[1][0];
  }
}

// ---- host ---------------------------------------------------------------------------------
Quadrature::Quadrature(const int* p, const int* nknots, const double* const* knots, int gauss_per_span) {
  deg = p[0];
  for (int l = 1; l < 3; ++l)
    if (p[l] != deg) throw NotImplErr("device quadrature: equal degrees per direction required");
  g = gauss_per_span > 0 ? gauss_per_span : deg + 1;
  if (g > 32) throw ValueErr("gauss_pts_per_span must be <= 32");
  for (int l = 0; l < 3; ++l) {
    Knots kv(p[l], knots[l], nknots[l]);
    QDir& D = dir[l];
    D.n_el = kv.n_el();
    D.nfull = kv.nfun();
    gauss_rule(kv, g, D.x, D.w);
    Csr B[2] = {collocation(kv, D.x, 0), collocation(kv, D.x, 1)};
    const int NB = deg + 1, ng = D.n_el * g;
    std::vector<double> tab((size_t)2 * ng * NB, 0.0);
    std::vector<int> first(D.n_el, 0);
    for (int e = 0; e < D.n_el; ++e) {
      int f = 1 << 30;
      for (int q = e * g; q < (e + 1) * g; ++q)
        for (int u = B[0].indptr[q]; u < B[0].indptr[q + 1]; ++u) f = std::min(f, B[0].indices[u]);
      first[e] = f;
      for (int d = 0; d < 2; ++d)
        for (int q = e * g; q < (e + 1) * g; ++q)
          for (int u = B[d].indptr[q]; u < B[d].indptr[q + 1]; ++u) {
            const int k = B[d].indices[u] - f;
            if (k < 0 || k > deg) throw NotImplErr("device quadrature: basis outside the element band");
            tab[((size_t)d * ng + q) * NB + k] = B[d].data[u];
          }
    }
    D.x_d.upload(D.x.data(), D.x.size());
    D.w_d.upload(D.w.data(), D.w.size());
    D.B_d.upload(tab.data(), tab.size());
    D.first_d.upload(first.data(), first.size());
    D.first = first;
  }
}

int Quadrature::window_max(int eb) const {
  int w = 0;
  for (int l = 0; l < 2; ++l)
    for (int e = 0; e < dir[l].n_el; e += eb) {
      const int ne = std::min(eb, dir[l].n_el - e);
      w = std::max(w, dir[l].first[e + ne - 1] + deg + 1 - dir[l].first[e]);
    }
  return w;
}

// largest element block (4, 2 or 1 elements per side) whose shared-memory plan fits one CTA
void Quadrature::pick_block(bool err, int& eb, int& w, size_t& smem) const {
  const int NB = deg + 1;
  for (eb = 4; eb >= 1; eb /= 2) {
    w = window_max(eb);
    const size_t EG = (size_t)eb * g;
    smem = sizeof(double) * (err ? (size_t)NB * w * w + 2 * (size_t)NB * w * EG + 3 * (size_t)NB * EG * EG
                                 : (size_t)g * EG * EG + (size_t)NB * EG * EG + (size_t)NB * w * EG);
    if (smem <= 200 * 1024) return;
  }
  throw NotImplErr("device quadrature: too many Gauss points per span for one CTA");
}

long long Quadrature::n_points() const {
  return (long long)dir[0].n_el * g * dir[1].n_el * g * dir[2].n_el * g;
}
long long Quadrature::n_dofs() const {
  return (long long)(dir[0].nfull - 2) * (dir[1].nfull - 2) * (dir[2].nfull - 2);
}

static QuadParams quad_params(const Quadrature& Q, int kind, const double* affine12, const double* J_dev, int case_id,
                              const double* fvals, const double* gvals) {
  QuadParams P;
  for (int l = 0; l < 3; ++l) {
    const auto& D = Q.dir[l];
    P.d[l] = QuadDirDev{D.n_el, D.nfull, D.nfull - 2, D.x_d.ptr, D.w_d.ptr, D.B_d.ptr, D.first_d.ptr};
  }
  P.p = Q.deg;
  P.g = Q.g;
  P.kind = kind;
  for (int i = 0; i < 9; ++i) P.A[i] = affine12 ? affine12[i] : (i % 4 == 0 ? 1.0 : 0.0);
  for (int i = 0; i < 3; ++i) P.b[i] = affine12 ? affine12[9 + i] : 0.0;
  P.J = J_dev;
  P.case_id = case_id;
  P.fvals = fvals;
  P.gvals = gvals;
  P.ng1 = Q.dir[0].n_el * Q.g;
  P.ng2 = Q.dir[1].n_el * Q.g;
  if (kind == GEOM_JACOBIAN && !J_dev) throw ValueErr("Jacobian geometry needs the Jacobian at every Gauss point");
  if (kind == GEOM_JACOBIAN && case_id != QCASE_VALUES)
    throw ValueErr("a Jacobian-only geometry needs integrand values from the caller (no physical map on the device)");
  if (case_id == QCASE_VALUES && !fvals) throw ValueErr("integrand values missing");
  if (case_id < 0 || case_id > QCASE_RING_OSC) throw ValueErr("unknown manufactured case");
  return P;
}

void Quadrature::rhs(int kind, const double* affine12, const double* J_dev, int case_id, const double* fvals,
                     double* out, cudaStream_t s) {
  QuadParams P = quad_params(*this, kind, affine12, J_dev, case_id, fvals, nullptr);
  int EB;
  size_t smem;
  pick_block(false, EB, P.wmax, smem);
  P.EB = EB;
  MFWQ_CUDA(cudaFuncSetAttribute(rhs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  MFWQ_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * n_dofs(), s));
  dim3 grid((dir[0].n_el + EB - 1) / EB, (dir[1].n_el + EB - 1) / EB, dir[2].n_el);
  rhs_kernel<<<grid, 256, smem, s>>>(P, out); note_launch();
  MFWQ_CUDA(cudaGetLastError());
}

void Quadrature::errors(int kind, const double* affine12, const double* J_dev, int case_id, const double* uvals,
                        const double* gvals, const double* u, int with_grad, double* err_ref, cudaStream_t s) {
  if (case_id == QCASE_VALUES && with_grad && !gvals) throw ValueErr("gradient values missing");
  QuadParams P = quad_params(*this, kind, affine12, J_dev, case_id, uvals, gvals);
  int EB;
  size_t smem;
  pick_block(true, EB, P.wmax, smem);
  P.EB = EB;
  MFWQ_CUDA(cudaFuncSetAttribute(err_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  dim3 grid((dir[0].n_el + EB - 1) / EB, (dir[1].n_el + EB - 1) / EB, dir[2].n_el);
  const long long nb = (long long)grid.x * grid.y * grid.z;
  part_.alloc_at_least(2 * nb + 2);
  err_kernel<<<grid, 256, smem, s>>>(P, u, with_grad, part_.ptr); note_launch();
  MFWQ_CUDA(cudaGetLastError());
  sum_pairs_kernel<<<1, 256, 0, s>>>(part_.ptr, nb, part_.ptr + 2 * nb); note_launch();
  MFWQ_CUDA(cudaGetLastError());
  MFWQ_CUDA(cudaMemcpyAsync(err_ref, part_.ptr + 2 * nb, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
}

}  // namespace mfwq
