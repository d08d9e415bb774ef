// MF-WQ stiffness operator: setup, coefficient grids (K5), and the generic
// correctness-first path (K1 banded mode contractions composed exactly like
// operators.py:185-204).  The fused hot path lives in fused_matvec.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "ops.h"

namespace mfwq {

// ---------------------------------------------------------------------------
// CSR -> band packing
// ---------------------------------------------------------------------------
BandHost csr_to_band(const Csr& A, int r0, int r1, int c0, int c1) {
  BandHost b;
  b.rows = r1 - r0;
  b.cols = c1 - c0;
  b.start.assign(b.rows, 0);
  int width = 1;
  std::vector<int> lo(b.rows, 0), hi(b.rows, -1);
  for (int r = r0; r < r1; ++r) {
    int mn = 1 << 30, mx = -1;
    for (int u = A.indptr[r]; u < A.indptr[r + 1]; ++u) {
      int c = A.indices[u];
      if (c < c0 || c >= c1) continue;
      mn = std::min(mn, c - c0);
      mx = std::max(mx, c - c0);
    }
    if (mx < 0) { mn = 0; mx = 0; }
    lo[r - r0] = mn;
    hi[r - r0] = mx;
    width = std::max(width, mx - mn + 1);
  }
  b.width = width;
  b.vals.assign(size_t(b.rows) * width, 0.0);
  for (int r = r0; r < r1; ++r) {
    int s = std::min(lo[r - r0], std::max(0, b.cols - width));  // keep start+width <= cols
    b.start[r - r0] = s;
    for (int u = A.indptr[r]; u < A.indptr[r + 1]; ++u) {
      int c = A.indices[u] - c0;
      if (c < 0 || c >= b.cols) continue;
      b.vals[size_t(r - r0) * width + (c - s)] = A.data[u];
    }
  }
  return b;
}

static long long csr_nnz_in(const Csr& A, int r0, int r1, int c0, int c1) {
  long long k = 0;
  for (int r = r0; r < r1; ++r)
    for (int u = A.indptr[r]; u < A.indptr[r + 1]; ++u)
      if (A.indices[u] >= c0 && A.indices[u] < c1) ++k;
  return k;
}

void Stiffness::init(const int* p, const int* nknots, const double* const* knots, const int* npts,
                     const double* const* pts, const int* const* indptr, const int* const* indices,
                     const double* const* data) {
  for (int l = 0; l < 3; ++l) {
    Dir1D& d = dir[l];
    Knots kv(p[l], knots[l], nknots[l]);
    d.p = p[l];
    d.n_el = kv.n_el();
    d.knots = kv.t;
    const int nfun = kv.nfun();
    d.n = nfun - 2;
    if (d.n < 1) throw ValueErr("each direction needs at least one interior function");
    d.m = npts[l];
    d.pts.assign(pts[l], pts[l] + npts[l]);
    // CSR order per direction: W00, W01, W10, W11 (nfun x m), B0, B1 (m x nfun)
    Csr mats[6];
    for (int k = 0; k < 6; ++k) {
      Csr& c = mats[k];
      c.rows = k < 4 ? nfun : d.m;
      c.cols = k < 4 ? d.m : nfun;
      c.indptr.assign(indptr[l * 6 + k], indptr[l * 6 + k] + c.rows + 1);
      int nnz = c.indptr.back();
      c.indices.assign(indices[l * 6 + k], indices[l * 6 + k] + nnz);
      c.data.assign(data[l * 6 + k], data[l * 6 + k] + nnz);
    }
    for (int k = 0; k < 4; ++k) {
      d.W[k].h = csr_to_band(mats[k], 1, nfun - 1, 0, d.m);
      d.W[k].upload();
      nnz_[l][2 + k] = csr_nnz_in(mats[k], 1, nfun - 1, 0, d.m);
    }
    for (int k = 0; k < 2; ++k) {
      d.B[k].h = csr_to_band(mats[4 + k], 0, d.m, 1, nfun - 1);
      d.B[k].upload();
      nnz_[l][k] = csr_nnz_in(mats[4 + k], 0, d.m, 1, nfun - 1);
    }
    // element ownership of quadrature points (right-continuous spans)
    d.elem_q0.assign(d.n_el + 1, d.m);
    for (int q = d.m - 1; q >= 0; --q) {
      int e = kv.span(d.pts[q]) - kv.p;
      e = std::min(std::max(e, 0), d.n_el - 1);
      d.elem_q0[e] = q;
    }
    for (int e = d.n_el - 1; e >= 0; --e) d.elem_q0[e] = std::min(d.elem_q0[e], d.elem_q0[e + 1]);
    d.pts_d.upload(d.pts.data(), d.pts.size());
  }
  N = (long long)dir[0].n * dir[1].n * dir[2].n;
  Nq = (long long)dir[0].m * dir[1].m * dir[2].m;
  m1p = (dir[0].m + 3) / 4 * 4;
  set_slab(0, dir[2].n_el);
  compute_flops();
}

// CostMeter count (kron.py:90-96, operators.py:191-203) restricted to the
// terms in `mask` (bit 3a+b); mask 0x1FF is the reference's full count.
long long Stiffness::flops_for(int mask) const {
  const long long n1 = dir[0].n, n2 = dir[1].n, n3 = dir[2].n;
  const long long m1 = dir[0].m, m2 = dir[1].m, m3 = dir[2].m;
  // S(A; s, t) with contraction order 3, 2, 1 (kron.py:83-96)
  auto S = [&](long long z1, long long z2, long long z3, long long s1, long long s2, long long s3, long long t1,
               long long t2) { (void)s1; return 2 * z3 * t1 * t2 + 2 * z2 * s3 * t1 + 2 * z1 * s3 * s2; };
  long long F = 0;
  for (int b = 0; b < 3; ++b) {
    if (!(mask & (0x49 << b))) continue;  // no active term (a, b)
    long long z[3];
    for (int l = 0; l < 3; ++l) z[l] = nnz_[l][l == b ? 1 : 0];
    F += S(z[0], z[1], z[2], m1, m2, m3, n1, n2);
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      if (!(mask & (1 << (3 * a + b)))) continue;
      long long z[3];
      for (int l = 0; l < 3; ++l) z[l] = nnz_[l][2 + 2 * (l == a) + (l == b)];
      F += S(z[0], z[1], z[2], n1, n2, n3, m1, m2) + Nq + 2 * N;
    }
  return F;
}

void Stiffness::compute_flops() { flops = flops_for(0x1FF); }

// Slab of z-elements [elo, ehi): element e touches interior DoF planes
// e-1 .. e+p-1 on the B side and rows e-2 .. e+p-1 on the W side (the breakpoint at
// the start of e closes the support of full function e-1).
void Stiffness::set_slab(int elo, int ehi) {
  const Dir1D& z = dir[2];
  if (elo < 0 || ehi > z.n_el || elo >= ehi) throw ValueErr("invalid slab element range");
  e_lo = elo;
  e_hi = ehi;
  v_lo = std::max(elo - 1, 0);
  v_hi = std::min(ehi + z.p - 1, z.n);
  y_lo = std::max(elo - 2, 0);
  y_hi = std::min(ehi + z.p - 1, z.n);
  q_lo = z.elem_q0[elo];
  q_hi = z.elem_q0[ehi];
  fused2_plan.reset();
  pcg_graphs.reset();
  coeffs_ready = false;
}

// ---------------------------------------------------------------------------
// K5: coefficient grids (operators.py:64-84, geometry.py:47-96)
// ---------------------------------------------------------------------------
__global__ void coeff_kernel(int kind, const double* __restrict__ x1, const double* __restrict__ x2,
                             const double* __restrict__ x3, int m1, int m2, int m3, int m1p, double A00,
                             double A01, double A02, double A10, double A11, double A12, double A20,
                             double A21, double A22, int kconst, double K00, double K01, double K02,
                             double K10, double K11, double K12, double K20, double K21, double K22,
                             const double* __restrict__ Jfield, const double* __restrict__ Kfield,
                             double* __restrict__ C, size_t gstride, unsigned long long* bad, int* nonzero) {
  const long long Nq = (long long)m1 * m2 * m3;
  unsigned nzmask = 0;  // grids with a non-zero value at this thread's points (terms to keep, detect_nonzero)
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < Nq; q += (long long)gridDim.x * blockDim.x) {
    const int q1 = int(q % m1);
    const long long r = q / m1;
    const int q2 = int(r % m2), q3 = int(r / m2);
    double J[3][3];
    if (kind == GEOM_IDENTITY) {
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) J[i][j] = i == j ? 1.0 : 0.0;
    } else if (kind == GEOM_AFFINE) {
      J[0][0] = A00; J[0][1] = A01; J[0][2] = A02;
      J[1][0] = A10; J[1][1] = A11; J[1][2] = A12;
      J[2][0] = A20; J[2][1] = A21; J[2][2] = A22;
    } else if (kind == GEOM_RING) {  // geometry.py:84-94
      const double rr = 1.0 + x1[q1];
      const double th = M_PI / 2 * x2[q2];
      double s, c;
      sincos(th, &s, &c);
      J[0][0] = c; J[0][1] = -M_PI / 2 * rr * s; J[0][2] = 0.0;
      J[1][0] = s; J[1][1] = M_PI / 2 * rr * c; J[1][2] = 0.0;
      J[2][0] = 0.0; J[2][1] = 0.0; J[2][2] = 1.0;
    } else {
      const double* Jq = Jfield + 9 * q;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) J[i][j] = Jq[3 * i + j];
    }
    double Kq[3][3];
    if (Kfield) {
      const double* kk = Kfield + 9 * q;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Kq[i][j] = kk[3 * i + j];
    } else if (kconst) {
      Kq[0][0] = K00; Kq[0][1] = K01; Kq[0][2] = K02;
      Kq[1][0] = K10; Kq[1][1] = K11; Kq[1][2] = K12;
      Kq[2][0] = K20; Kq[2][1] = K21; Kq[2][2] = K22;
    } else {
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Kq[i][j] = i == j ? 1.0 : 0.0;
    }
    // cofactors
    double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    if (!(det > 0.0)) atomicMin(bad, (unsigned long long)q);
    const double id = 1.0 / det;
    double Ji[3][3];
    Ji[0][0] = c00 * id;
    Ji[1][0] = c01 * id;
    Ji[2][0] = c02 * id;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
    // C = (Ji K Ji^T) * det
    double T[3][3];
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) T[i][k] = Ji[i][0] * Kq[0][k] + Ji[i][1] * Kq[1][k] + Ji[i][2] * Kq[2][k];
    const size_t o = ((size_t)q3 * m2 + q2) * m1p + q1;
    const int keys[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
    for (int g = 0; g < 6; ++g) {
      const int a = keys[g][0], b = keys[g][1];
      const double v = T[a][0] * Ji[b][0] + T[a][1] * Ji[b][1] + T[a][2] * Ji[b][2];
      const double c = v * det;
      C[g * gstride + o] = c;
      if (c != 0.0) nzmask |= 1u << g;
    }
  }
  if (nonzero) {  // one atomic per warp and grid that saw a non-zero value
    nzmask = __reduce_or_sync(0xffffffffu, nzmask);
    if ((threadIdx.x & 31) == 0)
      for (int g = 0; g < 6; ++g)
        if (nzmask >> g & 1) atomicOr(nonzero + g, 1);
  }
}

__global__ void pad_zero_kernel(double* C, int m1, int m1p, long long rows, size_t gstride) {
  // zero the x-padding columns of all 6 grids
  long long tot = rows * (m1p - m1) * 6;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
    int w = m1p - m1;
    long long g = i / (rows * w), rr = (i / w) % rows, c = i % w;
    C[g * gstride + rr * m1p + m1 + c] = 0.0;
  }
}

__global__ void any_nonzero_kernel(const double* __restrict__ C, size_t n, int* flag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (C[i] != 0.0) { *flag = 1; return; }
}

void Stiffness::set_geometry(int kind, const double* A, const double* K9, const double* J_dev,
                             const double* Kfield_dev, cudaStream_t s) {
  otf = false;
  pcg_graphs.reset();  // captured iterations hold the old coefficient pointers / tensor maps
  cx.release();
  const size_t G = grid_elems();
  coeff.alloc(6 * G);
  DevBuf<unsigned long long> bad(1);
  unsigned long long init = ~0ull;
  MFWQ_CUDA(cudaMemcpyAsync(bad.ptr, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  flag_.alloc(6);  // which grids are not identically zero, found by the coefficient kernel itself
  MFWQ_CUDA(cudaMemsetAsync(flag_.ptr, 0, 6 * sizeof(int), s));
  double a[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, k[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (A) std::copy(A, A + 9, a);
  if (K9) std::copy(K9, K9 + 9, k);
  const int m1 = dir[0].m, m2 = dir[1].m, m3 = q_hi - q_lo;  // local quadrature planes
  const long long nql = (long long)m1 * m2 * m3;
  // J_dev / Kfield_dev are full-domain (Nq, 3, 3) arrays (like the grids set_coeffs takes): a slab
  // handle reads its own quadrature planes from q_lo on
  const size_t qoff = (size_t)9 * q_lo * m1 * m2;
  if (J_dev) J_dev += qoff;
  if (Kfield_dev) Kfield_dev += qoff;
  int blocks = std::min<long long>((nql + 255) / 256, 148LL * 16);
  coeff_kernel<<<blocks, 256, 0, s>>>(kind, dir[0].pts_d.ptr, dir[1].pts_d.ptr, dir[2].pts_d.ptr + q_lo, m1, m2, m3, m1p,
                                      a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], K9 ? 1 : 0, k[0], k[1],
                                      k[2], k[3], k[4], k[5], k[6], k[7], k[8], J_dev, Kfield_dev, coeff.ptr, G,
                                      bad.ptr, flag_.ptr); note_launch();
  MFWQ_CUDA(cudaGetLastError());
  if (m1p > m1) {
    pad_zero_kernel<<<148, 256, 0, s>>>(coeff.ptr, m1, m1p, (long long)m2 * m3, G); note_launch();
    MFWQ_CUDA(cudaGetLastError());
  }
  unsigned long long hbad = 0;
  int hnz[6];
  MFWQ_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, sizeof(hbad), cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaMemcpyAsync(hnz, flag_.ptr, sizeof hnz, cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
  if (hbad != ~0ull) {
    long long q = (long long)hbad;
    int q1 = int(q % m1), q2 = int((q / m1) % m2), q3 = int(q / ((long long)m1 * m2));
    char msg[256];
    snprintf(msg, sizeof msg, "non-positive Jacobian determinant at parametric point (%.17g, %.17g, %.17g)",
             dir[0].pts[q1], dir[1].pts[q2], dir[2].pts[q_lo + q3]);
    throw DegenerateErr(msg);
  }
  coeffs_ready = true;
  for (int g = 0; g < 6; ++g) grid_nonzero[g] = hnz[g] != 0;
}

// On-the-fly mode: C(xi1) = C(xi1, 0, 0) by the same formula as the grids (coeff_kernel); for the
// identity and affine maps it is constant, for the quarter ring (K = I) it depends on xi1 only
// (theta drops out of det J J^-1 J^-T; theta = 0 gives the exactly diagonal value).
void Stiffness::set_on_the_fly(int kind, const double* A, const double* K9, cudaStream_t s) {
  if (kind != GEOM_IDENTITY && kind != GEOM_AFFINE && kind != GEOM_RING)
    throw NotImplErr("on-the-fly coefficients need an analytic map (identity, affine or quarter ring)");
  if (kind == GEOM_RING && K9) {
    for (int i = 0; i < 9; ++i)
      if (K9[i] != ((i % 4 == 0) ? 1.0 : 0.0))
        throw NotImplErr("on-the-fly coefficients on the quarter ring need K = I (C would depend on theta)");
  }
  geo_kind = kind;
  geo_hasK = K9 != nullptr;
  if (A) std::copy(A, A + 9, geo_A);
  if (K9) std::copy(K9, K9 + 9, geo_K);
  const int m1 = dir[0].m;
  cx.alloc(6 * (size_t)m1);
  DevBuf<double> zero(1);
  DevBuf<unsigned long long> bad(1);
  unsigned long long init = ~0ull;
  MFWQ_CUDA(cudaMemsetAsync(zero.ptr, 0, sizeof(double), s));
  MFWQ_CUDA(cudaMemcpyAsync(bad.ptr, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  const double* a = geo_A;
  const double* k = geo_K;
  coeff_kernel<<<(m1 + 127) / 128, 128, 0, s>>>(kind, dir[0].pts_d.ptr, zero.ptr, zero.ptr, m1, 1, 1, m1, a[0], a[1],
                                                a[2], a[3], a[4], a[5], a[6], a[7], a[8], geo_hasK ? 1 : 0, k[0],
                                                k[1], k[2], k[3], k[4], k[5], k[6], k[7], k[8], nullptr, nullptr,
                                                cx.ptr, (size_t)m1, bad.ptr, nullptr); note_launch();
  MFWQ_CUDA(cudaGetLastError());
  std::vector<double> h(6 * (size_t)m1);
  unsigned long long hbad = 0;
  MFWQ_CUDA(cudaMemcpyAsync(h.data(), cx.ptr, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, sizeof(hbad), cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
  if (hbad != ~0ull) {
    char msg[160];
    snprintf(msg, sizeof msg, "non-positive Jacobian determinant at parametric xi1 = %.17g", dir[0].pts[hbad]);
    throw DegenerateErr(msg);
  }
  for (int g = 0; g < 6; ++g) {
    grid_nonzero[g] = false;
    for (int q = 0; q < m1; ++q) grid_nonzero[g] = grid_nonzero[g] || h[(size_t)g * m1 + q] != 0.0;
  }
  coeff.release();
  otf = true;
  coeffs_ready = true;
  fused2_plan.reset();
  pcg_graphs.reset();
}

void Stiffness::set_coeffs(const double* const* grids, cudaStream_t s) {
  otf = false;
  pcg_graphs.reset();
  cx.release();
  // grids: 6 device arrays, unpadded (m3, m2, m1) -> repack into the padded layout
  const size_t G = grid_elems();
  coeff.alloc(6 * G);
  MFWQ_CUDA(cudaMemsetAsync(coeff.ptr, 0, 6 * G * sizeof(double), s));
  const int m1 = dir[0].m;
  for (int g = 0; g < 6; ++g)  // the slab's quadrature planes of the full (m3, m2, m1) grids
    MFWQ_CUDA(cudaMemcpy2DAsync(coeff.ptr + g * G, m1p * sizeof(double),
                                grids[g] + (size_t)q_lo * dir[1].m * m1, m1 * sizeof(double), m1 * sizeof(double),
                                (size_t)dir[1].m * (q_hi - q_lo), cudaMemcpyDeviceToDevice, s));
  coeffs_ready = true;
  detect_nonzero(s);
}

void Stiffness::get_coeffs(int g, double* out, cudaStream_t s) const {
  const size_t G = grid_elems();
  const int m1 = dir[0].m;
  MFWQ_CUDA(cudaMemcpy2DAsync(out, m1 * sizeof(double), coeff.ptr + g * G, m1p * sizeof(double),
                              m1 * sizeof(double), (size_t)dir[1].m * (q_hi - q_lo), cudaMemcpyDeviceToDevice, s));
}

void Stiffness::detect_nonzero(cudaStream_t s) {
  // Terms whose coefficient grid is identically zero contribute exact zeros
  // to w (operators.py:197-201); they are skipped.  This is exact, not an
  // approximation: W (0 * g) == 0.
  const size_t G = grid_elems();
  flag_.alloc(6);
  MFWQ_CUDA(cudaMemsetAsync(flag_.ptr, 0, 6 * sizeof(int), s));
  for (int g = 0; g < 6; ++g) {
    any_nonzero_kernel<<<148 * 4, 256, 0, s>>>(coeff.ptr + g * G, G, flag_.ptr + g); note_launch();
    MFWQ_CUDA(cudaGetLastError());
  }
  int h[6];
  MFWQ_CUDA(cudaMemcpyAsync(h, flag_.ptr, sizeof h, cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
  for (int g = 0; g < 6; ++g) grid_nonzero[g] = h[g] != 0;
}

static inline int gkey(int a, int b) {
  int lo = std::min(a, b), hi = std::max(a, b);
  static const int tab[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  return tab[lo][hi];
}

int Stiffness::term_mask() const {
  int mask = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      if (grid_nonzero[gkey(a, b)]) mask |= 1 << (3 * a + b);
  return mask;
}

// ---------------------------------------------------------------------------
// K1: generic banded one-mode contraction
//   out(.., r, ..) (+)= sum_k A[r][k] * in(.., start[r]+k, ..)
// tensors are (d3, d2, d1) with d1 fastest; ax = 0 (x), 1 (y), 2 (z)
// ---------------------------------------------------------------------------
__global__ void band_contract_kernel(const double* __restrict__ in, double* __restrict__ out, int d1, int d2,
                                     int d3, int ax, BandView A, int accumulate) {
  int o1 = ax == 0 ? A.rows : d1, o2 = ax == 1 ? A.rows : d2, o3 = ax == 2 ? A.rows : d3;
  long long total = (long long)o1 * o2 * o3;
  long long in_stride = ax == 0 ? 1 : (ax == 1 ? d1 : (long long)d1 * d2);
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total; o += (long long)gridDim.x * blockDim.x) {
    int i1 = int(o % o1);
    long long t = o / o1;
    int i2 = int(t % o2), i3 = int(t / o2);
    int r = ax == 0 ? i1 : (ax == 1 ? i2 : i3);
    long long base = ax == 0 ? ((long long)i3 * d2 + i2) * d1
                             : (ax == 1 ? (long long)i3 * d2 * d1 + i1 : (long long)i2 * d1 + i1);
    const int s = A.start[r];
    const double* a = A.vals + (size_t)r * A.width;
    double acc = 0.0;
    for (int k = 0; k < A.width; ++k) {
      int c = s + k;
      if (c < A.cols) acc += a[k] * in[base + c * in_stride];
    }
    if (accumulate) out[o] += acc; else out[o] = acc;
  }
}

__global__ void scale_kernel(const double* __restrict__ C, const double* __restrict__ g, double* __restrict__ t,
                             int m1, int m1p, long long Nq) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < Nq; q += (long long)gridDim.x * blockDim.x) {
    long long row = q / m1;
    int c = int(q % m1);
    t[q] = C[row * m1p + c] * g[q];
  }
}

static void contract(const double* in, double* out, int d1, int d2, int d3, int ax, const Band& A, int acc,
                     cudaStream_t s) {
  long long o = (long long)(ax == 0 ? A.h.rows : d1) * (ax == 1 ? A.h.rows : d2) * (ax == 2 ? A.h.rows : d3);
  int blocks = (int)std::min<long long>((o + 255) / 256, 148LL * 32);
  band_contract_kernel<<<std::max(blocks, 1), 256, 0, s>>>(in, out, d1, d2, d3, ax, A.view(), acc); note_launch();
  MFWQ_CUDA(cudaGetLastError());
}

void Stiffness::apply_generic(const double* x, double* y, cudaStream_t s) {
  if (is_slab()) throw NotImplErr("slab operators run on the fused kernel only");
  const int n1 = dir[0].n, n2 = dir[1].n, n3 = dir[2].n;
  const int m1 = dir[0].m, m2 = dir[1].m, m3 = dir[2].m;
  if (!g_.ptr) {
    g_.alloc(Nq);
    t_.alloc(Nq);
    s1_.alloc(std::max((long long)m3 * n2 * n1, (long long)n3 * m2 * m1));
    s2_.alloc(std::max((long long)m3 * m2 * n1, (long long)n3 * n2 * m1));
  }
  MFWQ_CUDA(cudaMemsetAsync(y, 0, N * sizeof(double), s));
  const size_t G = grid_elems();
  for (int b = 0; b < 3; ++b) {
    bool any = false;
    for (int a = 0; a < 3; ++a) any |= grid_nonzero[gkey(a, b)];
    if (!any) continue;
    // g_b = (B3 x B2 x B1) v, direction 3 first (kron.py:83)
    contract(x, s1_.ptr, n1, n2, n3, 2, dir[2].B[b == 2], 0, s);
    contract(s1_.ptr, s2_.ptr, n1, n2, m3, 1, dir[1].B[b == 1], 0, s);
    contract(s2_.ptr, g_.ptr, n1, m2, m3, 0, dir[0].B[b == 0], 0, s);
    for (int a = 0; a < 3; ++a) {
      int key = gkey(a, b);
      if (!grid_nonzero[key]) continue;
      int blocks = (int)std::min<long long>((Nq + 255) / 256, 148LL * 32);
      scale_kernel<<<blocks, 256, 0, s>>>(coeff.ptr + key * G, g_.ptr, t_.ptr, m1, m1p, Nq); note_launch();
      MFWQ_CUDA(cudaGetLastError());
      auto widx = [&](int l) { return 2 * (l == a) + (l == b); };
      contract(t_.ptr, s1_.ptr, m1, m2, m3, 2, dir[2].W[widx(2)], 0, s);
      contract(s1_.ptr, s2_.ptr, m1, m2, n3, 1, dir[1].W[widx(1)], 0, s);
      contract(s2_.ptr, y, m1, n2, n3, 0, dir[0].W[widx(0)], 1, s);
    }
  }
}

// ---------------------------------------------------------------------------
// Mass operator (operators.py:46-61, 87-132), composed from the K1 band contractions
// ---------------------------------------------------------------------------
__global__ void mass_coeff_kernel(int kind, const double* __restrict__ x1, const double* __restrict__ x2, int m1,
                                  int m2, int m3, int m1p, double A00, double A01, double A02, double A10, double A11,
                                  double A12, double A20, double A21, double A22, const double* __restrict__ Jfield,
                                  double alpha, const double* __restrict__ afield, double* __restrict__ out,
                                  unsigned long long* bad) {
  const long long Nq = (long long)m1 * m2 * m3;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < Nq; q += (long long)gridDim.x * blockDim.x) {
    const int q1 = int(q % m1);
    const long long r = q / m1;
    const int q2 = int(r % m2);
    double det;
    if (kind == GEOM_IDENTITY) {
      det = 1.0;
    } else if (kind == GEOM_AFFINE) {
      det = A00 * (A11 * A22 - A12 * A21) + A01 * (A12 * A20 - A10 * A22) + A02 * (A10 * A21 - A11 * A20);
    } else if (kind == GEOM_RING) {  // geometry.py:84-94: det J = (pi/2) r (cos^2 + sin^2)
      const double rr = 1.0 + x1[q1];
      double sn, cs;
      sincos(M_PI / 2 * x2[q2], &sn, &cs);
      det = cs * (M_PI / 2 * rr * cs) + (M_PI / 2 * rr * sn) * sn;
    } else {
      const double* J = Jfield + 9 * q;
      det = J[0] * (J[4] * J[8] - J[5] * J[7]) + J[1] * (J[5] * J[6] - J[3] * J[8]) + J[2] * (J[3] * J[7] - J[4] * J[6]);
    }
    if (!(det > 0.0)) atomicMin(bad, (unsigned long long)q);
    out[(r / m2 * m2 + q2) * (long long)m1p + q1] = (afield ? afield[q] : alpha) * det;
  }
}

void Stiffness::set_mass(int kind, const double* A, const double* J_dev, double alpha, const double* afield,
                         int on_the_fly, cudaStream_t s) {
  if (is_slab()) throw NotImplErr("the mass operator is not slab-partitioned");
  if (kind == GEOM_JACOBIAN && on_the_fly) throw NotImplErr("on-the-fly mass needs an analytic map");
  geo_kind = kind;
  if (A) std::copy(A, A + 9, geo_A);
  mass_alpha = alpha;
  mass_alpha_field = afield;
  mass_otf = on_the_fly != 0;
  mass_grid.release();
  if (!mass_otf) {
    mass_grid.alloc(grid_elems());
    eval_mass(mass_grid.ptr, J_dev, s);
  }
  mass_ready = true;
}

void Stiffness::eval_mass(double* out, const double* J_dev, cudaStream_t s) {
  const int m1 = dir[0].m, m2 = dir[1].m, m3 = dir[2].m;
  DevBuf<unsigned long long> bad(1);
  unsigned long long init = ~0ull;
  MFWQ_CUDA(cudaMemcpyAsync(bad.ptr, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (m1p > m1) MFWQ_CUDA(cudaMemsetAsync(out, 0, grid_elems() * sizeof(double), s));
  const double* a = geo_A;
  const int blocks = (int)std::min<long long>((Nq + 255) / 256, 148LL * 16);
  mass_coeff_kernel<<<blocks, 256, 0, s>>>(geo_kind, dir[0].pts_d.ptr, dir[1].pts_d.ptr, m1, m2, m3, m1p, a[0], a[1],
                                           a[2], a[3], a[4], a[5], a[6], a[7], a[8], J_dev, mass_alpha,
                                           mass_alpha_field, out, bad.ptr); note_launch();
  MFWQ_CUDA(cudaGetLastError());
  unsigned long long hbad = 0;
  MFWQ_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, sizeof(hbad), cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
  if (hbad != ~0ull) {
    const long long q = (long long)hbad;
    char msg[256];
    snprintf(msg, sizeof msg, "non-positive Jacobian determinant at parametric point (%.17g, %.17g, %.17g)",
             dir[0].pts[q % m1], dir[1].pts[(q / m1) % m2], dir[2].pts[q / ((long long)m1 * m2)]);
    throw DegenerateErr(msg);
  }
}

// w = (W00 x W00 x W00)(m o (B0 x B0 x B0) v), contracted direction 3 first (kron.py:83)
void Stiffness::apply_mass(const double* x, double* y, cudaStream_t s) {
  if (!mass_ready) throw ValueErr("mass coefficients not set");
  // the fused kernel's one-term case on the stored alpha det J grid; the composed K1 path below
  // serves on-the-fly mass, path = generic, and rules outside the element-blocked structure
  if (!mass_otf && path != 1 && fused2_apply_mass(*this, x, y, s)) return;
  const int n1 = dir[0].n, n2 = dir[1].n, n3 = dir[2].n;
  const int m1 = dir[0].m, m2 = dir[1].m, m3 = dir[2].m;
  if (!g_.ptr) {
    g_.alloc(Nq);
    t_.alloc(Nq);
    s1_.alloc(std::max((long long)m3 * n2 * n1, (long long)n3 * m2 * m1));
    s2_.alloc(std::max((long long)m3 * m2 * n1, (long long)n3 * n2 * m1));
  }
  DevBuf<double> fly;
  const double* m = mass_grid.ptr;
  if (mass_otf) {  // operators.py:121-125: evaluated for this apply and dropped
    fly.alloc(grid_elems());
    eval_mass(fly.ptr, nullptr, s);
    m = fly.ptr;
  }
  contract(x, s1_.ptr, n1, n2, n3, 2, dir[2].B[0], 0, s);
  contract(s1_.ptr, s2_.ptr, n1, n2, m3, 1, dir[1].B[0], 0, s);
  contract(s2_.ptr, g_.ptr, n1, m2, m3, 0, dir[0].B[0], 0, s);
  const int blocks = (int)std::min<long long>((Nq + 255) / 256, 148LL * 32);
  scale_kernel<<<blocks, 256, 0, s>>>(m, g_.ptr, t_.ptr, m1, m1p, Nq); note_launch();
  MFWQ_CUDA(cudaGetLastError());
  contract(t_.ptr, s1_.ptr, m1, m2, m3, 2, dir[2].W[0], 0, s);
  contract(s1_.ptr, s2_.ptr, m1, m2, n3, 1, dir[1].W[0], 0, s);
  contract(s2_.ptr, y, m1, n2, n3, 0, dir[0].W[0], 0, s);
}

// CostMeter count of one mass apply (operators.py:118-132): S(B0) + N_q + S(W00)
long long Stiffness::mass_flops() const {
  const long long n1 = dir[0].n, n2 = dir[1].n, n3 = dir[2].n;
  const long long m1 = dir[0].m, m2 = dir[1].m, m3 = dir[2].m;
  auto S = [&](long long z1, long long z2, long long z3, long long s2, long long s3, long long t1, long long t2) {
    return 2 * z3 * t1 * t2 + 2 * z2 * s3 * t1 + 2 * z1 * s3 * s2;
  };
  return S(nnz_[0][0], nnz_[1][0], nnz_[2][0], m2, m3, n1, n2) + Nq +
         S(nnz_[0][2], nnz_[1][2], nnz_[2][2], n2, n3, m1, m2);
}

void Stiffness::apply(const double* x, double* y, cudaStream_t s) {
  if (!coeffs_ready) throw ValueErr("coefficient grids not set");
  if (otf) {
    if (path != 1 && fused2_apply(*this, x, y, s)) return;
    // the element-blocked kernel cannot take this rule (or a composed path was asked for): evaluate
    // the grids for this apply only, as the reference's on-the-fly mode does per grid
    bool nz[6];
    std::copy(grid_nonzero, grid_nonzero + 6, nz);
    const double* K9 = geo_hasK ? geo_K : nullptr;
    DevBuf<double> keep;
    std::swap(keep.ptr, cx.ptr);
    std::swap(keep.n, cx.n);
    set_geometry(geo_kind, geo_A, K9, nullptr, nullptr, s);
    std::copy(nz, nz + 6, grid_nonzero);
    if (path == 1) apply_generic(x, y, s);
    else apply_fused(x, y, s);
    coeff.release();
    std::swap(keep.ptr, cx.ptr);
    std::swap(keep.n, cx.n);
    otf = true;
    fused2_plan.reset();
    return;
  }
  if (path == 1) { apply_generic(x, y, s); return; }
  apply_fused(x, y, s);
}

}  // namespace mfwq

namespace mfwq {
// Dense Kronecker apply (A_d x ... x A_1) x on the device, direction d first
// (kron.py:70-100); test/utility entry point built on the K1 kernel.
void kron_apply_dense(int d, const int* rows, const int* cols, const double* const* A, const double* x, double* y,
                      int accumulate, cudaStream_t s) {
  if (d < 1 || d > 3) throw ValueErr("kron_apply supports 1 to 3 factors");
  Band bands[3];
  int in_dims[3] = {1, 1, 1};  // (d1, d2, d3)
  for (int l = 0; l < d; ++l) {
    BandHost& b = bands[l].h;
    b.rows = rows[l];
    b.cols = cols[l];
    b.width = cols[l];
    b.start.assign(rows[l], 0);
    b.vals.assign(A[l], A[l] + size_t(rows[l]) * cols[l]);
    bands[l].upload();
    in_dims[l] = cols[l];
  }
  long long mx = 1;
  {
    int dims[3] = {in_dims[0], in_dims[1], in_dims[2]};
    for (int l = d - 1; l >= 0; --l) {
      dims[l] = rows[l];
      mx = std::max(mx, (long long)dims[0] * dims[1] * dims[2]);
    }
    mx = std::max(mx, (long long)in_dims[0] * in_dims[1] * in_dims[2]);
  }
  DevBuf<double> b0(mx), b1(mx);
  const double* cur = x;
  int dims[3] = {in_dims[0], in_dims[1], in_dims[2]};
  for (int l = d - 1; l >= 0; --l) {
    const bool last = l == 0;
    double* dst = last ? y : ((d - 1 - l) % 2 == 0 ? b0.ptr : b1.ptr);
    contract(cur, dst, dims[0], dims[1], dims[2], l, bands[l], last ? accumulate : 0, s);
    dims[l] = rows[l];
    cur = dst;
  }
  MFWQ_CUDA(cudaStreamSynchronize(s));
}
}  // namespace mfwq
