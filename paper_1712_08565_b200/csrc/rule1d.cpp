// Host-side univariate setup: B-spline collocation, weighted-quadrature
// points and weights, exact 1D stiffness/mass.  This is the native
// replacement of the reference's Python setup that feeds the hot path:
//   splines.py:74-192  (span search, Cox-de Boor values/derivatives, collocation)
//   wq.py:41-164       (Gauss rule, exact Gram, WQ points, per-row min-norm
//                       least-squares weights, boundary-point retry loop)
//   solvers.py:48-62   (exact interior 1D stiffness/mass for FD)
// Min-norm least squares: LAPACK dgelsd with np.linalg.lstsq's calling sequence when the host
// process registers a LAPACK (mfwq_set_lapack), else a one-sided Jacobi SVD with numpy's default
// truncation (rcond = eps * max(rows, cols)).
#include "rule1d.h"

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <stdexcept>
#include <string>

namespace mfwq {

static const double kExactnessTol = 1e-10;  // wq.py:25

Knots::Knots(int p_, const double* t_, int nt) : p(p_), t(t_, t_ + nt) {
  if (p < 1) throw ValueErr("degree must be >= 1");
  if (nt < 2 * (p + 1)) throw ValueErr("knot vector too short for the given degree");
  for (int i = 1; i < nt; ++i)
    if (t[i] < t[i - 1]) throw ValueErr("knots must be nondecreasing");
  if (t[0] != 0.0 || t[nt - 1] != 1.0) throw ValueErr("knot vector must start at 0 and end at 1");
  for (int i = 0; i <= p; ++i)
    if (t[i] != 0.0 || t[nt - 1 - i] != 1.0) throw ValueErr("knot vector must be open");
  if (t[p + 1] == 0.0 || t[nt - p - 2] == 1.0) throw ValueErr("endpoint multiplicity must be exactly p+1");
  brk.push_back(t[0]);
  for (int i = 1; i < nt; ++i)
    if (t[i] != brk.back()) brk.push_back(t[i]);
}

// splines.py:74-85: right-continuous span, left limit at x = 1
int Knots::span(double x) const {
  int k = int(std::upper_bound(t.begin(), t.end(), x) - t.begin()) - 1;
  return std::min(std::max(k, p), nfun() - 1);
}

// Cox-de Boor triangle for degree `deg` (splines.py:99-116)
static void basis_vals(const std::vector<double>& t, int deg, double x, int s, double* N) {
  double L[32], R[32];
  N[0] = 1.0;
  for (int j = 1; j <= deg; ++j) {
    L[j] = x - t[s + 1 - j];
    R[j] = t[s + j] - x;
    double carry = 0.0;
    for (int r = 0; r < j; ++r) {
      double den = R[r + 1] + L[j - r];
      double tmp = den != 0.0 ? N[r] / den : 0.0;
      N[r] = carry + R[r + 1] * tmp;
      carry = L[j - r] * tmp;
    }
    N[j] = carry;
  }
}

// two-term derivative formula on the degree p-1 values (splines.py:119-162)
static void basis_d1(const std::vector<double>& t, int p, double x, int s, double* D) {
  double low[32];
  if (p == 1) low[0] = 1.0; else basis_vals(t, p - 1, x, s, low);
  const int first = s - p + 1;
  for (int a = 0; a <= p; ++a) {
    int i = s - p + a;
    double acc = 0.0;
    if (i >= first && i <= s) {
      double den = t[i + p] - t[i];
      if (den != 0.0) acc += p * low[i - first] / den;
    }
    if (i + 1 >= first && i + 1 <= s) {
      double den = t[i + p + 1] - t[i + 1];
      if (den != 0.0) acc -= p * low[i + 1 - first] / den;
    }
    D[a] = acc;
  }
}

// collocation_matrix (splines.py:165-192): rows = points, zeros eliminated
Csr collocation(const Knots& kv, const std::vector<double>& x, int deriv) {
  const int p = kv.p;
  Csr A;
  A.rows = int(x.size());
  A.cols = kv.nfun();
  A.indptr.assign(1, 0);
  double v[32];
  for (double xq : x) {
    if (xq < 0.0 || xq > 1.0) throw ValueErr("point outside [0, 1]");
    int s = kv.span(xq);
    if (deriv == 0) basis_vals(kv.t, p, xq, s, v); else basis_d1(kv.t, p, xq, s, v);
    for (int a = 0; a <= p; ++a)
      if (v[a] != 0.0) { A.indices.push_back(s - p + a); A.data.push_back(v[a]); }
    A.indptr.push_back(int(A.indices.size()));
  }
  return A;
}

// numpy's pairwise summation of a contiguous double array (np.sum; numpy/_core loops_utils):
// fewer than 8 values sequentially from -0.0, up to 128 in eight interleaved partial sums
static double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double r = -0.0;
    for (int i = 0; i < n; ++i) r += a[i];
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[i];
  return res;
}

// numpy.polynomial.legendre.legval for the coefficient vector c (length nc), Clenshaw form
static double np_legval(double x, const double* c, int nc) {
  if (nc == 1) return c[0] + 0.0 * x;
  if (nc == 2) return c[0] + c[1] * x;
  int nd = nc;
  double c0 = c[nc - 2], c1 = c[nc - 1];
  for (int i = 3; i <= nc; ++i) {
    const double tmp = c0;
    nd = nd - 1;
    c0 = c[nc - i] - c1 * (double(nd - 1) / double(nd));
    c1 = tmp + c1 * x * (double(2 * nd - 1) / double(nd));
  }
  return c0 + c1 * x;
}

// numpy.polynomial.legendre.leggauss, operation for operation: eigenvalues of the scaled
// companion matrix (LAPACK dsyevd, as np.linalg.eigvalsh), one Newton step, weights from
// L_{n-1} and L_n' (the latter at the unrefined roots), symmetrised and scaled by 2 / np.sum.
// The reference's Gauss rules (wq.py:41-49) come from it, so the exact Gram matrices and with
// them the WQ right-hand sides are bit-identical.
static dsyevd64_t g_dsyevd = nullptr;
static bool leggauss_numpy(int n, std::vector<double>& z, std::vector<double>& w) {
  if (!g_dsyevd) return false;
  if (n == 1) {
    z.assign(1, 0.0);
    w.assign(1, 2.0);
    return true;
  }
  typedef long long i64;
  std::vector<double> mat(size_t(n) * n, 0.0), scl(n), x(n);
  for (int k = 0; k < n; ++k) scl[k] = 1.0 / std::sqrt(double(2 * k + 1));
  for (int k = 1; k < n; ++k) mat[size_t(k - 1) * n + k] = mat[size_t(k) * n + k - 1] = double(k) * scl[k - 1] * scl[k];
  {  // np.linalg.eigvalsh(m) (UPLO='L', workspace query first); m is symmetric
    const char jobz = 'N', uplo = 'L';
    i64 N = n, lda = n, lwork = -1, liwork = -1, info = 0, iwq = 0;
    double wq = 0.0;
    g_dsyevd(&jobz, &uplo, &N, mat.data(), &lda, x.data(), &wq, &lwork, &iwq, &liwork, &info, 1, 1);
    if (info != 0) return false;
    lwork = i64(wq);
    liwork = iwq;
    std::vector<double> work(size_t(std::max<i64>(lwork, 1)));
    std::vector<i64> iwork(size_t(std::max<i64>(liwork, 1)));
    g_dsyevd(&jobz, &uplo, &N, mat.data(), &lda, x.data(), work.data(), &lwork, iwork.data(), &liwork, &info, 1, 1);
    if (info != 0) return false;
  }
  std::vector<double> c(n + 1, 0.0), der(n), cc(n + 1);
  c[n] = 1.0;
  cc = c;  // legder(c): derivative coefficients
  for (int j = n; j > 2; --j) {
    der[j - 1] = double(2 * j - 1) * cc[j];
    cc[j - 2] += cc[j];
  }
  if (n > 1) der[1] = 3.0 * cc[2];
  der[0] = cc[1];
  std::vector<double> dy(n), df(n), fm(n), ww(n);
  for (int k = 0; k < n; ++k) {
    dy[k] = np_legval(x[k], c.data(), n + 1);
    df[k] = np_legval(x[k], der.data(), n);
  }
  for (int k = 0; k < n; ++k) x[k] -= dy[k] / df[k];
  double fmax = 0.0, dmax = 0.0;
  for (int k = 0; k < n; ++k) {
    fm[k] = np_legval(x[k], c.data() + 1, n);
    fmax = std::max(fmax, std::fabs(fm[k]));
    dmax = std::max(dmax, std::fabs(df[k]));
  }
  for (int k = 0; k < n; ++k) {
    fm[k] /= fmax;
    df[k] /= dmax;
    ww[k] = 1.0 / (fm[k] * df[k]);
  }
  z.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int k = 0; k < n; ++k) {
    w[k] = (ww[k] + ww[n - 1 - k]) / 2.0;
    z[k] = (x[k] - x[n - 1 - k]) / 2.0;
  }
  const double f = 2.0 / np_pairwise_sum(w.data(), n);
  for (int k = 0; k < n; ++k) w[k] *= f;
  return true;
}

// Gauss-Legendre on [-1,1]: numpy's leggauss when a LAPACK is registered, else Newton on P_n
static void legendre(int n, std::vector<double>& z, std::vector<double>& w) {
  if (leggauss_numpy(n, z, w)) return;
  z.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
      if (n == 1) { p1 = x; p0 = 1.0; }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-17) break;
    }
    double p0 = 1.0, p1 = x;
    for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
    if (n == 1) { p1 = x; p0 = 1.0; }
    dp = n * (x * p1 - p0) / (x * x - 1.0);
    z[n - 1 - i] = x;
    w[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  for (int i = 0; i < n / 2; ++i) {  // exact symmetry, as leggauss
    double a = 0.5 * (z[n - 1 - i] - z[i]), b = 0.5 * (w[i] + w[n - 1 - i]);
    z[i] = -a; z[n - 1 - i] = a; w[i] = w[n - 1 - i] = b;
  }
  if (n % 2) z[n / 2] = 0.0;
}

// wq.py:41-49
void gauss_rule(const Knots& kv, int npts, std::vector<double>& x, std::vector<double>& w) {
  std::vector<double> z, wz;
  legendre(npts, z, wz);
  x.clear(); w.clear();
  for (size_t e = 0; e + 1 < kv.brk.size(); ++e) {
    double a = kv.brk[e], b = kv.brk[e + 1];
    for (int k = 0; k < npts; ++k) {
      x.push_back((a + b) / 2 + (b - a) / 2 * z[k]);
      w.push_back((b - a) / 2 * wz[k]);
    }
  }
}

// dense (nfun x nfun) exact Gram  int D^a b_i D^b b_j  (wq.py:52-59)
static std::vector<double> exact_gram(const Knots& kv, int a, int b) {
  std::vector<double> x, w;
  gauss_rule(kv, kv.p + 1, x, w);
  Csr Ba = collocation(kv, x, a), Bb = collocation(kv, x, b);
  const int n = kv.nfun();
  std::vector<double> G(size_t(n) * n, 0.0);
  for (int q = 0; q < Ba.rows; ++q)
    for (int u = Ba.indptr[q]; u < Ba.indptr[q + 1]; ++u)
      for (int v = Bb.indptr[q]; v < Bb.indptr[q + 1]; ++v)
        G[size_t(Ba.indices[u]) * n + Bb.indices[v]] += Ba.data[u] * w[q] * Bb.data[v];
  return G;
}

// wq.py:62-83
std::vector<double> wq_points(const Knots& kv, int extra) {
  std::vector<double> pts(kv.brk);
  for (size_t e = 0; e + 1 < kv.brk.size(); ++e) pts.push_back(0.5 * (kv.brk[e] + kv.brk[e + 1]));
  if (extra > 0 && kv.brk.size() >= 2) {
    const size_t nb = kv.brk.size();
    double spans[2][2] = {{kv.brk[0], kv.brk[1]}, {kv.brk[nb - 2], kv.brk[nb - 1]}};
    for (auto& ab : spans)
      for (int k = 1; k <= extra; ++k)  // np.linspace(a, b, extra+2)[1:-1]
        pts.push_back(ab[0] + k * ((ab[1] - ab[0]) / (extra + 1)));
  }
  std::sort(pts.begin(), pts.end());
  std::vector<double> out{pts[0]};
  for (size_t i = 1; i < pts.size(); ++i)
    if (pts[i] - pts[i - 1] > 1e-12) out.push_back(pts[i]);
  return out;
}

// LAPACK dgelsd (ILP64 interface), the driver np.linalg.lstsq calls (wq.py:97).  When the host
// process provides one (mfwq_set_lapack: numpy's own bundled LAPACK), the rows are solved by it
// with numpy's exact calling sequence, so the weights are the reference's bit for bit; otherwise
// the self-contained Jacobi SVD below is used (same truncation rule, conditioning-limited agreement).
static dgelsd64_t g_dgelsd = nullptr;
void set_lapack(dgelsd64_t gelsd, dsyevd64_t syevd) {
  g_dgelsd = gelsd;
  g_dsyevd = syevd;
}
bool have_dgelsd() { return g_dgelsd != nullptr && g_dsyevd != nullptr; }

// numpy/linalg/umath_linalg.cpp (lstsq gufunc): A copied column-major, b into a max(m, n) x 1
// buffer, workspace sizes from an LWORK = -1 query, rcond = eps * max(m, n) (np.linalg.lstsq with
// rcond=None); the solution is the first n entries of the b buffer.
static void lstsq_dgelsd(int r, int c, const double* E, const double* g, double* w) {
  typedef long long i64;
  i64 m = r, n = c, nrhs = 1, lda = std::max<i64>(m, 1), ldb = std::max<i64>(std::max(m, n), 1), rank = 0,
      info = 0, lwork = -1;
  std::vector<double> A(size_t(m) * n), B(size_t(ldb), 0.0), S(size_t(std::min(m, n)));
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < m; ++i) A[size_t(j * m + i)] = E[size_t(i) * c + j];
  for (i64 i = 0; i < m; ++i) B[size_t(i)] = g[i];
  const double rcond = 2.220446049250313e-16 * double(std::max(m, n));
  double wq = 0.0;
  i64 iwq = 0;
  g_dgelsd(&m, &n, &nrhs, A.data(), &lda, B.data(), &ldb, S.data(), &rcond, &rank, &wq, &lwork, &iwq, &info);
  if (info != 0) throw ValueErr("dgelsd workspace query failed (info " + std::to_string(info) + ")");
  lwork = i64(wq);
  std::vector<double> work(size_t(std::max<i64>(lwork, 1)));
  std::vector<i64> iwork(size_t(std::max<i64>(iwq, 1)));
  g_dgelsd(&m, &n, &nrhs, A.data(), &lda, B.data(), &ldb, S.data(), &rcond, &rank, work.data(), &lwork,
           iwork.data(), &info);
  if (info != 0) throw ValueErr("dgelsd: SVD did not converge (info " + std::to_string(info) + ")");
  for (i64 j = 0; j < n; ++j) w[j] = B[size_t(j)];
}

// min-norm least squares E w = g (E: r x c, row-major) via one-sided Jacobi
// SVD of E^T; singular values <= eps*max(r,c)*smax are dropped (gelsd rule).
static void minnorm_lstsq(int r, int c, const double* E, const double* g, double* w) {
  if (g_dgelsd) {
    lstsq_dgelsd(r, c, E, g, w);
    return;
  }
  // A = E^T (c x r), columns a_k = row k of E
  std::vector<double> A(E, E + size_t(r) * c);  // A[k*c + i] = column k of E^T
  std::vector<double> V(size_t(r) * r, 0.0);
  for (int k = 0; k < r; ++k) V[size_t(k) * r + k] = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0;
    for (int j = 0; j < r; ++j)
      for (int k = j + 1; k < r; ++k) {
        double *aj = &A[size_t(j) * c], *ak = &A[size_t(k) * c];
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < c; ++i) { al += aj[i] * aj[i]; be += ak[i] * ak[i]; ga += aj[i] * ak[i]; }
        if (ga == 0.0 || std::fabs(ga) <= 1e-17 * std::sqrt(al * be)) continue;
        off = std::max(off, std::fabs(ga) / std::sqrt(al * be));
        double zeta = (be - al) / (2 * ga);
        double tt = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1 + zeta * zeta));
        double cs = 1 / std::sqrt(1 + tt * tt), sn = cs * tt;
        for (int i = 0; i < c; ++i) { double x = aj[i], y = ak[i]; aj[i] = cs * x - sn * y; ak[i] = sn * x + cs * y; }
        double *vj = &V[size_t(j) * r], *vk = &V[size_t(k) * r];
        for (int i = 0; i < r; ++i) { double x = vj[i], y = vk[i]; vj[i] = cs * x - sn * y; vk[i] = sn * x + cs * y; }
      }
    if (off < 1e-16) break;
  }
  std::vector<double> s(r);
  double smax = 0;
  for (int k = 0; k < r; ++k) {
    double nn = 0;
    for (int i = 0; i < c; ++i) nn += A[size_t(k) * c + i] * A[size_t(k) * c + i];
    s[k] = std::sqrt(nn);
    smax = std::max(smax, s[k]);
  }
  const double thr = 2.220446049250313e-16 * std::max(r, c) * smax;
  for (int i = 0; i < c; ++i) w[i] = 0.0;
  // E = V S U^T with U_k = a_k / s_k  =>  w = sum_k U_k (V_k . g) / s_k
  for (int k = 0; k < r; ++k) {
    if (!(s[k] > thr)) continue;
    double vg = 0;
    for (int i = 0; i < r; ++i) vg += V[size_t(k) * r + i] * g[i];
    double f = vg / (s[k] * s[k]);
    for (int i = 0; i < c; ++i) w[i] += A[size_t(k) * c + i] * f;
  }
}

struct WQFail { int row; double resid; };

// wq.py:86-123 for all rows of one (a, b) family
static Csr wq_matrix(const Knots& kv, const std::vector<double>& pts, int a, int b) {
  const int n = kv.nfun(), nq = int(pts.size());
  Csr Cb = collocation(kv, pts, b);
  std::vector<double> colb(size_t(n) * nq, 0.0);  // (nfun x npts) dense
  for (int q = 0; q < nq; ++q)
    for (int u = Cb.indptr[q]; u < Cb.indptr[q + 1]; ++u) colb[size_t(Cb.indices[u]) * nq + q] = Cb.data[u];
  std::vector<double> G = exact_gram(kv, a, b);
  // rows are independent least-squares problems: solve them on all host cores, then assemble the
  // CSR in row order and report the first failing row, exactly like the sequential loop
  std::vector<std::vector<int>> rq(n);
  std::vector<std::vector<double>> rw(n);
  std::vector<double> rres(n, 0.0);
  auto solve_row = [&](int i, std::vector<double>& E, std::vector<double>& g, std::vector<int>& js) {
    double lo = kv.t[i], hi = kv.t[i + kv.p + 1];
    std::vector<int>& qs = rq[i];
    js.clear();
    for (int q = 0; q < nq; ++q)
      if (pts[q] >= lo - 1e-14 && pts[q] <= hi + 1e-14) qs.push_back(q);
    for (int j = 0; j < n; ++j)
      if (kv.t[j + kv.p + 1] > lo + 1e-14 && kv.t[j] < hi - 1e-14) js.push_back(j);
    const int r = int(js.size()), c = int(qs.size());
    E.assign(size_t(r) * c, 0.0);
    g.assign(r, 0.0);
    std::vector<double>& w = rw[i];
    w.assign(c, 0.0);
    for (int u = 0; u < r; ++u) {
      for (int v = 0; v < c; ++v) E[size_t(u) * c + v] = colb[size_t(js[u]) * nq + qs[v]];
      g[u] = G[size_t(i) * n + js[u]];
    }
    if (r > 0 && c > 0) minnorm_lstsq(r, c, E.data(), g.data(), w.data());
    double res = 0.0;
    for (int u = 0; u < r; ++u) {
      double acc = 0;
      for (int v = 0; v < c; ++v) acc += E[size_t(u) * c + v] * w[v];
      res = std::max(res, std::fabs(acc - g[u]));
    }
    rres[i] = res;
  };
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nth = int(std::min<unsigned>(hw, unsigned(std::max(1, n / 16))));
  std::atomic<int> next{0};
  auto worker = [&]() {
    std::vector<double> E, g;
    std::vector<int> js;
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) solve_row(i, E, g, js);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nth; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  Csr W;
  W.rows = n;
  W.cols = nq;
  W.indptr.assign(1, 0);
  for (int i = 0; i < n; ++i) {
    if (rres[i] > kExactnessTol) throw WQFail{i, rres[i]};
    for (size_t v = 0; v < rq[i].size(); ++v) { W.indices.push_back(rq[i][v]); W.data.push_back(rw[i][v]); }
    W.indptr.push_back(int(W.indices.size()));
  }
  return W;
}

// wq.py:144-164: default point set, retry with more boundary points
Rule1D build_rule(const Knots& kv) {
  // wq.py:72-73: interior knot multiplicity must be 1
  const size_t lo = size_t(kv.p) + 1, hi = kv.t.size() - size_t(kv.p) - 1;  // interior = t[lo:hi]
  for (size_t i = lo; i + 1 < hi; ++i)
    if (kv.t[i + 1] == kv.t[i]) throw ValueErr("weighted quadrature requires interior multiplicity 1");
  WQFail last{-1, 0.0};
  for (int extra = std::max(kv.p - 1, 0); extra <= 3 * kv.p; ++extra) {
    Rule1D R;
    R.extra = extra;
    R.pts = wq_points(kv, extra);
    try {
      const int ab[4][2] = {{0, 0}, {0, 1}, {1, 0}, {1, 1}};
      for (int k = 0; k < 4; ++k) R.W[k] = wq_matrix(kv, R.pts, ab[k][0], ab[k][1]);
    } catch (const WQFail& f) {
      last = f;
      continue;
    }
    R.B[0] = collocation(kv, R.pts, 0);
    R.B[1] = collocation(kv, R.pts, 1);
    return R;
  }
  throw WQErr("exactness system for row " + std::to_string(last.row) + " unsolvable (residual " +
              std::to_string(last.resid) + ")");
}

// solvers.py:48-62 (interior = drop first/last function)
void univariate_km(const Knots& kv, std::vector<double>& K, std::vector<double>& M) {
  std::vector<double> x, w;
  gauss_rule(kv, kv.p + 1, x, w);
  Csr B0 = collocation(kv, x, 0), B1 = collocation(kv, x, 1);
  const int n = kv.nfun() - 2;
  K.assign(size_t(n) * n, 0.0);
  M.assign(size_t(n) * n, 0.0);
  auto acc = [&](const Csr& B, std::vector<double>& T) {
    for (int q = 0; q < B.rows; ++q)
      for (int u = B.indptr[q]; u < B.indptr[q + 1]; ++u) {
        int i = B.indices[u] - 1;
        if (i < 0 || i >= n) continue;
        for (int v = B.indptr[q]; v < B.indptr[q + 1]; ++v) {
          int j = B.indices[v] - 1;
          if (j < 0 || j >= n) continue;
          T[size_t(i) * n + j] += B.data[u] * w[q] * B.data[v];
        }
      }
  };
  acc(B1, K);
  acc(B0, M);
}

}  // namespace mfwq
