// Host-side univariate spline / weighted-quadrature setup (see rule1d.cpp).
#pragma once
#include <stdexcept>
#include <string>
#include <vector>

namespace mfwq {

// Exception types mapped 1:1 onto the reference's Python exceptions by the C-ABI.
struct ValueErr : std::runtime_error { using std::runtime_error::runtime_error; };       // ValueError
struct WQErr : std::runtime_error { using std::runtime_error::runtime_error; };          // WQConstructionError
struct DegenerateErr : std::runtime_error { using std::runtime_error::runtime_error; };  // DegenerateGeometryError
struct EigenErr : std::runtime_error { using std::runtime_error::runtime_error; };       // EigenSolveError
struct IndefiniteErr : std::runtime_error { using std::runtime_error::runtime_error; };  // IndefiniteOperatorError
struct CudaErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct NotImplErr : std::runtime_error { using std::runtime_error::runtime_error; };

struct Csr {
  int rows = 0, cols = 0;
  std::vector<int> indptr, indices;
  std::vector<double> data;
};

struct Knots {
  int p;
  std::vector<double> t, brk;
  Knots(int p, const double* t, int nt);
  int nfun() const { return int(t.size()) - p - 1; }
  int n_el() const { return int(brk.size()) - 1; }
  int span(double x) const;
};

struct Rule1D {
  int extra = 0;
  std::vector<double> pts;
  Csr W[4];  // (a,b) = (0,0),(0,1),(1,0),(1,1): nfun x npts
  Csr B[2];  // deriv 0, 1: npts x nfun
};

// LAPACK dgelsd, ILP64 (all integers 64-bit), Fortran calling convention
typedef void (*dgelsd64_t)(const long long* m, const long long* n, const long long* nrhs, double* a,
                           const long long* lda, double* b, const long long* ldb, double* s, const double* rcond,
                           long long* rank, double* work, const long long* lwork, long long* iwork, long long* info);
// LAPACK dsyevd, ILP64, Fortran convention (+ the two hidden character-argument lengths)
typedef void (*dsyevd64_t)(const char* jobz, const char* uplo, const long long* n, double* a, const long long* lda,
                           double* w, double* work, const long long* lwork, long long* iwork,
                           const long long* liwork, long long* info, unsigned long jobz_len, unsigned long uplo_len);
// register (both) or clear (nullptr) the host LAPACK used for bit-exact numpy parity
void set_lapack(dgelsd64_t gelsd, dsyevd64_t syevd);
bool have_dgelsd();

Csr collocation(const Knots& kv, const std::vector<double>& x, int deriv);
void gauss_rule(const Knots& kv, int npts, std::vector<double>& x, std::vector<double>& w);
std::vector<double> wq_points(const Knots& kv, int extra);
Rule1D build_rule(const Knots& kv);
void univariate_km(const Knots& kv, std::vector<double>& K, std::vector<double>& M);

}  // namespace mfwq
