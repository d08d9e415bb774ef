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

Csr collocation(const Knots& kv, const std::vector<double>& x, int deriv);
void gauss_rule(const Knots& kv, int npts, std::vector<double>& x, std::vector<double>& w);
std::vector<double> wq_points(const Knots& kv, int extra);
Rule1D build_rule(const Knots& kv);
void univariate_km(const Knots& kv, std::vector<double>& K, std::vector<double>& M);

}  // namespace mfwq
