// Internal C++ interfaces of the MF-WQ B200 library (no CUDA syntax here).
#pragma once
#include <cuda_runtime.h>

#include <array>
#include <memory>
#include <vector>

#include "common.cuh"

namespace mfwq {

enum GeomKind { GEOM_IDENTITY = 0, GEOM_RING = 1, GEOM_AFFINE = 2, GEOM_JACOBIAN = 3 };

// Per-direction data of the tensor-product WQ discretisation.
struct Dir1D {
  int p = 0, n_el = 0;
  int n = 0;  // interior DoFs
  int m = 0;  // quadrature points
  std::vector<double> knots, pts;
  std::vector<int> elem_q0;  // first q of element e (size n_el+1, last = m)
  Band B[2];                 // (m x n) interior columns of colloc[0], colloc[1]
  Band W[4];                 // (n x m) interior rows of weights (0,0),(0,1),(1,0),(1,1)
  DevBuf<double> pts_d;
};

class Stiffness {
 public:
  Dir1D dir[3];
  long long N = 0, Nq = 0;
  int m1p = 0;                    // padded x pitch of the coefficient grids
  DevBuf<double> coeff;           // 6 grids, (a,b) = 00,01,02,11,12,22
  bool grid_nonzero[6] = {true, true, true, true, true, true};
  bool coeffs_ready = false;
  long long flops = 0;            // CostMeter count of one apply (kron.py:90-96)
  int path = 0;                   // 0 = auto (fused), 1 = generic (K1 composition), 2 = fused
  std::shared_ptr<void> fused2_plan;  // element-blocked tables + tiles of the fused kernel
  long long nnz_[3][6] = {};      // interior-restricted nnz per direction: B0,B1,W00,W01,W10,W11

  // slab (multi-GPU) window, global indices: local z-elements [e_lo, e_hi), input planes
  // [v_lo, v_hi), output rows [y_lo, y_hi), local quadrature planes [q_lo, q_hi)
  int e_lo = 0, e_hi = 0, v_lo = 0, v_hi = 0, y_lo = 0, y_hi = 0, q_lo = 0, q_hi = 0;
  bool is_slab() const { return e_lo != 0 || e_hi != dir[2].n_el; }
  void set_slab(int elo, int ehi);
  size_t in_elems() const { return size_t(v_hi - v_lo) * dir[0].n * dir[1].n; }
  size_t out_elems() const { return size_t(y_hi - y_lo) * dir[0].n * dir[1].n; }

  DevBuf<double> pcg_ws;  // PCG work vectors (r, z, p, Ap) + reduction partials, reused across solves
  DevBuf<double> dist_ws;  // slab-distributed PCG workspace of this rank (dist.cu)
  std::shared_ptr<void> pcg_graphs;  // captured PCG iteration bodies (pcg.cu)
  // deterministic accumulation of the fused matvec: per-CTA output boxes summed in a fixed order
  // (bitwise reproducible applies) instead of fp64 atomics
  bool deterministic = false;
  DevBuf<double> det_scratch;

  // on-the-fly coefficients (operators.py:171-183, 207-220): for the analytic maps C depends on
  // xi1 at most, so the kernel reads C(xi1) from a [6][m1] table instead of 6 N_q grids
  bool otf = false;
  DevBuf<double> cx;
  int geo_kind = 0;
  double geo_A[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, geo_K[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  bool geo_hasK = false;
  void set_on_the_fly(int kind, const double* affine9, const double* K9, cudaStream_t s);

  // mass operator on the same 1D factors (operators.py:87-132): w = (W00 x W00 x W00)(m o (B0 x B0 x B0) v),
  // m = alpha det J (operators.py:46-61); `mass_grid` (m3, m2, m1p) stored unless on the fly
  DevBuf<double> mass_grid;
  bool mass_ready = false, mass_otf = false;
  double mass_alpha = 1.0;
  const double* mass_alpha_field = nullptr;  // caller-owned (Nq) alpha values, on-the-fly mode only
  void set_mass(int kind, const double* affine9, const double* J_dev, double alpha, const double* alpha_field_dev,
                int on_the_fly, cudaStream_t s);
  void eval_mass(double* out, const double* J_dev, cudaStream_t s);
  void apply_mass(const double* x, double* y, cudaStream_t s);
  long long mass_flops() const;

  // generic-path scratch
  DevBuf<double> g_, t_, s1_, s2_;
  DevBuf<int> flag_;

  void init(const int* p, const int* nknots, const double* const* knots, const int* npts,
            const double* const* pts, const int* const* indptr, const int* const* indices,
            const double* const* data);
  // Coefficient grids C = det J J^-1 K J^-T (operators.py:64-84).
  void set_geometry(int kind, const double* affine9, const double* K9, const double* J_dev,
                    const double* Kfield_dev, cudaStream_t s);
  void set_coeffs(const double* const* grids_dev, cudaStream_t s);
  void get_coeffs(int key, double* out_dev, cudaStream_t s) const;
  void apply(const double* x, double* y, cudaStream_t s);
  void apply_generic(const double* x, double* y, cudaStream_t s);
  void apply_fused(const double* x, double* y, cudaStream_t s);
  size_t grid_elems() const { return size_t(q_hi - q_lo) * dir[1].m * m1p; }
  int term_mask() const;
  long long flops_for(int mask) const;
 private:
  void compute_flops();
  void detect_nonzero(cudaStream_t s);
};

class FastDiag {
 public:
  int n[3] = {0, 0, 0};
  long long N = 0;
  double sigma = 0;
  std::vector<double> lam_h[3], U_h[3];  // U row-major n x n (U[i][k] = eigvec k, comp i)
  DevBuf<double> U[3], Ut[3], lam[3];
  DevBuf<double> s1_, s2_;
  void init(const int* n, const double* const* K, const double* const* M, double sigma);
  void apply(const double* r, double* z, cudaStream_t s);
  // one direction of the transform on a local (nz, ny, n1) block (multi-GPU building block)
  void apply_dir(int dir, int inverse, int scale, const double* x, double* y, int nz, int ny, int row_lo,
                 cudaStream_t s);
};

struct KrylovOut {
  int iterations = 0, converged = 0, matvecs = 0, precs = 0;
};

// device-resident PCG (solvers.py:137-173)
void pcg_solve(Stiffness& A, FastDiag* P, const double* b, double* x, long long N, double tol, int maxit,
               std::vector<double>& hist, KrylovOut& out, cudaStream_t s);

// element-blocked fused matvec (fused2.cu); false when the rule is outside its structure
bool fused2_apply(Stiffness& S, const double* x, double* y, cudaStream_t s);
bool fused2_accepts(Stiffness& S);  // the rule fits the element-blocked structure (plans it)
bool fused2_apply_mass(Stiffness& S, const double* x, double* y, cudaStream_t s);  // mass as the one-term case

void kron_apply_dense(int d, const int* rows, const int* cols, const double* const* A, const double* x, double* y,
                      int accumulate, cudaStream_t s);

// vector kernels
double dev_dot(const double* a, const double* b, long long N, cudaStream_t s);
// PCG building blocks (pcg.cu): deterministic two-level dot into *out; x += a p, r -= a Ap with
// a = *rz / *pAp and ||r||^2 into *rr; p = z + (*rz_new / *rz) p then *rz = *rz_new.
// Vectors 16-byte aligned; `partial` holds vec_partials() doubles.
void vec_dot_to(const double* a, const double* b, long long N, double* partial, double* out, cudaStream_t s);
void vec_update_xr(double* x, double* r, const double* p, const double* Ap, long long N, const double* rz,
                   const double* pAp, double* partial, double* rr, cudaStream_t s);
void vec_update_p(double* p, const double* z, long long N, const double* rz_new, double* rz, cudaStream_t s);
int vec_partials();

// slab-distributed PCG (dist.cu): transports and the comm variant of pcg_solve
struct Transport;
Transport* transport_local(int world);
Transport* transport_nccl(const char* lib, const unsigned char* id128, int world, int rank);
void transport_destroy(Transport* t);
void transport_info(const Transport* t, int* world, int* nlocal, int* first);
void nccl_unique_id(const char* lib, unsigned char* id128);
void dist_pcg_solve(Transport& T, Stiffness* const* slabs, FastDiag* P, const double* const* b, double* const* x,
                    double tol, int maxit, std::vector<double>& hist, KrylovOut& out, cudaStream_t s);

// BiCGStab fused vector updates (bicgstab.cu; solvers.py:176-249); reductions return to the host
void bicg_p(double* p, const double* r, const double* v, long long N, double beta, double omega, cudaStream_t s);
double bicg_s(double* sv, const double* r, const double* v, long long N, double alpha, cudaStream_t s);
void dot2(const double* a, const double* b, long long N, double* aa_ab, cudaStream_t s);
double dot_fast(const double* a, const double* b, long long N, cudaStream_t s);
double bicg_xr(double* x, double* r, const double* ph, const double* sh, const double* sv, const double* t, long long N,
               double alpha, double omega, cudaStream_t s);
void axpy(double* y, const double* x, long long N, double a, cudaStream_t s);

// Tensor-Gauss quadrature on the device (assembly.py:201-230, problems.py:97-164): load vector
// and L2 / H1 error integrals, sum-factorised over element blocks (csrc/quadrature.cu).
struct Quadrature {
  struct QDir {
    int n_el = 0, nfull = 0;
    std::vector<double> x, w;
    std::vector<int> first;  // first full basis index of each element
    DevBuf<double> x_d, w_d, B_d;
    DevBuf<int> first_d;
  };
  QDir dir[3];
  int deg = 0, g = 0;
  DevBuf<double> part_;
  Quadrature(const int* p, const int* nknots, const double* const* knots, int gauss_per_span);
  long long n_points() const;
  long long n_dofs() const;
  int window_max(int eb) const;
  void pick_block(bool err, int& eb, int& w, size_t& smem) const;
  void rhs(int kind, const double* affine12, const double* J_dev, int case_id, const double* fvals, double* out,
           cudaStream_t s);
  void errors(int kind, const double* affine12, const double* J_dev, int case_id, const double* uvals,
              const double* gvals, const double* u, int with_grad, double* err_ref, cudaStream_t s);
};

}  // namespace mfwq
