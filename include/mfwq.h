/*
 * mfwq.h -- C-ABI of the B200-native MF-WQ hot path (libmfwq.so).
 *
 * Drop-in boundary for the reference's Python operator API (igamf 0.1.0,
 * /root/reference/pkg/src/igamf).  Plain pointers and sizes only; device
 * buffers are fp64 CUDA pointers on the current device, streams are
 * cudaStream_t passed as void*.  Every function returns MFWQ_OK or an error
 * code; mfwq_last_error() gives the message (thread-local).  Error codes map
 * onto the reference's exception types (see MFWQ_E_*).
 *
 * Reference interfaces replaced (file:line in pkg/src/igamf):
 *   mfwq_rule1d_*          build_wq_rule / wq_points / wq_weights      wq.py:62-164
 *                          collocation_matrix                          splines.py:165-192
 *   mfwq_univariate_km     univariate_parametric_matrices              solvers.py:48-62
 *   mfwq_stiffness_create  StiffnessOperator.__init__ / setup_stiffness operators.py:138-163, 227
 *   mfwq_stiffness_set_*   _eval_stiffness_coeffs                      operators.py:64-84
 *   mfwq_stiffness_apply   StiffnessOperator.apply                     operators.py:185-204
 *   mfwq_stiffness_apply_host / _host_join  (same, host buffers, pipelined)  operators.py:185-204
 *   mfwq_stiffness_apply_pageable          (same, pageable host buffers)     operators.py:185-204
 *   mfwq_stiffness_flops   CostMeter count of one apply                kron.py:90-96, operators.py:199-203
 *   mfwq_fd_create         FDPreconditioner.__init__                   solvers.py:72-101
 *   mfwq_fd_apply          FDPreconditioner.apply                      solvers.py:107-115
 *   mfwq_pcg_solve         cg (device-resident loop)                   solvers.py:137-173
 *   mfwq_pcg_solve_comm    cg over xi3 slabs (multi-GPU, NCCL)          solvers.py:137-173, 107-115
 *   mfwq_bicg_*, mfwq_dot2 bicgstab vector updates                     solvers.py:176-249
 *   mfwq_stiffness_set_on_the_fly  on_the_fly=True coefficient mode    operators.py:171-183, 207-220
 *   mfwq_mass_*            MassOperator / setup_mass                   operators.py:46-61, 87-132
 */
#ifndef MFWQ_H_
#define MFWQ_H_

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define MFWQ_OK 0
#define MFWQ_E_VALUE 1        /* ValueError                 */
#define MFWQ_E_WQ 2           /* WQConstructionError        (wq.py:29-39)        */
#define MFWQ_E_DEGENERATE 3   /* DegenerateGeometryError    (operators.py:25-31) */
#define MFWQ_E_EIGEN 4        /* EigenSolveError            (solvers.py:28)      */
#define MFWQ_E_INDEFINITE 5   /* IndefiniteOperatorError    (solvers.py:24)      */
#define MFWQ_E_CUDA 6         /* CUDA runtime failure                            */
#define MFWQ_E_NOTIMPL 7      /* NotImplementedError                             */
#define MFWQ_E_INTERNAL 8

/* geometry kinds for mfwq_stiffness_set_geometry (geometry.py:47-96) */
#define MFWQ_GEOM_IDENTITY 0
#define MFWQ_GEOM_RING 1      /* quarter_ring_map (analytic polar map)           */
#define MFWQ_GEOM_AFFINE 2    /* affine_map: J = A (row-major 3x3)               */
#define MFWQ_GEOM_JACOBIAN 3  /* caller-supplied device Jacobians, (Nq,3,3)      */

const char* mfwq_last_error(void);
int mfwq_version(void);
/* number of kernels this library has launched so far (process-wide) */
long long mfwq_launch_count(void);

/* ---------------- 1D weighted-quadrature rule (host) ---------------- */
typedef struct mfwq_rule1d_s* mfwq_rule1d_t;
/* Register the LAPACK whose dgelsd (ILP64: 64-bit integers, Fortran convention) solves the
   per-row min-norm least-squares systems of the WQ weights, the driver np.linalg.lstsq calls
   (wq.py:86-99).  lib_path: a shared library (dlopen'ed); symbol: its dgelsd (numpy's bundled
   OpenBLAS exports "scipy_dgelsd_64_"); its dsyevd (same name with "syevd") also builds the
   Gauss-Legendre rules the way numpy.polynomial.legendre.leggauss does (wq.py:41-49, the exact
   Gram right-hand sides).  With the host's numpy LAPACK the weights are the reference's bit for
   bit; with none registered a built-in Jacobi SVD solves the rows (same
   truncation rule).  MFWQ_E_VALUE if the library or symbol cannot be loaded. */
int mfwq_set_lapack(const char* lib_path, const char* symbol);
/* 1 when a LAPACK dgelsd is registered, else 0 */
int mfwq_lapack_active(void);
/* knots: open knot vector of degree p on [0,1] (splines.py:16-49) */
int mfwq_rule1d_build(int p, int nknots, const double* knots, mfwq_rule1d_t* out);
/* npts, nfun, boundary extra used, nnz[6] of W00,W01,W10,W11 (nfun x npts), B0,B1 (npts x nfun) */
int mfwq_rule1d_sizes(mfwq_rule1d_t r, int* npts, int* nfun, int* extra, int* nnz6);
/* copy out points and the six CSR matrices (caller-allocated, sizes from _sizes) */
int mfwq_rule1d_export(mfwq_rule1d_t r, double* pts, int* const* indptr6, int* const* indices6,
                       double* const* data6);
void mfwq_rule1d_destroy(mfwq_rule1d_t r);
/* interior (n x n, n = nfun-2) exact 1D stiffness K and mass M, row-major */
int mfwq_univariate_km(int p, int nknots, const double* knots, double* K, double* M);

/* ---------------- MF-WQ stiffness operator (device) ---------------- */
typedef struct mfwq_stiffness_s* mfwq_stiffness_t;
typedef struct {
  int p[3];
  int nknots[3];
  const double* knots[3];
  int npts[3];
  const double* pts[3];
  /* per direction l, the rule's full factors in CSR (host), index l*6 + k with
     k = 0..3: W00,W01,W10,W11 (nfun x npts), k = 4,5: B0,B1 (npts x nfun) */
  const int* indptr[18];
  const int* indices[18];
  const double* data[18];
} mfwq_stiffness_desc;

int mfwq_stiffness_create(const mfwq_stiffness_desc* d, mfwq_stiffness_t* out);
/* kind: MFWQ_GEOM_*; affine9: row-major A for AFFINE; K9: constant diffusion
   (NULL = identity); J_dev: device (Nq,3,3) for JACOBIAN; Kfield_dev: device
   (Nq,3,3) per-point diffusion or NULL.  Both are FULL-domain arrays (all m3 quadrature planes),
   also on slab handles, which read their own planes [q_lo, q_hi) from them.  Raises MFWQ_E_DEGENERATE if det J <= 0. */
int mfwq_stiffness_set_geometry(mfwq_stiffness_t h, int kind, const double* affine9, const double* K9,
                                const double* J_dev, const double* Kfield_dev, void* stream);
/* on-the-fly coefficients (operators.py:138, 171-183, 207-220: on_the_fly=True): no N_q grids are
   stored; the kernel evaluates C at the quadrature points from C(xi1), which is exact for the
   analytic maps (identity / affine with constant K, quarter ring with K = I).  Other geometries
   return MFWQ_E_NOTIMPL.  A later set_geometry / set_coeffs returns to stored grids. */
int mfwq_stiffness_set_on_the_fly(mfwq_stiffness_t h, int kind, const double* affine9, const double* K9,
                                  void* stream);
/* ---- mass operator (operators.py:46-61, 87-132: MassOperator / setup_mass) ------------------
   Built on a stiffness handle (same 1D factors): w = (W00 x W00 x W00)(alpha det J o (B0 x B0 x B0) v).
   alpha: constant, or alpha_field_dev (Nq values of alpha at the mapped points, caller-owned) when
   non-NULL.  on_the_fly: the alpha det J grid is evaluated per apply instead of stored
   (operators.py:121-125; analytic maps only).  MFWQ_E_DEGENERATE if det J <= 0.                */
int mfwq_mass_set(mfwq_stiffness_t h, int kind, const double* affine9, const double* J_dev, double alpha,
                  const double* alpha_field_dev, int on_the_fly, void* stream);
/* y = M x (device pointers, length N); y is overwritten */
int mfwq_mass_apply(mfwq_stiffness_t h, const double* x_dev, double* y_dev, void* stream);
/* CostMeter count of one mass apply: S(B0) + N_q + S(W00)  (kron.py:90-96, operators.py:118-132) */
int mfwq_mass_flops(mfwq_stiffness_t h, long long* flops);
/* six device grids (a<=b order 00,01,02,11,12,22), each (m3,m2,m1) contiguous */
int mfwq_stiffness_set_coeffs(mfwq_stiffness_t h, const double* const* grids6_dev, void* stream);
int mfwq_stiffness_get_coeff(mfwq_stiffness_t h, int key, double* out_dev, void* stream);
/* sizes: n[3], m[3], N, Nq */
int mfwq_stiffness_sizes(mfwq_stiffness_t h, int* n3, int* m3, long long* N, long long* Nq);
/* y = K x  (device pointers, length N); y is overwritten */
int mfwq_stiffness_apply(mfwq_stiffness_t h, const double* x_dev, double* y_dev, void* stream);
/* y_host = K x_host with HOST buffers (pinned for full overlap), asynchronous: H2D on the handle's
   copy stream into one of two device staging buffers, the kernel on `stream`, D2H on the handle's
   second copy stream.  Consecutive calls (on any handles) overlap both copy directions and the
   kernels; y_host is valid after mfwq_stiffness_host_join(h, stream) + a sync of `stream`.
   (operators.py:185-204 with numpy in / numpy out, as a streaming pipeline) */
int mfwq_stiffness_apply_host(mfwq_stiffness_t h, const double* x_host, double* y_host, void* stream);
/* make `stream` wait for every outstanding D2H of h's host pipeline */
int mfwq_stiffness_host_join(mfwq_stiffness_t h, void* stream);
/* y_host = A x_host on pageable host memory (e.g. numpy arrays), synchronous like the reference's
   numpy apply (operators.py:185-204): the vectors are staged in chunks through pinned buffers by a
   pool of host threads, each chunk's host copy overlapping the previous chunk's DMA. */
int mfwq_stiffness_apply_pageable(mfwq_stiffness_t h, const double* x_host, double* y_host, void* stream);
/* Multi-GPU slab: restrict the operator to z-elements [e_lo, e_hi).
   Must precede set_geometry/set_coeffs (only the slab's quadrature planes are stored).
   apply() then maps the input window of interior DoF planes [v_lo, v_hi) to the
   output window [y_lo, y_hi) (partial sums on the p+1 rows shared with neighbours). */
int mfwq_stiffness_set_slab(mfwq_stiffness_t h, int e_lo, int e_hi);
/* info6 = {e_lo, e_hi, v_lo, v_hi, y_lo, y_hi} */
int mfwq_stiffness_slab_info(mfwq_stiffness_t h, int* info6);
/* select kernel path: 0 = auto (fused), 1 = generic K1 composition, 2 = fused */
int mfwq_stiffness_set_path(mfwq_stiffness_t h, int path);
/* deterministic = 1: the fused kernel stores each CTA's output window into its own scratch box and
   a gather sums the boxes covering every DoF in a fixed order, so applies (and solves built on
   them) are bitwise reproducible like the reference's; 0 (default): fp64 atomics, whose last
   bits depend on the arrival order. */
int mfwq_stiffness_set_deterministic(mfwq_stiffness_t h, int on);
/* term_mask: bit 3a+b set when C_ab is not identically zero; fused_ok: the rule fits the fused
   kernel's element-blocked structure; kernel_terms: term class the fused kernel runs (3, 5 or 9) */
int mfwq_stiffness_info(mfwq_stiffness_t h, int* term_mask, int* fused_ok, int* kernel_terms);
int mfwq_stiffness_flops(mfwq_stiffness_t h, long long* flops);
/* same count restricted to the terms with a non-zero coefficient grid (what the kernels execute) */
int mfwq_stiffness_flops_active(mfwq_stiffness_t h, long long* flops);
void mfwq_stiffness_destroy(mfwq_stiffness_t h);

/* ---------------- tensor-Gauss quadrature: load vector, error norms -------------
   mfwq_quad_create   per-direction Gauss rule (gauss_pts_per_span points per knot span; <= 0 means p+1)
                      and collocation tables          wq.py:41-49 gauss_points_weights, assembly.py:78-87
   mfwq_quad_rhs      f_i = int det J b_i (f o F)       assembly.py:201-230 assemble_rhs
   mfwq_quad_errors   err2, ref2 of the relative L2 / H1 error   problems.py:97-164 _error_integrals
   Integrand: case_id MFWQ_CASE_CUBE_SINE / MFWQ_CASE_RING_OSC are evaluated in the kernel at the mapped
   Gauss points (problems.py:77-94); MFWQ_CASE_VALUES reads caller values at every Gauss point (device
   arrays, q1 fastest: fvals [Ng]; error: u values [Ng] and grad u [Ng][3]).  Geometry: kind as for the
   stiffness operator; affine12 = A (row-major 3x3) then b (3) for MFWQ_GEOM_AFFINE; J_dev [Ng][9] for
   MFWQ_GEOM_JACOBIAN (then the integrand must be MFWQ_CASE_VALUES).                                      */
typedef struct mfwq_quad_s* mfwq_quad_t;
#define MFWQ_CASE_VALUES 0
#define MFWQ_CASE_CUBE_SINE 1
#define MFWQ_CASE_RING_OSC 2
int mfwq_quad_create(const int* p3, const int* nknots3, const double* const* knots3, int gauss_pts_per_span,
                     mfwq_quad_t* out);
/* ng3: Gauss points per direction; npts = prod ng3; ndofs = interior DoFs */
int mfwq_quad_sizes(mfwq_quad_t q, int* ng3, long long* npts, long long* ndofs);
/* host copy of the 1D Gauss points and weights of direction dir (ng3[dir] values each) */
int mfwq_quad_points(mfwq_quad_t q, int dir, double* x, double* w);
/* rhs_dev (ndofs) is overwritten */
int mfwq_quad_rhs(mfwq_quad_t q, int kind, const double* affine12, const double* J_dev, int case_id,
                  const double* fvals_dev, double* rhs_dev, void* stream);
/* err_ref (host, 2 doubles) = {err2, ref2}; with_grad = 1: H1 (value + gradient terms), 0: L2.
   Synchronises the stream. */
int mfwq_quad_errors(mfwq_quad_t q, int kind, const double* affine12, const double* J_dev, int case_id,
                     const double* uvals_dev, const double* gvals_dev, const double* u_dev, int with_grad,
                     double* err_ref, void* stream);
void mfwq_quad_destroy(mfwq_quad_t q);

/* ---------------- fast diagonalisation preconditioner ---------------- */
typedef struct mfwq_fd_s* mfwq_fd_t;
/* K3/M3: host row-major (n_l x n_l) interior 1D stiffness / mass per direction */
int mfwq_fd_create(const int* n3, const double* const* K3, const double* const* M3, double sigma, mfwq_fd_t* out);
int mfwq_fd_apply(mfwq_fd_t h, const double* r_dev, double* z_dev, void* stream);
/* one direction of the transform on a local (nz, ny, n1) block, for the multi-GPU
   slab path: forward applies U_dir^T, inverse U_dir; scale (dir 2, forward) fuses
   1/(l1[i1] + l2[row_lo + i2] + l3[i3] + sigma).  dir 1 needs ny == n2, dir 2 nz == n3. */
int mfwq_fd_apply_dir(mfwq_fd_t h, int dir, int inverse, int scale, const double* x_dev, double* y_dev, int nz,
                      int ny, int row_lo, void* stream);
/* host copies of eigenvalues (n) and M-orthonormal eigenvectors U (row-major n x n) */
int mfwq_fd_eigen(mfwq_fd_t h, int dir, double* lam, double* U);
void mfwq_fd_destroy(mfwq_fd_t h);

/* ---------------- preconditioned CG (device-resident) ---------------- */
typedef struct {
  int iterations;
  int converged;
  int matvecs;
  int precond_applies;
  int n_residuals; /* entries written to `residuals` (host, capacity maxit+1) */
} mfwq_krylov_report;

/* P may be NULL (identity).  b_dev, x_dev: device vectors of length N. */
int mfwq_pcg_solve(mfwq_stiffness_t A, mfwq_fd_t P, const double* b_dev, double* x_dev, double tol, int maxit,
                   double* residuals, mfwq_krylov_report* report, void* stream);

/* ---------------- slab-distributed PCG: the `comm` variant ----------------------
   The tensor grid is cut along xi3: rank r owns z-elements [E_r, E_r+1), E_r = r n_el / world,
   and the interior DoF planes [E_r - 1, E_r+1 - 1) (rank 0 from 0, the last rank up to n3); its
   vectors are that contiguous slice of the flat vector.  A communicator drives `nlocal` ranks from
   this process: NCCL (one rank per process / GPU over NVLink) or the in-process transport (every
   rank of the partition from one process on one device, one cudaMemcpyAsync per message; the
   single-GPU emulation of the multi-GPU path with the same solver, kernels and messages). */
typedef struct mfwq_comm_s* mfwq_comm_t;
/* nccl_lib: path of the NCCL shared library to use (torch's bundled libnccl.so.2) */
int mfwq_nccl_unique_id(const char* nccl_lib, unsigned char* id128);
int mfwq_comm_create_nccl(const char* nccl_lib, const unsigned char* id128, int world, int rank, mfwq_comm_t* out);
int mfwq_comm_create_local(int world, mfwq_comm_t* out);
int mfwq_comm_info(mfwq_comm_t c, int* world, int* nlocal, int* first_rank);
void mfwq_comm_destroy(mfwq_comm_t c);
/* cg (solvers.py:137-173) over the slabs, device resident: slabs[l] is local rank (first_rank + l)'s
   slab operator (mfwq_stiffness_set_slab with that rank's elements), P the FD preconditioner of the
   whole space (required), b[l] / x[l] its owned slices (device).  Halo exchanges for the matvec,
   all-to-all for the FD direction 3, allreduced scalars for the dots; one host read per iteration.
   The report and residual history are the global ones (identical on every rank). */
int mfwq_pcg_solve_comm(mfwq_comm_t comm, const mfwq_stiffness_t* slabs, mfwq_fd_t P, const double* const* b,
                        double* const* x, double tol, int maxit, double* residuals, mfwq_krylov_report* report,
                        void* stream);

/* dense Kronecker apply y (+)= (A_d x ... x A_1) x on the device, direction d
   first (kron.py:70-100); A_l host row-major (rows[l] x cols[l]), d <= 3 */
int mfwq_kron_apply(int d, const int* rows, const int* cols, const double* const* A_host, const double* x_dev,
                    double* y_dev, int accumulate, void* stream);

/* device dot product a.b (deterministic two-level reduction), result on the host */
int mfwq_dot(const double* a_dev, const double* b_dev, long long n, double* out, void* stream);

/* ---- BiCGStab vector updates (solvers.py:176-249: bicgstab) ----------------------------------
   The reference's iteration is host logic over numpy vector ops (solvers.py:198-248); these are the
   fused device passes a binding calls in their place.  Reductions are returned to the host.      */
/* aa_ab[0] = a.a, aa_ab[1] = a.b   (solvers.py:239-240: tt = t@t, t@s) */
int mfwq_dot2(const double* a_dev, const double* b_dev, long long n, double* aa_ab, void* stream);
/* y += a x   (solvers.py:233: x += alpha*phat at the early exit) */
int mfwq_axpy(double* y_dev, const double* x_dev, long long n, double a, void* stream);
/* p = r + beta (p - omega v)   (solvers.py:212) */
int mfwq_bicg_p(double* p_dev, const double* r_dev, const double* v_dev, long long n, double beta, double omega,
                void* stream);
/* s = r - alpha v, *ss = ||s||^2   (solvers.py:230-231) */
int mfwq_bicg_s(double* s_dev, const double* r_dev, const double* v_dev, long long n, double alpha, double* ss,
                void* stream);
/* x += alpha phat + omega shat ; r = s - omega t ; *rr = ||r||^2   (solvers.py:242-244) */
int mfwq_bicg_xr(double* x_dev, double* r_dev, const double* phat_dev, const double* shat_dev, const double* s_dev,
                 const double* t_dev, long long n, double alpha, double omega, double* rr, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MFWQ_H_ */
