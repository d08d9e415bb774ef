// Device-resident preconditioned CG (solvers.py:137-173) with fused
// reduction/update kernels.  All vectors stay in HBM; per iteration the host
// reads back two scalars (p.Ap and ||r||^2) for the indefiniteness and
// stopping tests, exactly where the reference takes those decisions.
#include <cmath>

#include "ops.h"

namespace mfwq {

constexpr int RB = 256;             // threads per reduction block
constexpr int RGRID = 148 * 4;      // blocks (multiple of the SM count)

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[RB / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = threadIdx.x < RB / 32 ? sh[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// partial[b] = sum over the block's grid-stride slice of a.b
__global__ void __launch_bounds__(RB) dot_partial(const double* __restrict__ a, const double* __restrict__ b,
                                                  long long N, double* __restrict__ partial) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RB + threadIdx.x; i < N; i += (long long)gridDim.x * RB) s += a[i] * b[i];
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// deterministic final reduction of RGRID partials into out[slot]
__global__ void __launch_bounds__(RB) finish_sum(const double* __restrict__ partial, int n, double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += RB) s += partial[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
}

// x += alpha p ; r -= alpha Ap ; partial ||r||^2     (alpha = sc[0] / sc[1])
__global__ void __launch_bounds__(RB) update_xr(double* __restrict__ x, double* __restrict__ r,
                                                const double* __restrict__ p, const double* __restrict__ Ap,
                                                long long N, const double* __restrict__ rz,
                                                const double* __restrict__ pAp, double* __restrict__ partial) {
  const double alpha = *rz / *pAp;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RB + threadIdx.x; i < N; i += (long long)gridDim.x * RB) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    s += ri * ri;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// p = z + (rz_new / rz) p ; rz = rz_new
__global__ void __launch_bounds__(RB) update_p(double* __restrict__ p, const double* __restrict__ z, long long N,
                                               const double* __restrict__ rz_new, const double* __restrict__ rz) {
  const double beta = *rz_new / *rz;
  for (long long i = blockIdx.x * (long long)RB + threadIdx.x; i < N; i += (long long)gridDim.x * RB)
    p[i] = z[i] + beta * p[i];
}

__global__ void copy_scalar(const double* src, double* dst) { *dst = *src; }

static void dot_to(const double* a, const double* b, long long N, double* partial, double* out, cudaStream_t s) {
  dot_partial<<<RGRID, RB, 0, s>>>(a, b, N, partial); note_launch();
  finish_sum<<<1, RB, 0, s>>>(partial, RGRID, out); note_launch();
}

double dev_dot(const double* a, const double* b, long long N, cudaStream_t s) {
  DevBuf<double> part(RGRID), out(1);
  dot_to(a, b, N, part.ptr, out.ptr, s);
  double h;
  MFWQ_CUDA(cudaMemcpyAsync(&h, out.ptr, sizeof h, cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
  return h;
}

void pcg_solve(Stiffness& A, FastDiag* P, const double* b, double* x, long long N, double tol, int maxit,
               std::vector<double>& hist, KrylovOut& out, cudaStream_t s) {
  hist.clear();
  out = KrylovOut{};
  MFWQ_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), s));
  // persistent workspace on the operator (no cudaMalloc/cudaFree inside the solve)
  A.pcg_ws.alloc_at_least(4 * N + RGRID + 4);
  double* r = A.pcg_ws.ptr;
  double* z = r + N;
  double* p = z + N;
  double* Ap = p + N;
  struct { double* ptr; } part{Ap + N}, sc{Ap + N + RGRID};  // sc: 0 rz, 1 pAp, 2 rr, 3 rz_new
  double* rz = sc.ptr;
  double* pAp = sc.ptr + 1;
  double* rr = sc.ptr + 2;
  double* rzn = sc.ptr + 3;
  dot_to(b, b, N, part.ptr, rr, s);
  double h2[2];
  MFWQ_CUDA(cudaMemcpyAsync(h2, rr, sizeof(double), cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
  const double bnorm = std::sqrt(h2[0]);
  if (bnorm == 0.0) {  // solvers.py:142-143
    hist.push_back(0.0);
    out.converged = 1;
    return;
  }
  MFWQ_CUDA(cudaMemcpyAsync(r, b, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (P) P->apply(r, z, s);
  else MFWQ_CUDA(cudaMemcpyAsync(z, r, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  out.precs = 1;
  MFWQ_CUDA(cudaMemcpyAsync(p, z, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  dot_to(r, z, N, part.ptr, rz, s);
  hist.push_back(1.0);
  for (int k = 1; k <= maxit; ++k) {
    A.apply(p, Ap, s);
    out.matvecs++;
    dot_to(p, Ap, N, part.ptr, pAp, s);
    update_xr<<<RGRID, RB, 0, s>>>(x, r, p, Ap, N, rz, pAp, part.ptr); note_launch();
    finish_sum<<<1, RB, 0, s>>>(part.ptr, RGRID, rr); note_launch();
    MFWQ_CUDA(cudaGetLastError());
    MFWQ_CUDA(cudaMemcpyAsync(h2, pAp, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    MFWQ_CUDA(cudaStreamSynchronize(s));
    if (h2[0] <= 0) {  // solvers.py:156-160
      char m[128];
      snprintf(m, sizeof m, "nonpositive curvature p.Ap = %.3e at iteration %d", h2[0], k);
      throw IndefiniteErr(m);
    }
    const double rel = std::sqrt(h2[1]) / bnorm;
    hist.push_back(rel);
    if (rel <= tol) {
      out.iterations = k;
      out.converged = 1;
      return;
    }
    if (P) P->apply(r, z, s);
    else MFWQ_CUDA(cudaMemcpyAsync(z, r, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    out.precs++;
    dot_to(r, z, N, part.ptr, rzn, s);
    update_p<<<RGRID, RB, 0, s>>>(p, z, N, rzn, rz); note_launch();
    copy_scalar<<<1, 1, 0, s>>>(rzn, rz); note_launch();
    MFWQ_CUDA(cudaGetLastError());
  }
  out.iterations = maxit;
  out.converged = 0;
}

}  // namespace mfwq
