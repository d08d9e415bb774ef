// Fused vector kernels of right-preconditioned BiCGStab (solvers.py:176-249).
//
// The iteration itself (breakdown tests, the seeded restart, the stopping test) runs on the
// host exactly as the reference orders it; every vector update is one pass over HBM with its
// reduction fused in:
//   p  = r + beta (p - omega v)                          k_bicg_p
//   s  = r - alpha v,          ||s||^2                   k_bicg_s
//   t.t, t.s                                             k_dot2
//   x += alpha phat + omega shat ; r = s - omega t, ||r||^2   k_bicg_xr
// Reductions are deterministic two-level sums (block partials, then one block).
#include "ops.h"

namespace mfwq {

namespace {
constexpr int BB = 256;        // threads per block
constexpr int BG = 148 * 4;    // blocks: a multiple of the SM count

__device__ __forceinline__ double bsum(double v) {
  __shared__ double sh[BB / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // sh reused by consecutive calls in one kernel
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = threadIdx.x < BB / 32 ? sh[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

#define GRID_STRIDE(i, N) for (long long i = blockIdx.x * (long long)BB + threadIdx.x; i < (N); i += (long long)gridDim.x * BB)

__global__ void __launch_bounds__(BB) k_bicg_p(double* __restrict__ p, const double* __restrict__ r,
                                               const double* __restrict__ v, long long N, double beta, double omega) {
  GRID_STRIDE(i, N) p[i] = r[i] + beta * (p[i] - omega * v[i]);
}

__global__ void __launch_bounds__(BB) k_bicg_s(double* __restrict__ s, const double* __restrict__ r,
                                               const double* __restrict__ v, long long N, double alpha,
                                               double* __restrict__ part) {
  double acc = 0.0;
  GRID_STRIDE(i, N) {
    const double si = r[i] - alpha * v[i];
    s[i] = si;
    acc += si * si;
  }
  acc = bsum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// part[0][b] = sum a.a (if two) / a.b ; part[1][b] = sum a.b
__global__ void __launch_bounds__(BB) k_dot2(const double* __restrict__ a, const double* __restrict__ b, long long N,
                                             double* __restrict__ part) {
  double aa = 0.0, ab = 0.0;
  GRID_STRIDE(i, N) {
    const double ai = a[i];
    aa += ai * ai;
    ab += ai * b[i];
  }
  aa = bsum(aa);
  ab = bsum(ab);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = aa;
    part[BG + blockIdx.x] = ab;
  }
}

__global__ void __launch_bounds__(BB) k_dot(const double* __restrict__ a, const double* __restrict__ b, long long N,
                                            double* __restrict__ part) {
  double ab = 0.0;
  GRID_STRIDE(i, N) ab += a[i] * b[i];
  ab = bsum(ab);
  if (threadIdx.x == 0) part[blockIdx.x] = ab;
}

__global__ void __launch_bounds__(BB) k_bicg_xr(double* __restrict__ x, double* __restrict__ r,
                                                const double* __restrict__ ph, const double* __restrict__ sh,
                                                const double* __restrict__ s, const double* __restrict__ t, long long N,
                                                double alpha, double omega, double* __restrict__ part) {
  double acc = 0.0;
  GRID_STRIDE(i, N) {
    x[i] += alpha * ph[i] + omega * sh[i];
    const double ri = s[i] - omega * t[i];
    r[i] = ri;
    acc += ri * ri;
  }
  acc = bsum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(BB) k_axpy(double* __restrict__ y, const double* __restrict__ x, long long N, double a) {
  GRID_STRIDE(i, N) y[i] += a * x[i];
}

// out[j] = sum_b part[j][b], one block per j
__global__ void __launch_bounds__(BB) k_finish(const double* __restrict__ part, double* __restrict__ out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < BG; i += BB) acc += part[blockIdx.x * BG + i];
  acc = bsum(acc);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

// reduction workspace shared by the calls of one host thread (the library is not reentrant per stream)
DevBuf<double>& red_ws() {
  static thread_local DevBuf<double> ws;
  ws.alloc_at_least(2 * BG + 2);
  return ws;
}

void finish_to_host(double* ws, int k, double* host, cudaStream_t s) {
  k_finish<<<k, BB, 0, s>>>(ws, ws + 2 * BG); note_launch();
  MFWQ_CUDA(cudaGetLastError());
  MFWQ_CUDA(cudaMemcpyAsync(host, ws + 2 * BG, k * sizeof(double), cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

void bicg_p(double* p, const double* r, const double* v, long long N, double beta, double omega, cudaStream_t s) {
  k_bicg_p<<<BG, BB, 0, s>>>(p, r, v, N, beta, omega); note_launch();
  MFWQ_CUDA(cudaGetLastError());
}

double bicg_s(double* sv, const double* r, const double* v, long long N, double alpha, cudaStream_t s) {
  double* ws = red_ws().ptr;
  k_bicg_s<<<BG, BB, 0, s>>>(sv, r, v, N, alpha, ws); note_launch();
  double h;
  finish_to_host(ws, 1, &h, s);
  return h;
}

void dot2(const double* a, const double* b, long long N, double* aa_ab, cudaStream_t s) {
  double* ws = red_ws().ptr;
  k_dot2<<<BG, BB, 0, s>>>(a, b, N, ws); note_launch();
  finish_to_host(ws, 2, aa_ab, s);
}

double dot_fast(const double* a, const double* b, long long N, cudaStream_t s) {
  double* ws = red_ws().ptr;
  k_dot<<<BG, BB, 0, s>>>(a, b, N, ws); note_launch();
  double h;
  finish_to_host(ws, 1, &h, s);
  return h;
}

double bicg_xr(double* x, double* r, const double* ph, const double* sh, const double* sv, const double* t, long long N,
               double alpha, double omega, cudaStream_t s) {
  double* ws = red_ws().ptr;
  k_bicg_xr<<<BG, BB, 0, s>>>(x, r, ph, sh, sv, t, N, alpha, omega, ws); note_launch();
  double h;
  finish_to_host(ws, 1, &h, s);
  return h;
}

void axpy(double* y, const double* x, long long N, double a, cudaStream_t s) {
  k_axpy<<<BG, BB, 0, s>>>(y, x, N, a); note_launch();
  MFWQ_CUDA(cudaGetLastError());
}

}  // namespace mfwq
