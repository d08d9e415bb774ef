// Fast-diagonalisation preconditioner (solvers.py:65-127) on B200.
//   setup : generalized 1D eigenproblems K U = M U diag(lam) via cuSOLVER sygvd
//   apply : P^-1 r = (U3 x U2 x U1) diag(1/(l1+l2+l3+sigma)) (U3 x U2 x U1)^T r
//           as six fp64 tensor-core GEMMs (mma.sync m8n8k4 f64 -> SASS DMMA),
//           with the eigenvalue scaling fused into the epilogue of the
//           forward direction-3 GEMM.
#include <cusolverDn.h>

#include <algorithm>
#include <cstdio>

#include "modal_gemm.h"
#include "ops.h"

namespace mfwq {

// ---------------------------------------------------------------------------
// fp64 DMMA GEMM:  C[b] = A[b] (M x K) * B[b] (K x N), row-major, batched.
// Optional epilogue scale 1/(lam1[j%n1] + lam2[j/n1] + lam3[i] + sigma).
// ---------------------------------------------------------------------------
namespace gemm {
constexpr int BM = 64, BN = 64, BK = 16, APAD = 4, BPAD = 8, THREADS = 128;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct Epi {
  const double* lam1;
  const double* lam2;
  const double* lam3;
  int n1;
  double sigma;
};

__global__ void __launch_bounds__(THREADS) dgemm_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                        double* __restrict__ C, int M, int N, int K, int lda, int ldb,
                                                        int ldc, long long sa, long long sb, long long sc, Epi epi) {
  __shared__ __align__(16) double As[2][BM][BK + APAD];
  __shared__ __align__(16) double Bs[2][BK][BN + BPAD];
  const int bz = blockIdx.z;
  A += bz * sa;
  B += bz * sb;
  C += bz * sc;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;

  auto load = [&](int buf, int k0) {
    // A: BM x BK = 1024 doubles, 8 per thread
#pragma unroll
    for (int i = 0; i < (BM * BK) / THREADS; ++i) {
      int idx = tid + i * THREADS;
      int r = idx / BK, c = idx % BK;
      int gr = m0 + r, gc = k0 + c;
      bool ok = gr < M && gc < K;
      cp_async8(&As[buf][r][c], A + (ok ? (long long)gr * lda + gc : 0), ok);
    }
#pragma unroll
    for (int i = 0; i < (BK * BN) / THREADS; ++i) {
      int idx = tid + i * THREADS;
      int r = idx / BN, c = idx % BN;
      int gr = k0 + r, gc = n0 + c;
      bool ok = gr < K && gc < N;
      cp_async8(&Bs[buf][r][c], B + (ok ? (long long)gr * ldb + gc : 0), ok);
    }
    cp_commit();
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (K + BK - 1) / BK;
  load(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      load(buf ^ 1, (kt + 1) * BK);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][wm + i * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + (lane >> 2);
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn + j * 8 + 2 * (lane & 3) + h;
        if (c >= N) continue;
        double v = acc[i][j][h];
        if (epi.lam1) {
          // solvers.py:93-101 accumulation order: ((0 + l1) + l2) + l3, then + sigma
          double ls = epi.lam1[c % epi.n1] + epi.lam2[c / epi.n1];
          ls = ls + epi.lam3[r];
          v = v * (1.0 / (ls + epi.sigma));
        }
        C[(long long)r * ldc + c] = v;
      }
    }
  }
}

void dgemm(const double* A, const double* B, double* C, int M, int N, int K, int lda, int ldb, int ldc, int batch,
           long long sa, long long sb, long long sc, Epi epi, cudaStream_t s) {
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  dgemm_kernel<<<grid, THREADS, 0, s>>>(A, B, C, M, N, K, lda, ldb, ldc, sa, sb, sc, epi); note_launch();
  MFWQ_CUDA(cudaGetLastError());
}
}  // namespace gemm

// ---------------------------------------------------------------------------
// setup
// ---------------------------------------------------------------------------
static void check_solver(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS) {
    char m[128];
    snprintf(m, sizeof m, "%s failed (cusolver status %d)", what, int(st));
    throw EigenErr(m);
  }
}

void FastDiag::init(const int* nn, const double* const* K, const double* const* M, double sig) {
  if (sig < 0) throw ValueErr("sigma must be nonnegative");
  sigma = sig;
  cusolverDnHandle_t h;
  check_solver(cusolverDnCreate(&h), "cusolverDnCreate");
  for (int l = 0; l < 3; ++l) {
    n[l] = nn[l];
    const int nl = n[l];
    // reuse an identical direction (isotropic spaces)
    int same = -1;
    for (int k = 0; k < l; ++k)
      if (n[k] == nl && std::equal(K[k], K[k] + size_t(nl) * nl, K[l]) &&
          std::equal(M[k], M[k] + size_t(nl) * nl, M[l]))
        same = k;
    if (same >= 0) {
      lam_h[l] = lam_h[same];
      U_h[l] = U_h[same];
    } else {
      DevBuf<double> dA(size_t(nl) * nl), dB(size_t(nl) * nl), dW(nl);
      DevBuf<int> info(1);
      dA.upload(K[l], size_t(nl) * nl);
      dB.upload(M[l], size_t(nl) * nl);
      int lwork = 0;
      check_solver(cusolverDnDsygvd_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                               CUBLAS_FILL_MODE_LOWER, nl, dA.ptr, nl, dB.ptr, nl, dW.ptr, &lwork),
                   "sygvd_bufferSize");
      DevBuf<double> work(std::max(lwork, 1));
      check_solver(cusolverDnDsygvd(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, nl,
                                    dA.ptr, nl, dB.ptr, nl, dW.ptr, work.ptr, lwork, info.ptr),
                   "sygvd");
      int hinfo = 0;
      MFWQ_CUDA(cudaMemcpy(&hinfo, info.ptr, sizeof(int), cudaMemcpyDeviceToHost));
      if (hinfo != 0) {
        char m[160];
        snprintf(m, sizeof m, "generalized eigensolve failed (direction %d, info %d)", l, hinfo);
        throw EigenErr(m);
      }
      lam_h[l].resize(nl);
      std::vector<double> Z(size_t(nl) * nl);
      MFWQ_CUDA(cudaMemcpy(lam_h[l].data(), dW.ptr, nl * sizeof(double), cudaMemcpyDeviceToHost));
      MFWQ_CUDA(cudaMemcpy(Z.data(), dA.ptr, Z.size() * sizeof(double), cudaMemcpyDeviceToHost));
      // column-major Z: Z[k*nl + i] = component i of eigenvector k -> U[i][k]
      U_h[l].resize(Z.size());
      for (int i = 0; i < nl; ++i)
        for (int k = 0; k < nl; ++k) U_h[l][size_t(i) * nl + k] = Z[size_t(k) * nl + i];
    }
    // device copies with an even, zero-padded pitch (16-byte cp.async of A tiles)
    const int ld = nl + (nl & 1);
    std::vector<double> Up(size_t(nl) * ld, 0.0), T(size_t(nl) * ld, 0.0);
    for (int i = 0; i < nl; ++i)
      for (int k = 0; k < nl; ++k) {
        Up[size_t(i) * ld + k] = U_h[l][size_t(i) * nl + k];
        T[size_t(k) * ld + i] = U_h[l][size_t(i) * nl + k];
      }
    U[l].upload(Up.data(), Up.size());
    Ut[l].upload(T.data(), T.size());
    lam[l].upload(lam_h[l].data(), nl);
  }
  cusolverDnDestroy(h);
  MFWQ_CUDA(cudaDeviceSynchronize());
  N = (long long)n[0] * n[1] * n[2];
}

// ---------------------------------------------------------------------------
// apply: forward x -> y -> z(+scale), inverse z -> y -> x
// ---------------------------------------------------------------------------
void FastDiag::apply(const double* r, double* z, cudaStream_t s) {
  const int n1 = n[0], n2 = n[1], n3 = n[2];
  if (!s1_.ptr) {
    s1_.alloc(N);
    s2_.alloc(N);
  }
  const long long n12 = (long long)n1 * n2;
  // mode views of the (n3, n2, n1) tensor: k = contracted index, j = the other two
  const ModeView vx{1, (long long)n3 * n2, 0, n1};    // k = i1, j = (i3, i2)
  const ModeView vy{n1, n1, n12, 1};                  // k = i2, j = (i3, i1)
  const ModeView vz{n12, n12, 0, 1};                  // k = i3, j = (i2, i1)
  const Scale none{nullptr, nullptr, nullptr, 1, 0.0};
  const Scale lam_scale{lam[0].ptr, lam[1].ptr, lam[2].ptr, n1, sigma};
  // forward  (U3 x U2 x U1)^T r, eigenvalue scaling fused into the direction-3 epilogue
  auto ld = [](int v) { return v + (v & 1); };
  modal_gemm(Ut[0].ptr, ld(n1), n1, n1, r, vx, s1_.ptr, vx, (long long)n3 * n2, none, true, s);
  modal_gemm(Ut[1].ptr, ld(n2), n2, n2, s1_.ptr, vy, s2_.ptr, vy, (long long)n3 * n1, none, false, s);
  modal_gemm(Ut[2].ptr, ld(n3), n3, n3, s2_.ptr, vz, s1_.ptr, vz, n12, lam_scale, false, s);
  // inverse  (U3 x U2 x U1) y
  modal_gemm(U[2].ptr, ld(n3), n3, n3, s1_.ptr, vz, s2_.ptr, vz, n12, none, false, s);
  modal_gemm(U[1].ptr, ld(n2), n2, n2, s2_.ptr, vy, s1_.ptr, vy, (long long)n3 * n1, none, false, s);
  modal_gemm(U[0].ptr, ld(n1), n1, n1, s1_.ptr, vx, z, vx, (long long)n3 * n2, none, true, s);
}

}  // namespace mfwq

namespace mfwq {
// Direction `dir` of P^-1 on a local (nz, ny, n1) block: forward applies U_dir^T,
// inverse applies U_dir; `scale` (direction 3 forward only) fuses
// 1/(l1[i1] + l2[row_lo + i2] + l3[i3] + sigma).  dir 1 needs ny == n2, dir 2 nz == n3.
void FastDiag::apply_dir(int dir, int inverse, int scale, const double* x, double* y, int nz, int ny, int row_lo,
                         cudaStream_t s) {
  if (dir < 0 || dir > 2) throw ValueErr("direction out of range");
  const int n1 = n[0];
  if ((dir == 1 && ny != n[1]) || (dir == 2 && nz != n[2])) throw ValueErr("block does not span the direction");
  if (scale && (dir != 2 || inverse)) throw ValueErr("the eigenvalue scale belongs to the forward direction-3 step");
  const long long plane = (long long)ny * n1;
  const double* A = inverse ? U[dir].ptr : Ut[dir].ptr;
  const int nl = n[dir], ld = nl + (nl & 1);
  Scale sc{nullptr, nullptr, nullptr, 1, 0.0};
  if (scale) sc = Scale{lam[0].ptr, lam[1].ptr + row_lo, lam[2].ptr, n1, sigma};
  if (dir == 0) {
    const ModeView v{1, (long long)nz * ny, 0, n1};
    modal_gemm(A, ld, nl, nl, x, v, y, v, (long long)nz * ny, sc, true, s);
  } else if (dir == 1) {
    const ModeView v{n1, n1, plane, 1};
    modal_gemm(A, ld, nl, nl, x, v, y, v, (long long)nz * n1, sc, false, s);
  } else {
    const ModeView v{plane, plane, 0, 1};
    modal_gemm(A, ld, nl, nl, x, v, y, v, plane, sc, false, s);
  }
}
}  // namespace mfwq
