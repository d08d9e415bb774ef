// Modal fp64 tensor-core GEMM for the fast-diagonalisation preconditioner.
//
//   C(m, j) = sum_k A[m][k] * X(k, j)      (optionally scaled by 1/(l1+l2+l3+sigma))
//
// A is a small dense n x n factor (row-major); X and C are strided "mode views"
// of an (n3, n2, n1) tensor: element (k, j) lives at k*sk + (j/jdiv)*jhi +
// (j%jdiv)*jlo, so one kernel applies a 1D factor along any of the three
// directions (solvers.py:107-115 contracts each direction with kron.py:86-89).
// The whole mode (n <= 136) is one CTA tile in M, so 130-wide modes waste 4%
// instead of 32% with square 64x64 tiles.  mma.sync m8n8k4 f64 -> SASS DMMA.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "modal_gemm.h"

namespace mfwq {
namespace mg {

constexpr int BK = 16, APAD = 4, BPAD = 4, STAGES = 3;  // BN + 4 = 4 mod 16: conflict-free [k][n] B fragments

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp8(double* dst, const double* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp16(double* dst, const double* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_groups() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ long long colpart(const ModeView& v, long long j) {
  const unsigned q = (unsigned)j / (unsigned)v.jdiv, r = (unsigned)j - q * (unsigned)v.jdiv;  // N < 2^31
  return (long long)q * v.jhi + (long long)r * v.jlo;
}

// MT m8-tiles per warp along M, WM x WN warps, NTW n8-tiles per warp along N.
// BL, the B-tile layout: 0 = [k][n], 8-byte copies walking j (X strided along k);
// 1 = [n][k], 8-byte copies walking k (X contiguous along k); 2 = [n][k], 16-byte copies of
// k-pairs (X contiguous along k and every column 16-byte aligned); 3 = [k][n], 16-byte copies of
// j-pairs (X contiguous along j in runs of even length, even strides).  [n][k] with pitch 20 keeps
// both the copies and the B-fragment reads free of bank conflicts.
template <int MT, int WM, int WN, int NTW, int BL>
__global__ void __launch_bounds__(WM * WN * 32, 2)
    modal_kernel(const double* __restrict__ A, int lda, int M, int K, const double* __restrict__ X, ModeView xv,
                 double* __restrict__ C, ModeView cv, long long N, Scale sc) {
  constexpr int BM = 8 * MT * WM;
  constexpr int THREADS = WM * WN * 32, BN = WN * NTW * 8;
  constexpr bool KN = BL == 0 || BL == 3;  // [k][n] tile
  constexpr int PA = BK + APAD, PB = KN ? BN + BPAD : BK + 4;
  constexpr int BSZ = KN ? BK * PB : BN * PB;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                          // [STAGES][BM][PA]
  double* Bs = sm + STAGES * BM * PA;       // [STAGES][BK][PB] or [STAGES][BN][PB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  // M tiles of one N block are adjacent in launch order, so they share the X tile in L2
  const long long n0 = (long long)blockIdx.y * BN;
  const int m0 = blockIdx.x * BM;

  // the B-tile columns a thread loads are the same for every k-tile: precompute their offsets
  constexpr int KPER = (BL >= 2) ? 2 : 1;
  constexpr int BPER = (BK * BN) / (THREADS * KPER);
  long long bcol[BPER];
  int brow[BPER], bcc[BPER];
  bool bok[BPER];
#pragma unroll
  for (int i = 0; i < BPER; ++i) {
    const int e = tid + i * THREADS;
    if (BL == 2) { bcc[i] = e / (BK / 2); brow[i] = 2 * (e % (BK / 2)); }  // 8 lanes: one column's 16 k
    else if (BL == 1) { bcc[i] = e / BK; brow[i] = e % BK; }              // consecutive lanes walk k
    else if (BL == 3) { brow[i] = e / (BN / 2); bcc[i] = 2 * (e % (BN / 2)); }  // lanes walk j-pairs
    else { brow[i] = e / BN; bcc[i] = e % BN; }                           // consecutive lanes walk j
    bok[i] = n0 + bcc[i] < N;
    bcol[i] = bok[i] ? colpart(xv, n0 + bcc[i]) : 0;
  }
  auto load_a = [&](int stage, int k0) {
    double* as = As + stage * BM * PA;
    for (int e = tid; e < BM * (BK / 2); e += THREADS) {  // 16-byte copies: lda even, A zero-padded
      const int r = e / (BK / 2), c = 2 * (e % (BK / 2)), gm = m0 + r, gk = k0 + c;
      const bool ok = gm < M && gk < lda;
      cp16(as + r * PA + c, ok ? A + (long long)gm * lda + gk : A, ok);
    }
  };
  auto load_b = [&](int stage, int k0) {
    double* bs = Bs + stage * BSZ;
#pragma unroll
    for (int i = 0; i < BPER; ++i) {
      const int gk = k0 + brow[i];
      if (BL == 2) {  // K even, so a pair is either wholly inside or wholly past K
        const bool ok = bok[i] && gk < K;
        cp16(bs + bcc[i] * PB + brow[i], ok ? X + gk + bcol[i] : X, ok);
      } else if (BL == 3) {  // N even, so a pair is either wholly inside or wholly past N
        const bool ok = bok[i] && gk < K;
        cp16(bs + brow[i] * PB + bcc[i], ok ? X + (long long)gk * xv.sk + bcol[i] : X, ok);
      } else {
        const bool ok = bok[i] && gk < K;
        double* d = BL == 1 ? bs + bcc[i] * PB + brow[i] : bs + brow[i] * PB + bcc[i];
        cp8(d, ok ? X + (long long)gk * xv.sk + bcol[i] : X, ok);
      }
    }
  };

  double acc[MT][NTW][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (K + BK - 1) / BK;
  // The factor A never depends on the previous kernel: its first stages are fetched before waiting
  // on the preceding grid (programmatic dependent launch), X only after it has completed.
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s)
    if (s < nk) load_a(s, s * BK);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_b(s, s * BK);
    commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    wait_groups<STAGES - 2>();
    __syncthreads();
    {  // prefetch k-tile kt + STAGES - 1 into the slot freed at kt - 1
      const int kn = kt + STAGES - 1;
      if (kn < nk) {
        load_a(kn % STAGES, kn * BK);
        load_b(kn % STAGES, kn * BK);
      }
      commit();
    }
    const double* as = As + (kt % STAGES) * BM * PA + (wm * MT * 8 + (lane >> 2)) * PA + (lane & 3);
    const double* bs = KN ? Bs + (kt % STAGES) * BSZ + (lane & 3) * PB + wn * NTW * 8 + (lane >> 2)
                               : Bs + (kt % STAGES) * BSZ + (wn * NTW * 8 + (lane >> 2)) * PB + (lane & 3);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if (kt == nk - 1 && kt * BK + kk >= K) break;  // zero-padded k-steps of the last tile (warp-uniform)
      double b[NTW];
#pragma unroll
      for (int j = 0; j < NTW; ++j) b[j] = KN ? bs[kk * PB + j * 8] : bs[j * 8 * PB + kk];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double a = as[i * 8 * PA + kk];
#pragma unroll
        for (int j = 0; j < NTW; ++j) dmma(acc[i][j][0], acc[i][j][1], a, b[j]);
      }
    }
  }
  // the next mode product may start its independent prologue now (it still waits for this grid)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  // epilogue: the output columns (and their eigenvalue sums) depend on (j, h) only
  long long coff[NTW][2];
  double l12[NTW][2];
  bool cok[NTW][2];
#pragma unroll
  for (int j = 0; j < NTW; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long col = n0 + (wn * NTW + j) * 8 + 2 * (lane & 3) + h;
      cok[j][h] = col < N;
      coff[j][h] = cok[j][h] ? colpart(cv, col) : 0;
      l12[j][h] = 0.0;
      if (sc.lam1 && cok[j][h]) {  // solvers.py:93-101: ((l1 + l2) + l3) + sigma; N < 2^31
        const unsigned c = (unsigned)col, q = c / (unsigned)sc.n1;
        l12[j][h] = sc.lam1[c - q * (unsigned)sc.n1] + sc.lam2[q];
      }
    }
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int m = m0 + (wm * MT + i) * 8 + (lane >> 2);
    if (m >= M) continue;
    const double l3 = sc.lam1 ? sc.lam3[m] : 0.0;
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      double v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        v[h] = acc[i][j][h];
        if (sc.lam1) v[h] = v[h] * (1.0 / ((l12[j][h] + l3) + sc.sigma));
      }
      double* o = C + (long long)m * cv.sk + coff[j][0];
      if (BL == 3 && cok[j][1]) {  // the column pair is adjacent and 16-byte aligned
        *reinterpret_cast<double2*>(o) = make_double2(v[0], v[1]);
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (cok[j][h]) C[(long long)m * cv.sk + coff[j][h]] = v[h];
      }
    }
  }
}

static bool pdl_enabled() {  // MFWQ_NO_PDL=1: plain stream-ordered launches (timing experiments)
  static const int on = [] {
    const char* e = getenv("MFWQ_NO_PDL");
    return (e && *e && *e != '0') ? 0 : 1;
  }();
  return on != 0;
}

template <int MT, int WM, int WN, int NTW>
static void launch(const double* A, int lda, int M, int K, const double* X, ModeView xv, double* C, ModeView cv,
                   long long N, Scale sc, bool kc, cudaStream_t s) {
  constexpr int BM = 8 * MT * WM, THREADS = WM * WN * 32, BN = WN * NTW * 8;
  // X contiguous along k with 16-byte aligned columns (even column offsets, even K): k-pair copies
  const bool pairs = kc && xv.sk == 1 && (xv.jhi % 2 == 0) && (xv.jlo % 2 == 0) && (K % 2 == 0) &&
                     ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  // X and C contiguous along j in even runs with even strides (modes 2 and 3 of an even plane): j-pair copies
  auto jpairs = [&](const ModeView& v, const void* p) {
    return v.jlo == 1 && v.jdiv % 2 == 0 && v.sk % 2 == 0 && v.jhi % 2 == 0 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
  };
  const bool jp = !kc && N % 2 == 0 && jpairs(xv, X) && jpairs(cv, C);
  const int bl = kc ? (pairs ? 2 : 1) : (jp ? 3 : 0);
  const size_t smem = sizeof(double) * STAGES * (BM * (BK + APAD) + (bl == 0 || bl == 3 ? BK * (BN + BPAD) : BN * (BK + 4)));
  dim3 grid((M + BM - 1) / BM, (unsigned)((N + BN - 1) / BN));
  auto go = [&](auto kern) {
    MFWQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MFWQ_CUDA(cudaLaunchKernelEx(&cfg, kern, A, lda, M, K, X, xv, C, cv, N, sc));
    note_launch();
  };
  if (bl == 3) go(modal_kernel<MT, WM, WN, NTW, 3>);
  else if (bl == 2) go(modal_kernel<MT, WM, WN, NTW, 2>);
  else if (bl == 1) go(modal_kernel<MT, WM, WN, NTW, 1>);
  else go(modal_kernel<MT, WM, WN, NTW, 0>);
  MFWQ_CUDA(cudaGetLastError());
}

}  // namespace mg

void modal_gemm(const double* A, int lda, int M, int K, const double* X, ModeView xv, double* C, ModeView cv,
                long long N, Scale sc, bool kcontig, cudaStream_t s) {
  if (const char* ev = getenv("MFWQ_MG_CFG")) {  // tuning experiments only
    const int c = atoi(ev);
    if (c == 1) { mg::launch<11, 1, 8, 1>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s); return; }
    if (c == 2) { mg::launch<9, 2, 4, 1>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s); return; }
    if (c == 3) { mg::launch<11, 1, 4, 2>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s); return; }
    if (c == 4) { mg::launch<9, 2, 4, 2>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s); return; }
    if (c == 5) { mg::launch<9, 1, 8, 1>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s); return; }
    if (c == 6) { mg::launch<17, 1, 8, 1>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s); return; }
    if (c == 7) { mg::launch<8, 2, 4, 2>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s); return; }
    if (c == 8) { mg::launch<11, 1, 8, 2>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s); return; }
  }
  // one mode <= 144 wide: a single 128-, 136- or 144-row tile (the narrowest that covers the mode);
  // wider modes: the row tiling (144, 128 or 88 rows) that pads M least, e.g. 258 = 3 x 88 - 6
  if (M <= 128) {
    mg::launch<8, 2, 4, 2>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s);
    return;
  }
  if (M <= 136) {
    mg::launch<17, 1, 8, 1>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s);
    return;
  }
  if (M <= 144) {
    mg::launch<9, 2, 4, 1>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s);
    return;
  }
  auto pad = [&](int bm) { return (M + bm - 1) / bm * bm - M; };
  const int p144 = pad(144), p128 = pad(128), p88 = pad(88);
  if (p88 < p144 && p88 < p128) mg::launch<11, 1, 8, 2>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s);
  else if (p144 <= p128) mg::launch<9, 2, 4, 2>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s);
  else mg::launch<8, 2, 4, 2>(A, lda, M, K, X, xv, C, cv, N, sc, kcontig, s);
}

}  // namespace mfwq
