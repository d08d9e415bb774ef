// Fused MF-WQ stiffness matvec, v2 (the hot path).
//
//   w = sum_{a,b} (Wz x Wy x Wx)^{ab} [ C_ab o (Bz x By x Bx)^b v ]     (operators.py:185-204)
//
// Decomposition: one CTA (256 threads) owns an element-aligned in-plane tile of
// <= 16 x 16 quadrature points (one q-column per thread) and streams a chunk of
// z-elements.  Per z-element e3 (stage s = e3 & 1):
//
//   prefetch : TMA (cp.async.bulk.tensor, mbarrier) brings the coefficient
//              planes of element e3+1 into shared memory; cp.async brings the
//              next DoF plane window of v.                      [HBM stream]
//   B side   : y-contraction of the DoF plane as DMMA tiles (16 x D x D),
//              x-contraction per thread (stationary coefficients), pushed into
//              a register ring of p+1 planes; z-contraction of the ring gives
//              grad v at the quadrature planes of e3 (DFMA, CTA-uniform coeffs).
//   point    : t_ab = C_ab(q) g_b(q), C read once from the TMA stage.
//   W side   : z-contraction first, into register accumulators of the p+2 open
//              DoF planes (DFMA); the completed plane goes through shared memory
//              for the in-plane x- and y-contractions as DMMA tiles; the y-step
//              sums the terms sharing a y-factor inside the MMA K loop; results
//              are added to w with fp64 atomics (tiles/chunks share p+1 rows).
//
// The in-plane band matrices are densified per tile from the operator's own
// element-blocked 1D tables (exact reference coefficients; any element-aligned
// tile shape, uniform or jittered knots).  Band tables:
//   Bt[b][q][k] = B_b(q, j = e(q)+k),    k = 0..p      (full index j)
//   Wt[w][q][k] = W_w(j = e(q)-1+k, q),  k = 0..p+1
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>

#include "ops.h"

#ifndef MFWQ_ABLATE
#define MFWQ_ABLATE 0  // timing experiments only (tools/ablate.sh); 0 in every product build
#endif
#if MFWQ_ABLATE == 9  // per-phase cycle counts of one CTA (timing experiment only)
#define PROF_DECL long long prof_t[10] = {0}; long long prof_last = clock64();
#define PROF(i) { long long now_ = clock64(); prof_t[i] += now_ - prof_last; prof_last = now_; }
#define PROF_DUMP if (blockIdx.x == 40 && blockIdx.y == 1 && threadIdx.x == 0) printf("PROF top %lld fetch %lld bdmma %lld bx %lld mbar %lld z %lld sT %lld wx %lld wy %lld plane %lld\n", prof_t[0], prof_t[1], prof_t[2], prof_t[3], prof_t[4], prof_t[5], prof_t[6], prof_t[7], prof_t[8], prof_t[9]);
#else
#define PROF_DECL
#define PROF(i)
#define PROF_DUMP
#endif

namespace mfwq {
namespace f2 {

constexpr int TQ = 16, NTHR = 256, NWARP = 8;
constexpr int PV = 24;   // pitch (doubles) of N-operand tiles (V, Wx^T, S, A): 24 = 8 mod 16 -> conflict-free B frags
constexpr int PK = 20;   // pitch of K-major A-operand tiles with K <= 16 (T, Wy)
constexpr int PKB = 28;  // pitch of By (K = window rows, up to 24)

struct Tile {
  int ea, eb;  // elements [ea, eb)
  int q0, nq;  // quadrature points [q0, q0+nq)
  int var;     // TMA box variant index along this direction (0 = 16 wide, 1 = narrow)
};

struct Params {
  const double* B[3];  // [2][m][NB]
  const double* W[3];  // [4][m][NW]
  const int* eq[3];    // element of each q
  const int* q0z;      // z: first q of element (n_el+1)
  const Tile* tx;
  const Tile* ty;
  const Tile* tz;
  int ntx, nty;
  int m[3];
  int nel3;
  int bwn;             // narrow box width (even)
  int qe;              // max quadrature planes per z-element
  const double* C;     // 6 grids (padded pitch m1p)
  size_t gstride;
  int m1p;
  const double* x;
  double* y;
  int n1, n2, n3;
};

struct Maps {
  CUtensorMap m[4][6];  // [variant = 2*ynarrow + xnarrow][grid]
};

template <int NT>
struct Terms {
  __host__ __device__ static constexpr int a(int t) { return NT == 3 ? t : (NT == 5 ? (t < 3 ? t : t - 3) : t / 3); }
  __host__ __device__ static constexpr int b(int t) {
    return NT == 3 ? t : (NT == 5 ? (t < 3 ? t : (t == 3 ? 1 : 0)) : t % 3);
  }
};
// symmetric grid index of (a,b): 00,01,02,11,12,22 -> 0..5 (non-recursive so it folds after unrolling)
__host__ __device__ constexpr int gkey(int a, int b) {
  return (a < b ? a : b) == 0 ? (a < b ? b : a) : ((a < b ? a : b) == 1 ? 2 + (a < b ? b : a) : 5);
}
__host__ __device__ constexpr int wtype(int a, int b, int l) { return 2 * (a == l) + (b == l); }
template <int NT>
__host__ __device__ constexpr bool grid_used(int g) {
  bool u = false;
  for (int t = 0; t < NT; ++t) u = u || gkey(Terms<NT>::a(t), Terms<NT>::b(t)) == g;
  return u;
}
template <int NT>
__host__ __device__ constexpr int n_grids() {
  int n = 0;
  for (int g = 0; g < 6; ++g) n += grid_used<NT>(g) ? 1 : 0;
  return n;
}
template <int NT>
__host__ __device__ constexpr int grid_slot(int g) {  // position of grid g among used grids
  int n = 0;
  for (int h = 0; h < g; ++h) n += grid_used<NT>(h) ? 1 : 0;
  return n;
}
template <int NT>
__host__ __device__ constexpr bool ytype_used(int w) {
  bool u = false;
  for (int t = 0; t < NT; ++t) u = u || wtype(Terms<NT>::a(t), Terms<NT>::b(t), 1) == w;
  return u;
}

// ---- PTX helpers -------------------------------------------------------------
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity));
}
__device__ __forceinline__ void tma_load_3d(double* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// ---- the kernel ----------------------------------------------------------------
template <int P, int NT>
struct Occ {  // 2 CTAs/SM where the register budget allows it
  static constexpr int MINB = ((NT == 3 && P <= 6) || (NT == 5 && P <= 2)) ? 2 : 1;
};

template <int P, int NT>
__global__ void __launch_bounds__(NTHR, Occ<P, NT>::MINB)
    k_fused(const __grid_constant__ Params prm, const __grid_constant__ Maps maps) {
  constexpr int NB = P + 1, NW = P + 2;
  constexpr int ZT = 2 * NB + 4 * NW;            // z-table doubles per quadrature plane
  constexpr int G = n_grids<NT>();
  constexpr int DMAX = TQ / 2 + P + 1;           // DoF window bound (8 elements + p + 1)
  constexpr int NTD = (DMAX + 7) / 8;            // 8-wide tiles over a window dimension
  constexpr int KB = ((DMAX + 3) / 4);           // k-steps over window rows (By)
  static_assert(DMAX <= PV, "window exceeds tile pitch");
  using T = Terms<NT>;

  const int QE = prm.qe;  // max quadrature planes per z-element
  extern __shared__ __align__(128) double sm[];
  double* sC = sm;                                  // [2][G][2][16*16] TMA stages (2 q-planes)
  double* sBy = sC + 4 * G * 256;                   // [2][16][PKB]    dense By(q2, r)
  double* sWxT = sBy + 2 * TQ * PKB;                // [4][16][PV]     dense Wx^T(ql, c)
  double* sWy = sWxT + 4 * TQ * PV;                 // [4][PV][PK]     dense Wy(r, q2)
  double* sV = sWy + 4 * PV * PK;                   // [2][PV][PV]     v plane windows
  double* sA = sV + 2 * PV * PV;                    // [2][16][PV]     B-side y result
  double* sT = sA + 2 * TQ * PV;                    // [NT][16][PK]    completed z rows
  double* sS = sT + NT * TQ * PK;                   // [NT][16][PV]    W x results
  double* sBx = sS + NT * TQ * PV;                  // [2][16][NB]
  double* sZ = sBx + 2 * TQ * NB;                   // [2][QE][ZT]     z tables of one element
  int* sEx = reinterpret_cast<int*>(sZ + 2 * QE * ZT);  // [16]
  int* sEy = sEx + TQ;                              // [16]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sEy + TQ);  // [2]
  int* sQ0 = reinterpret_cast<int*>(mbar + 2);      // chunk element -> first q (nez+1)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ql1 = tid & 15, ql2 = tid >> 4;
  const int bxi = blockIdx.x % prm.ntx, byi = blockIdx.x / prm.ntx;
  const Tile tx = prm.tx[bxi], ty = prm.ty[byi], tz = prm.tz[blockIdx.y];
  const int Tx = tx.nq, Ty = ty.nq;
  const int Dx = tx.eb - tx.ea + P + 1, Dy = ty.eb - ty.ea + P + 1;
  const int dax = tx.ea - 2, day = ty.ea - 2;
  const int n1 = prm.n1, n2 = prm.n2, n3 = prm.n3;
  const int m1 = prm.m[0], m2 = prm.m[1], m3 = prm.m[2];
  const int var = 2 * ty.var + tx.var;
  const int bw = tx.var ? prm.bwn : 16, bh = ty.var ? prm.bwn : 16;  // TMA box (x, y)
  const int nez = tz.eb - tz.ea;

  // ---- one-time staging: element offsets, dense band tiles -------------------
  if (tid < TQ) {
    sEx[tid] = tid < Tx ? prm.eq[0][tx.q0 + tid] - tx.ea : 0;
    sEy[tid] = tid < Ty ? prm.eq[1][ty.q0 + tid] - ty.ea : 0;
  }
  for (int i = tid; i <= nez; i += NTHR) sQ0[i] = prm.q0z[tz.ea + i];
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  for (int i = tid; i < 2 * PV * PV; i += NTHR) sV[i] = 0.0;
  __syncthreads();
  const double* __restrict__ Bx = prm.B[0];
  const double* __restrict__ By = prm.B[1];
  const double* __restrict__ Wx = prm.W[0];
  const double* __restrict__ Wy = prm.W[1];
  for (int i = tid; i < 2 * TQ * PKB; i += NTHR) {  // By(q2, r) = Bt[b][q2][r - e(q2) - 1]
    const int b = i / (TQ * PKB), q = (i / PKB) % TQ, r = i % PKB;
    const int k = r - sEy[q] - 1;
    sBy[i] = (q < Ty && k >= 0 && k < NB) ? By[((size_t)b * m2 + ty.q0 + q) * NB + k] : 0.0;
  }
  for (int i = tid; i < 4 * TQ * PV; i += NTHR) {  // Wx^T(ql, c) = Wt[w][ql][c - e(ql)]
    const int w = i / (TQ * PV), q = (i / PV) % TQ, c = i % PV;
    const int k = c - sEx[q];
    sWxT[i] = (q < Tx && k >= 0 && k < NW) ? Wx[((size_t)w * m1 + tx.q0 + q) * NW + k] : 0.0;
  }
  for (int i = tid; i < 4 * PV * PK; i += NTHR) {  // Wy(r, q2) = Wt[w][q2][r - e(q2)]
    const int w = i / (PV * PK), r = (i / PK) % PV, q = i % PK;
    const int k = q < TQ ? r - sEy[q] : -1;
    sWy[i] = (q < Ty && k >= 0 && k < NW) ? Wy[((size_t)w * m2 + ty.q0 + q) * NW + k] : 0.0;
  }
  for (int i = tid; i < 2 * TQ * NB; i += NTHR) {
    const int b = i / (TQ * NB), q = (i / NB) % TQ, k = i % NB;
    sBx[i] = q < Tx ? Bx[((size_t)b * m1 + tx.q0 + q) * NB + k] : 0.0;
  }
  __syncthreads();

  const bool active = ql1 < Tx && ql2 < Ty;
  const int ex = sEx[ql1];
  PROF_DECL
  double hx[NB], hy[NB], h0[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) hx[k] = hy[k] = h0[k] = 0.0;
  double acc[NT][NW];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int k = 0; k < NW; ++k) acc[t][k] = 0.0;

  const double* __restrict__ xv = prm.x;
  double* __restrict__ yv = prm.y;
  const double* __restrict__ ZB = prm.B[2];
  const double* __restrict__ ZW = prm.W[2];

  // v-plane window -> sV[buf] (cp.async, zero fill outside the domain); no commit
  auto fetch_plane = [&](int i3, int buf) {
    if (MFWQ_ABLATE == 5) return;
    const bool vp = i3 >= 0 && i3 < n3;
    double* dst = sV + buf * PV * PV;
    for (int r = warp; r < Dy; r += NWARP) {
      const int g2 = day + r;
      const bool rok = vp && g2 >= 0 && g2 < n2;
      const double* row = xv + ((size_t)(vp ? i3 : 0) * n2 + (rok ? g2 : 0)) * n1;
      for (int c = lane; c < Dx; c += 32) {
        const int g1 = dax + c;
        const bool ok = rok && g1 >= 0 && g1 < n1;
        cp_async8(dst + r * PV + c, ok ? row + g1 : xv, ok);
      }
    }
  };
  // z tables of chunk element el (local) -> sZ[buf]
  auto fetch_ztab = [&](int el, int buf) {
    if (MFWQ_ABLATE == 6) return;
    const int qa = sQ0[el], nq = sQ0[el + 1] - qa;
    double* dst = sZ + buf * QE * ZT;
    for (int i = tid; i < nq * ZT; i += NTHR) {
      const int zl = i / ZT, j = i % ZT;
      const double* src = j < 2 * NB ? ZB + ((size_t)(j / NB) * m3 + qa + zl) * NB + j % NB
                                     : ZW + ((size_t)((j - 2 * NB) / NW) * m3 + qa + zl) * NW + (j - 2 * NB) % NW;
      cp_async8(dst + i, src, true);
    }
  };
  // coefficient planes of chunk element el (2 quadrature planes) -> sC[stage] by TMA
  auto issue_coeff = [&](int el, int stage) {
    if (tid == 0) {
      const int qa = sQ0[el];
      mbar_expect_tx(&mbar[stage], G * 2 * bw * bh * 8);
#pragma unroll
      for (int g = 0; g < 6; ++g) {
        if (!grid_used<NT>(g)) continue;
        const int sl = grid_slot<NT>(g);
        tma_load_3d(sC + ((stage * G + sl) * 2 + 0) * 256, &maps.m[var][g], tx.q0, ty.q0, qa, &mbar[stage]);
        tma_load_3d(sC + ((stage * G + sl) * 2 + 1) * 256, &maps.m[var][g], tx.q0, ty.q0, qa + 1, &mbar[stage]);
      }
    }
  };

  // B side, in-plane: DMMA y-contraction of sV[buf] -> sA, then per-thread x -> ring
  auto bside = [&](int buf) {
    const double* V = sV + buf * PV * PV;
    for (int task = warp; task < (MFWQ_ABLATE == 2 ? 0 : 2 * 2 * NTD); task += NWARP) {  // (b, mt over q2, nt over c)
      const int b = task / (2 * NTD), mt = (task / NTD) % 2, nt = task % NTD;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      const double* ap = sBy + (b * TQ + mt * 8 + (lane >> 2)) * PKB + (lane & 3);
      const double* bp = V + (lane & 3) * PV + nt * 8 + (lane >> 2);
#pragma unroll
      for (int ks = 0; ks < KB; ks += 2) {
        dmma(d0, d1, ap[ks * 4], bp[ks * 4 * PV]);
        if (ks + 1 < KB) dmma(e0, e1, ap[ks * 4 + 4], bp[(ks * 4 + 4) * PV]);
      }
      double* o = sA + (b * TQ + mt * 8 + (lane >> 2)) * PV + nt * 8 + 2 * (lane & 3);
      o[0] = d0 + e0;
      o[1] = d1 + e1;
    }
    __syncthreads();
    PROF(2)
    double vx = 0.0, vy = 0.0, v0 = 0.0;
    const double* a0 = sA + ql2 * PV + ex + 1;
    const double* a1 = sA + (TQ + ql2) * PV + ex + 1;
    const double* b0 = sBx + ql1 * NB;
    const double* b1 = sBx + (TQ + ql1) * NB;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const double c0 = b0[k], c1 = b1[k], x0 = a0[k];
      vx = fma(c1, x0, vx);
      v0 = fma(c0, x0, v0);
      vy = fma(c0, a1[k], vy);
    }
#pragma unroll
    for (int k = 0; k < NB - 1; ++k) {
      hx[k] = hx[k + 1];
      hy[k] = hy[k + 1];
      h0[k] = h0[k + 1];
    }
    hx[NB - 1] = vx;
    hy[NB - 1] = vy;
    h0[NB - 1] = v0;
  };

  // W side: emit accumulator slot 0 as interior DoF plane i3, shift the window
  auto emit = [&](int i3) {
#pragma unroll
    for (int t = 0; t < NT; ++t) sT[(t * TQ + ql2) * PK + ql1] = active ? acc[t][0] : 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
#pragma unroll
      for (int k = 0; k < NW - 1; ++k) acc[t][k] = acc[t][k + 1];
      acc[t][NW - 1] = 0.0;
    }
    if (i3 < 0 || i3 >= n3) return;  // CTA-uniform
    PROF(5)
#if MFWQ_ABLATE == 1
    return;  // timing experiment only: skip the in-plane W contractions
#endif
    __syncthreads();
    PROF(6)
    // x-contraction per term: S_t(q2, c) = sum_ql T_t(q2, ql) Wx_t^T(ql, c)
    for (int task = warp; task < NT * 2 * NTD; task += NWARP) {
      const int t = task / (2 * NTD), mt = (task / NTD) % 2, nt = task % NTD;
      int wx = 0;
#pragma unroll
      for (int u = 0; u < NT; ++u)
        if (u == t) wx = wtype(T::a(u), T::b(u), 0);
      const double* ap = sT + (t * TQ + mt * 8 + (lane >> 2)) * PK + (lane & 3);
      const double* bp = sWxT + (wx * TQ + (lane & 3)) * PV + nt * 8 + (lane >> 2);
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      dmma(d0, d1, ap[0], bp[0]);
      dmma(e0, e1, ap[4], bp[4 * PV]);
      dmma(d0, d1, ap[8], bp[8 * PV]);
      dmma(e0, e1, ap[12], bp[12 * PV]);
      double* o = sS + (t * TQ + mt * 8 + (lane >> 2)) * PV + nt * 8 + 2 * (lane & 3);
      o[0] = d0 + e0;
      o[1] = d1 + e1;
    }
    __syncthreads();
    PROF(7)
    // y-contraction, summed over y-factor groups inside the K loop:
    //   out(r, c) = sum_w sum_q2 Wy_w(r, q2) * sum_{t: ytype(t)=w} S_t(q2, c)
    const size_t plane = (size_t)i3 * n2;
    for (int task = warp; task < NTD * NTD; task += NWARP) {
      const int mt = task / NTD, nt = task % NTD;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      int chain = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        if (!ytype_used<NT>(w)) continue;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int kq = ks * 4 + (lane & 3);
          const double a = sWy[(w * PV + mt * 8 + (lane >> 2)) * PK + kq];
          double bb = 0.0;
#pragma unroll
          for (int t = 0; t < NT; ++t)
            if (wtype(T::a(t), T::b(t), 1) == w) bb += sS[(t * TQ + kq) * PV + nt * 8 + (lane >> 2)];
          if (chain++ & 1) dmma(e0, e1, a, bb);
          else dmma(d0, d1, a, bb);
        }
      }
      d0 += e0;
      d1 += e1;
      const int r = mt * 8 + (lane >> 2), c = nt * 8 + 2 * (lane & 3);
      const int g2 = day + r, g1 = dax + c;
      if (r < Dy && g2 >= 0 && g2 < n2) {
#if MFWQ_ABLATE == 4  // timing experiment only: plain stores instead of atomics
        if (c < Dx && g1 >= 0 && g1 < n1) yv[(plane + g2) * n1 + g1] = d0;
        if (c + 1 < Dx && g1 + 1 >= 0 && g1 + 1 < n1) yv[(plane + g2) * n1 + g1 + 1] = d1;
#else
        if (c < Dx && g1 >= 0 && g1 < n1) atomicAdd(&yv[(plane + g2) * n1 + g1], d0);
        if (c + 1 < Dx && g1 + 1 >= 0 && g1 + 1 < n1) atomicAdd(&yv[(plane + g2) * n1 + g1 + 1], d1);
#endif
      }
    }
    __syncthreads();  // sT / sS free for the next row
    PROF(8)
  };

  // z-part for local plane zl of the element whose tables sit in sZ[zbuf]
  auto zpoint = [&](int qz, int zl, const double* zt, const double* cst, int pl) {
    const double* zb0 = zt + zl * ZT;
    const double* zb1 = zb0 + NB;
    const double* zw = zb0 + 2 * NB;
    double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const double c0 = zb0[k];
      gx = fma(c0, hx[k], gx);
      gy = fma(c0, hy[k], gy);
      gz = fma(zb1[k], h0[k], gz);
    }
    if (!active || MFWQ_ABLATE == 3) return;
    double cg[6];
#pragma unroll
    for (int g = 0; g < 6; ++g) {
      if (!grid_used<NT>(g)) { cg[g] = 0.0; continue; }
      if (cst) cg[g] = cst[(grid_slot<NT>(g) * 2 + pl) * 256 + ql2 * bw + ql1];
      else cg[g] = __ldg(prm.C + g * prm.gstride + ((size_t)qz * m2 + ty.q0 + ql2) * prm.m1p + tx.q0 + ql1);
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int b = T::b(t);
      const double gb = b == 0 ? gx : (b == 1 ? gy : gz);
      const double tv = cg[gkey(T::a(t), b)] * gb;
      const double* wz = zw + wtype(T::a(t), b, 2) * NW;
#pragma unroll
      for (int k = 0; k < NW; ++k) acc[t][k] = fma(wz[k], tv, acc[t][k]);
    }
  };

  // ---- prologue: fill the ring with planes ea-1 .. ea+p-2 ----------------------
  for (int k = 0; k < P; ++k) {
    fetch_plane(tz.ea - 1 + k, 0);
    cp_commit();
    cp_wait_all();
    __syncthreads();
    bside(0);
    __syncthreads();
  }
  fetch_plane(tz.ea + P - 1, 0);
  fetch_ztab(0, 0);
  cp_commit();
  if (sQ0[1] - sQ0[0] == 2) issue_coeff(0, 0);
  unsigned parity[2] = {0u, 0u};

  for (int el = 0; el < nez; ++el) {
    const int e3 = tz.ea + el;
    const int s = el & 1;
    cp_wait_all();
    __syncthreads();  // sV[s], sZ[s] landed; everyone done with step el-1 (stage s^1 reusable)
    PROF(0)
    if (el + 1 < nez) {
      fetch_plane(e3 + P, s ^ 1);
      PROF(9)
      fetch_ztab(el + 1, s ^ 1);
      cp_commit();
      if (sQ0[el + 2] - sQ0[el + 1] == 2) issue_coeff(el + 1, s ^ 1);
    }
    PROF(1)
    bside(s);  // ring: planes e3-1 .. e3+p-1
    PROF(3)
    const int qa = sQ0[el], nq = sQ0[el + 1] - qa;
    const double* zt = sZ + s * QE * ZT;
    if (nq == 2) {
      mbar_wait(&mbar[s], parity[s]);
      parity[s] ^= 1u;
      PROF(4)
      const double* cst = sC + s * G * 512;
      zpoint(qa, 0, zt, cst, 0);
      zpoint(qa + 1, 1, zt, cst, 1);
    } else {
      for (int zl = 0; zl < nq; ++zl) zpoint(qa + zl, zl, zt, nullptr, 0);
    }
    emit(e3 - 2);  // DoF plane j = e3-1 (full) is complete
  }
  for (int k = 0; k < NW - 1; ++k) {
    __syncthreads();
    emit(tz.eb - 2 + k);  // open planes (partial; neighbours add theirs)
  }
  PROF_DUMP
}

}  // namespace f2

// ---------------------------------------------------------------------------
// host: plan (element-blocked tables, tiles, tensor maps), dispatch
// ---------------------------------------------------------------------------
struct Fused2Plan {
  bool ok = false;
  int p = 0, bwn = 0;
  DevBuf<double> B[3], W[3];
  DevBuf<int> eq[3], q0z;
  DevBuf<f2::Tile> tiles[3];
  int ntile[3] = {0, 0, 0};
  int max_nqz = 0, qe = 0, max_chunk = 0;
  const double* maps_for = nullptr;  // coefficient buffer the maps were encoded for
  f2::Maps maps;
};

bool build_elem_tables(const Dir1D& d, std::vector<double>& B, std::vector<double>& W, std::vector<int>& eq);

static std::vector<f2::Tile> f2_tiles_inplane(const Dir1D& d) {
  std::vector<f2::Tile> t;
  const int n = d.n_el;
  auto nq = [&](int a, int b) { return d.elem_q0[b] - d.elem_q0[a]; };
  auto push = [&](int a, int b, int var) { t.push_back({a, b, d.elem_q0[a], nq(a, b), var}); };
  push(0, 1, 1);  // first element alone (boundary extras)
  int e = 1;
  while (e < n - 1) {
    int b = std::min(n - 1, e + 8);
    push(e, b, 0);
    e = b;
  }
  if (n > 1) push(n - 1, n, 1);
  return t;
}

static Fused2Plan* fused2_plan(Stiffness& S) {
  if (S.fused2_plan) return static_cast<Fused2Plan*>(S.fused2_plan.get());
  auto* F = new Fused2Plan();
  S.fused2_plan = std::shared_ptr<void>(F, [](void* q) { delete static_cast<Fused2Plan*>(q); });
  const int p = S.dir[0].p;
  bool ok = p >= 1 && p <= 10 && S.dir[1].p == p && S.dir[2].p == p;
  for (int l = 0; l < 3 && ok; ++l) ok = S.dir[l].n_el >= 2;
  int maxe = 0;
  for (int l = 0; l < 3 && ok; ++l) {
    std::vector<double> B, W;
    std::vector<int> eq;
    ok = build_elem_tables(S.dir[l], B, W, eq);
    if (!ok) break;
    F->B[l].upload(B.data(), B.size());
    F->W[l].upload(W.data(), W.size());
    F->eq[l].upload(eq.data(), eq.size());
    for (int e = 0; e < S.dir[l].n_el; ++e) maxe = std::max(maxe, S.dir[l].elem_q0[e + 1] - S.dir[l].elem_q0[e]);
    std::vector<f2::Tile> t;
    if (l < 2) {
      t = f2_tiles_inplane(S.dir[l]);
      for (auto& tt : t)
        if (tt.nq > f2::TQ || (tt.var == 0 && tt.nq != 2 * (tt.eb - tt.ea))) ok = false;
    } else {
      const long long inplane = (long long)F->ntile[0] * F->ntile[1];
      int chunk = int(std::max<long long>(4, (long long)S.dir[2].n_el * inplane / (148 * 4) + 1));
      chunk = std::min(chunk, 64);
      for (int e = 0; e < S.dir[2].n_el; e += chunk) {
        const int b = std::min(S.dir[2].n_el, e + chunk);
        t.push_back({e, b, S.dir[2].elem_q0[e], S.dir[2].elem_q0[b] - S.dir[2].elem_q0[e], 0});
        F->max_nqz = std::max(F->max_nqz, t.back().nq);
        F->max_chunk = std::max(F->max_chunk, b - e);
      }
      F->q0z.upload(S.dir[2].elem_q0.data(), S.dir[2].elem_q0.size());
    }
    F->ntile[l] = int(t.size());
    F->tiles[l].upload(t.data(), t.size());
  }
  F->bwn = (maxe + 1) / 2 * 2;
  F->qe = maxe;
  F->p = p;
  F->ok = ok && F->bwn <= 16;
  return F;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    MFWQ_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (!ptr || q != cudaDriverEntryPointSuccess) throw CudaErr("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static void encode_maps(Stiffness& S, Fused2Plan& F) {
  if (F.maps_for == S.coeff.ptr) return;
  auto enc = get_encode();
  const size_t G = S.grid_elems();
  for (int v = 0; v < 4; ++v)
    for (int g = 0; g < 6; ++g) {
      cuuint64_t dims[3] = {(cuuint64_t)S.dir[0].m, (cuuint64_t)S.dir[1].m, (cuuint64_t)S.dir[2].m};
      cuuint64_t strides[2] = {(cuuint64_t)S.m1p * 8, (cuuint64_t)S.m1p * S.dir[1].m * 8};
      cuuint32_t box[3] = {(cuuint32_t)((v & 1) ? F.bwn : 16), (cuuint32_t)((v & 2) ? F.bwn : 16), 1};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&F.maps.m[v][g], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)(S.coeff.ptr + g * G), dims,
                       strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw CudaErr("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    }
  F.maps_for = S.coeff.ptr;
}

template <int P, int NT>
static void launch2(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
  using namespace f2;
  encode_maps(S, F);
  Params prm;
  for (int l = 0; l < 3; ++l) {
    prm.B[l] = F.B[l].ptr;
    prm.W[l] = F.W[l].ptr;
    prm.eq[l] = F.eq[l].ptr;
    prm.m[l] = S.dir[l].m;
  }
  prm.q0z = F.q0z.ptr;
  prm.tx = F.tiles[0].ptr;
  prm.ty = F.tiles[1].ptr;
  prm.tz = F.tiles[2].ptr;
  prm.ntx = F.ntile[0];
  prm.nty = F.ntile[1];
  prm.nel3 = S.dir[2].n_el;
  prm.bwn = F.bwn;
  prm.C = S.coeff.ptr;
  prm.gstride = S.grid_elems();
  prm.m1p = S.m1p;
  prm.x = x;
  prm.y = y;
  prm.n1 = S.dir[0].n;
  prm.n2 = S.dir[1].n;
  prm.n3 = S.dir[2].n;
  constexpr int NB = P + 1, NW = P + 2, G = n_grids<NT>();
  prm.qe = F.qe;
  size_t smem = sizeof(double) * (4 * G * 256 + 2 * TQ * PKB + 4 * TQ * PV + 4 * PV * PK + 2 * PV * PV + 2 * TQ * PV +
                                  NT * TQ * PK + NT * TQ * PV + 2 * TQ * NB + (size_t)2 * F.qe * (2 * NB + 4 * NW)) +
                sizeof(int) * 2 * TQ + 16 + sizeof(int) * (F.max_chunk + 2);
  auto kern = k_fused<P, NT>;
  MFWQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  MFWQ_CUDA(cudaMemsetAsync(y, 0, S.N * sizeof(double), s));
  dim3 grid(F.ntile[0] * F.ntile[1], F.ntile[2]);
  kern<<<grid, NTHR, smem, s>>>(prm, F.maps); note_launch();
  MFWQ_CUDA(cudaGetLastError());
}

template <int P>
static void dispatch2(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
  const int mask = S.term_mask();
  if ((mask & ~0x111) == 0) launch2<P, 3>(S, F, x, y, s);
  else if ((mask & ~0x11B) == 0) launch2<P, 5>(S, F, x, y, s);
  else launch2<P, 9>(S, F, x, y, s);
}

bool fused2_apply(Stiffness& S, const double* x, double* y, cudaStream_t s) {
  Fused2Plan* F = fused2_plan(S);
  if (!F->ok) return false;
  switch (F->p) {
    case 1: dispatch2<1>(S, *F, x, y, s); break;
    case 2: dispatch2<2>(S, *F, x, y, s); break;
    case 3: dispatch2<3>(S, *F, x, y, s); break;
    case 4: dispatch2<4>(S, *F, x, y, s); break;
    case 5: dispatch2<5>(S, *F, x, y, s); break;
    case 6: dispatch2<6>(S, *F, x, y, s); break;
    case 7: dispatch2<7>(S, *F, x, y, s); break;
    case 8: dispatch2<8>(S, *F, x, y, s); break;
    case 9: dispatch2<9>(S, *F, x, y, s); break;
    case 10: dispatch2<10>(S, *F, x, y, s); break;
    default: return false;
  }
  return true;
}

}  // namespace mfwq
