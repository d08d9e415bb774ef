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
#include <cstdlib>
#include <type_traits>

#include "ops.h"

#ifndef MFWQ_ABLATE
#define MFWQ_ABLATE 0  // timing experiments only (tools/ablate.sh); 0 in every product build
#endif
#ifndef MFWQ_ABL_MASK
#define MFWQ_ABL_MASK 0  // timing experiments only: 1 bside_y, 2 z-part, 4 w_x, 8 w_y, 16 fetch, 32 push_x off
#endif
#if MFWQ_ABLATE == 9  // per-phase cycle counts of one CTA (timing experiment only)
#define PROF_DECL long long prof_t[10] = {0}; long long prof_last = clock64();
#define PROF(i) { long long now_ = clock64(); prof_t[i] += now_ - prof_last; prof_last = now_; }
#define PROF_DUMP if (blockIdx.x == 40 && blockIdx.y == 0 && (threadIdx.x & 31) == 0) printf("PROF w%d B2wait %lld bside %lld fetch %lld wx %lld mbar %lld z %lld B3wait %lld B4wait %lld wy %lld\n", threadIdx.x >> 5, prof_t[0], prof_t[1], prof_t[2], prof_t[3], prof_t[4], prof_t[5], prof_t[6], prof_t[7], prof_t[8]);
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
// B-fragment tiles (read as [k = lane&3][n = lane>>2], pitch PV) are XOR-swizzled: element (r, c) sits
// at r*PV + (c ^ swz(r)).  With PV = 8 mod 16, rows k and k+2 would share banks inside a half-warp;
// flipping column bit 2 on rows with bit 1 set makes the 16 lanes of each half hit 16 distinct
// 8-byte slots, and keeps the double2 pairs of C-fragment stores adjacent.
__host__ __device__ constexpr int swz(int r) { return (r & 2) << 1; }

struct Tile {
  int ea, eb;  // elements [ea, eb)
  int q0, nq;  // quadrature points [q0, q0+nq)
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
  int qe;              // max quadrature planes per z-element
  const double* C;     // 6 grids (padded pitch m1p)
  const double* Cm;    // the mass term's alpha det J grid (same layout), or null
  size_t gstride;
  int m1p;
  const double* x;
  double* y;
  int n1, n2, n3;
  // slab (multi-GPU) windows, global interior plane indices: x holds planes [v_lo, v_hi),
  // y holds rows [y_lo, y_hi); the coefficient grids hold quadrature planes from qzb on
  int v_lo, v_hi, y_lo, y_hi, qzb;
  // host-prepared operand blocks (see fused2_plan): per x-tile [4][16][PV] Wx^T + [2][16][NB] Bx,
  // per y-tile [2][16][PKB] By + [4][PV][PK] Wy; element offsets per tile; z table [m3][ZT]
  const double* xblk;
  const double* yblk;
  const int* exy;   // [ntx][16] then [nty][16]
  const double* ztab;
  int xblk_sz, yblk_sz;
  const double* cx;  // on-the-fly mode: C_g(xi1) table [6][m1]
  // deterministic mode: instead of atomics into y, each CTA stores its output window into its own
  // box [rows][DM][DM] of det (rows from the chunk's first output row ea3 - 2); f2_gather sums the
  // boxes covering each DoF in a fixed order.  null = atomics.
  double* det;
  long long det_box;
  int det_dm;
};


// coefficient grids: the six symmetric C_ab (a <= b) and, for the mass term, alpha det J
constexpr int NGRID = 7, MASS_GRID = 6, MASS_TERM = 0x200;

struct Maps {
  CUtensorMap m[2 * NGRID];  // per coefficient grid: 16 x 16 x 4 boxes, then 16 x 16 x 2 boxes (zero fill past the grid edge)
};

// Term set KS: bit 3a+b set when the term (a,b) runs in this kernel (0x111 diagonal C, 0x11B the
// stored quarter ring's diagonal + C01, 0x1FF general); the t-th term is the t-th set bit.
// bits 0..8: the stiffness terms (a,b); bit 9: the mass term (B0 / W00 in every direction, the
// alpha det J grid; operators.py:87-132), coded as (a, b) = (3, 3)
__host__ __device__ constexpr int popc9(int ks) {
  int n = 0;
  for (int i = 0; i < 10; ++i) n += (ks >> i) & 1;
  return n;
}
__host__ __device__ constexpr int nth_bit(int ks, int t) {
  for (int i = 0; i < 10; ++i)
    if ((ks >> i) & 1) {
      if (t == 0) return i;
      --t;
    }
  return 0;
}
template <int KS>
struct Terms {
  static constexpr int N = popc9(KS);
  // bit index of term t, tabulated once (a(t) / b(t) fold to constants in the unrolled loops)
  static constexpr int I0 = nth_bit(KS, 0), I1 = nth_bit(KS, 1), I2 = nth_bit(KS, 2), I3 = nth_bit(KS, 3),
                       I4 = nth_bit(KS, 4), I5 = nth_bit(KS, 5), I6 = nth_bit(KS, 6), I7 = nth_bit(KS, 7),
                       I8 = nth_bit(KS, 8), I9 = nth_bit(KS, 9);
  __host__ __device__ static constexpr int idx(int t) {
    return t == 0 ? I0 : t == 1 ? I1 : t == 2 ? I2 : t == 3 ? I3 : t == 4 ? I4 : t == 5 ? I5 : t == 6 ? I6 : t == 7 ? I7 : t == 8 ? I8 : I9;
  }
  __host__ __device__ static constexpr int a(int t) { return idx(t) == 9 ? 3 : idx(t) / 3; }
  __host__ __device__ static constexpr int b(int t) { return idx(t) == 9 ? 3 : idx(t) % 3; }
};
// symmetric grid index of (a,b): 00,01,02,11,12,22 -> 0..5, the mass term (3,3) -> 6
// (non-recursive so it folds after unrolling)
__host__ __device__ constexpr int gkey(int a, int b) {
  return a == 3 ? MASS_GRID
                : (a < b ? a : b) == 0 ? (a < b ? b : a) : ((a < b ? a : b) == 1 ? 2 + (a < b ? b : a) : 5);
}
__host__ __device__ constexpr int wtype(int a, int b, int l) { return 2 * (a == l) + (b == l); }
template <int KS>
__host__ __device__ constexpr bool grid_used(int g) {
  bool u = false;
  for (int t = 0; t < Terms<KS>::N; ++t) u = u || gkey(Terms<KS>::a(t), Terms<KS>::b(t)) == g;
  return u;
}
template <int KS>
__host__ __device__ constexpr int n_grids() {
  int n = 0;
  for (int g = 0; g < NGRID; ++g) n += grid_used<KS>(g) ? 1 : 0;
  return n;
}
template <int KS>
__host__ __device__ constexpr int grid_slot(int g) {  // position of grid g among used grids
  int n = 0;
  for (int h = 0; h < g; ++h) n += grid_used<KS>(h) ? 1 : 0;
  return n;
}
template <int KS>
__host__ __device__ constexpr bool ztype_used(int w) {
  bool u = false;
  for (int t = 0; t < Terms<KS>::N; ++t) u = u || wtype(Terms<KS>::a(t), Terms<KS>::b(t), 2) == w;
  return u;
}
template <int KS>
__host__ __device__ constexpr bool ytype_used(int w) {
  bool u = false;
  for (int t = 0; t < Terms<KS>::N; ++t) u = u || wtype(Terms<KS>::a(t), Terms<KS>::b(t), 1) == w;
  return u;
}

// ---- PTX helpers -------------------------------------------------------------
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  // not volatile: independent MMAs of different tiles may be interleaved by the scheduler
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
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
__device__ __forceinline__ void bulk_load(double* dst, const double* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(double* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// ---- the kernel ----------------------------------------------------------------
// CTAs per SM: 2 where the register state (ring 3(p+1) + accumulators NT(p+3) doubles) fits
// 128 registers without spilling, else 1 with up to 255 registers
// z-elements per step: 2, except the 5-term kernel at p = 3, where one element per step halves the
// stage buffers so that two CTAs fit in shared memory (ring p = 3: 2.78 -> 2.53 ms at n_el = 256;
// at p = 4 the same change spills and measured no faster, 2.89 vs 2.94 ms)
__host__ __device__ constexpr int zs_for(int p, int ks) {
  return (ks == 0x11B && p == 3) ? 1 : 2;
}
__host__ __device__ constexpr int occ_for(int p, int ks) {
  return ks == 0x111 ? (p <= 6 ? 2 : 1)
         : ks == 0x11B ? ((p <= 2 || zs_for(p, ks) == 1) ? 2 : 1)
         : ks == 0x200 ? 2  // the mass term: one ring, one accumulator set
                       : 1;
}
// gradient components the term set needs (b of its terms)
template <int KS>
__host__ __device__ constexpr bool bused(int b) {
  bool u = false;
  for (int t = 0; t < Terms<KS>::N; ++t) u = u || Terms<KS>::b(t) == b;
  return u;
}
template <int P, int KS>
struct Occ {
  static constexpr int MINB = occ_for(P, KS);
};
template <int KS>
__host__ __device__ constexpr int n_xtypes() {
  int n = 0;
  for (int w = 0; w < 4; ++w) {
    bool u = false;
    for (int t = 0; t < Terms<KS>::N; ++t) u = u || wtype(Terms<KS>::a(t), Terms<KS>::b(t), 0) == w;
    n += u ? 1 : 0;
  }
  return n;
}
template <int KS>
__host__ __device__ constexpr int xslot(int w) {  // compact index of x-type w among used x-types
  int n = 0;
  for (int v = 0; v < w; ++v) {
    bool u = false;
    for (int t = 0; t < Terms<KS>::N; ++t) u = u || wtype(Terms<KS>::a(t), Terms<KS>::b(t), 0) == v;
    n += u ? 1 : 0;
  }
  return n;
}
template <int KS>
__host__ __device__ constexpr int n_ytypes() {
  int n = 0;
  for (int w = 0; w < 4; ++w) n += ytype_used<KS>(w) ? 1 : 0;
  return n;
}
template <int KS>
__host__ __device__ constexpr int yslot(int w) {
  int n = 0;
  for (int v = 0; v < w; ++v) n += ytype_used<KS>(v) ? 1 : 0;
  return n;
}

// shared-memory plan (doubles), shared by kernel and host launch code
template <int P, int KS, int ZS, bool OTF>
struct Smem {
  static constexpr int NT = Terms<KS>::N;
  static constexpr int NB = P + 1, NW = P + 2;
  static constexpr int NBP = (NB + 1) & ~1, NWP = (NW + 1) & ~1;  // 16-byte aligned sub-tables
  static constexpr int ZT = 2 * NBP + 4 * NWP;                     // z-table doubles per plane
  static constexpr int G = n_grids<KS>(), NX = n_xtypes<KS>(), NY = n_ytypes<KS>();
  static constexpr int CST = OTF ? 0 : ZS * 2 * G * 256;            // the TMA coefficient stage
  static constexpr int DMAX = TQ / 2 + P + 1;                      // DoF window bound
  static constexpr int KB = (DMAX + 3) / 4, VR = 4 * KB;           // By k-steps, v-window rows read
  static constexpr int TSZ = ZS * NT * TQ * PK;                     // sT: emitted rows per term
  static constexpr int ASZ = ZS * 2 * TQ * PV, SSZ = ZS * NY * TQ * PV;
  // every buffer has its own space (no aliasing), so a step needs three CTA barriers
  static constexpr int oC = 0, oT = CST, oBy = oT + TSZ, oWx = oBy + 2 * TQ * PKB, oWy = oWx + NX * TQ * PV,
                       oV = oWy + NY * PV * PK, oA = oV + ZS * VR * PV, oS = oA + ASZ, oBx = oS + SSZ,
                       oCx = oBx + 2 * TQ * NB, oZ = oCx + (OTF ? G * TQ : 0);
  static constexpr int FPT = (DMAX * DMAX + NTHR - 1) / NTHR;       // v-window cells per thread
  static size_t bytes(int qe, int max_chunk) {
    return sizeof(double) * (size_t)(oZ + ZS * qe * ZT) + sizeof(int) * 2 * TQ + 16 + 32 + sizeof(int) * (max_chunk + 2) +
           sizeof(int) * FPT * NTHR + sizeof(int) * (max_chunk / ZS + 2);
  }
};

template <int P, int KS, int ZS, bool OTF>
__device__ __forceinline__ void fused_body(const Params& prm, const Maps& maps) {
  static_assert(!(OTF && (KS & MASS_TERM)), "the mass term runs on its stored alpha det J grid");
  using L = Smem<P, KS, ZS, OTF>;
  constexpr int NT = Terms<KS>::N;
  constexpr int NB = L::NB, NW = L::NW, NBP = L::NBP, NWP = L::NWP, ZT = L::ZT, G = L::G;
  constexpr int R = NB;                          // ring slots (B side): pushed right before use
  constexpr int A = NW;                          // accumulator slots (W side): retired per element
  constexpr int DMAX = L::DMAX;                  // DoF window bound (8 elements + p + 1)
  constexpr int NTD = (DMAX + 7) / 8;            // 8-wide tiles over a window dimension
  constexpr int KB = L::KB, VR = L::VR;          // k-steps over window rows (By), rows of a v window
  static_assert(DMAX <= PV, "window exceeds tile pitch");
  using T = Terms<KS>;

  const int QE = prm.qe;  // max quadrature planes per z-element
  extern __shared__ __align__(128) double sm[];
  double* sC = sm + L::oC;       // [G][ZS*2 planes][256]     TMA coefficient stage
  double* sT = sm + L::oT;       // [ZS][NT][16][PK]          emitted W rows (A operand of W x)
  double* sBy = sm + L::oBy;     // [2][16][PKB]              dense By(q2, r)
  double* sWxT = sm + L::oWx;    // [NX][16][PV]              dense Wx^T(ql, c), used x-types
  double* sWy = sm + L::oWy;     // [NY][PV][PK]              dense Wy(r, q2), used y-types
  double* sV = sm + L::oV;       // [ZS][VR][PV]              v plane windows
  double* sA = sm + L::oA;       // [ZS][2][16][PV]           B-side y result
  double* sS = sm + L::oS;       // [ZS][NY][16][PV]          W x results per y-factor group
  double* sBx = sm + L::oBx;     // [2][16][NB]
  double* sCx = sm + L::oCx;     // [G][16]                   on-the-fly C(xi1) of the tile's x-points
  double* sZ = sm + L::oZ;       // [ZS*QE][ZT]               z tables
  int* sEx = reinterpret_cast<int*>(sZ + ZS * QE * ZT);
  int* sEy = sEx + TQ;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sEy + TQ);
  // tile scalars live in shared memory (re-read after each barrier) instead of pinning
  // registers across the whole z loop
  struct TileInfo { int Dx, Dy, dax, day, nez, ea3, q0x, q0y, pend_nz, pend_i3; };
  TileInfo* sInf = reinterpret_cast<TileInfo*>(mbar + 2);
  int* sQ0 = reinterpret_cast<int*>(sInf + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ql1 = tid & 15, ql2 = tid >> 4;
  const int bxi = blockIdx.x % prm.ntx, byi = blockIdx.x / prm.ntx;
  const Tile tx = prm.tx[bxi], ty = prm.ty[byi], tz = prm.tz[blockIdx.y];
  const int Tx = tx.nq, Ty = ty.nq;
  const int Dx = tx.eb - tx.ea + P + 1, Dy = ty.eb - ty.ea + P + 1;
  const int dax = tx.ea - 2, day = ty.ea - 2;
  const int n1 = prm.n1, n2 = prm.n2;
  const int nez = tz.eb - tz.ea;

  // ---- one-time staging: bulk copies of the host-prepared operand blocks --------
  {
    const double* xb = prm.xblk + (size_t)bxi * prm.xblk_sz;
    const double* yb = prm.yblk + (size_t)byi * prm.yblk_sz;
    auto copy16 = [&](double* dst, const double* src, int n) {  // n doubles, even
      for (int i = 2 * tid; i < n; i += 2 * NTHR) cp_async16(dst + i, src + i);
    };
    copy16(sBy, yb, 2 * TQ * PKB);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if (xslot<KS>(w + 1) > xslot<KS>(w)) copy16(sWxT + xslot<KS>(w) * TQ * PV, xb + w * TQ * PV, TQ * PV);
      if (ytype_used<KS>(w)) copy16(sWy + yslot<KS>(w) * PV * PK, yb + 2 * TQ * PKB + w * PV * PK, PV * PK);
    }
    copy16(sBx, xb + 4 * TQ * PV, 2 * TQ * NB);
    cp_commit();
    if (tid < TQ) {
      sEx[tid] = prm.exy[bxi * TQ + tid];
      sEy[tid] = prm.exy[(prm.ntx + byi) * TQ + tid];
    }
    for (int i = tid; i <= nez; i += NTHR) sQ0[i] = prm.q0z[tz.ea + i];
    if (tid == 0) {
      *sInf = TileInfo{Dx, Dy, dax, day, nez, tz.ea, tx.q0, ty.q0, 0, 0};
      mbar_init(&mbar[0], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    for (int i = tid; i < ZS * VR * PV; i += NTHR) sV[i] = 0.0;
    if constexpr (OTF) {
#pragma unroll
      for (int g = 0; g < 6; ++g)
        if (grid_used<KS>(g) && tid < TQ)
          sCx[grid_slot<KS>(g) * TQ + tid] = tid < tx.nq ? prm.cx[(size_t)g * prm.m[0] + tx.q0 + tid] : 0.0;
    }
    cp_wait_all();
  }
  __syncthreads();

  const bool active = ql1 < Tx && ql2 < Ty;
  const int ex = sEx[ql1];
  PROF_DECL
  double hx[R], hy[R], h0[R];
#pragma unroll
  for (int k = 0; k < R; ++k) hx[k] = hy[k] = h0[k] = 0.0;
  double acc[NT][A];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int k = 0; k < A; ++k) acc[t][k] = 0.0;

  const double* __restrict__ xv = prm.x;
  double* __restrict__ yv = prm.y;

  // v-plane window -> sV[z] (cp.async, zero fill outside the domain); caller commits.
  // Each thread owns fixed window cells: their in-plane offsets are computed once.
  // Window cells outside the domain are never written (sV was zeroed once), so each thread
  // keeps only its in-domain cells.
  constexpr int FPT = L::FPT;
  int* sFP = sQ0 + (nez + 2);  // [FPT][NTHR] packed (global in-plane offset << 10 | window cell), -1 = none
  int* sStep = sFP + FPT * NTHR;  // per step of ZS elements: coefficient planes by TMA (1) or not (0)
  for (int k = 0; k < FPT; ++k) {
    const int e = tid + k * NTHR, r = e / Dx, c = e % Dx, g2 = day + r, g1 = dax + c;
    const bool ok = e < Dy * Dx && g2 >= 0 && g2 < n2 && g1 >= 0 && g1 < n1;
    sFP[k * NTHR + tid] = ok ? ((g2 * n1 + g1) << 10) | (r * PV + (c ^ swz(r))) : -1;
  }
  auto fetch_plane = [&](int i3, int z) {
    if (MFWQ_ABLATE == 5 || (MFWQ_ABL_MASK & 16)) return;
    const bool vp = i3 >= prm.v_lo && i3 < prm.v_hi;
    double* dst = sV + z * VR * PV;
    const double* src = xv + (vp ? (size_t)(i3 - prm.v_lo) * prm.n2 * prm.n1 : 0);
#pragma unroll
    for (int k = 0; k < FPT; ++k) {
      const int code = sFP[k * NTHR + tid];
      if (code >= 0) cp_async8(dst + (code & 1023), src + (code >> 10), vp);  // !vp: zero fill
    }
  };
  // one stage transaction (thread 0): the z tables of chunk elements [el, el+nz) as one bulk
  // copy of the flat [m3][ZT] table, plus (TMA steps) their coefficient planes -> sC
  // Warp 0 issues it in parallel: lane 0 arms the barrier, then one lane per copy (the buffers
  // were only read by the generic proxy since the last fill, and a CTA barrier orders those reads).
  // arm_stage (thread 0, once the previous phase has completed) sets the transaction bytes;
  // issue_stage (after the barrier that frees sC / sZ) spreads the copies over warps 0..G, lane 0
  // each: warp 0 the bulk z rows, warp 1 + slot one 16 x 16 x 4 coefficient box per used grid
  static_assert(ZS == 1 || ZS == 2, "one 16 x 16 x 2ZS box per grid covers a regular step's ZS x 2 planes");
  auto arm_stage = [&](int el, int nz) {
    if (tid != 0) return;
    const bool tma = !OTF && nz == ZS && sStep[el / ZS];
    const unsigned zbytes = (unsigned)((sQ0[el + nz] - sQ0[el]) * ZT * 8);
    mbar_expect_tx(&mbar[0], zbytes + (tma ? ZS * G * 2 * TQ * TQ * 8 : 0));
  };
  auto issue_stage = [&](int el, int nz) {
    if (lane != 0 || warp > G) return;
    const int qa = sQ0[el];
    if (warp == 0) {
      bulk_load(sZ, prm.ztab + (size_t)qa * ZT, (unsigned)((sQ0[el + nz] - qa) * ZT * 8), &mbar[0]);
    } else if (!OTF && nz == ZS && sStep[el / ZS]) {  // regular step: planes qa .. qa+2ZS-1 -> sC [slot][plane][256]
      const int sl = warp - 1;
      int g = 0;
#pragma unroll
      for (int h = 0; h < NGRID; ++h)
        if (grid_used<KS>(h) && grid_slot<KS>(h) == sl) g = h;
      tma_load_3d(sC + sl * (2 * ZS) * 256, &maps.m[(ZS == 2 ? 0 : NGRID) + g], sInf->q0x, sInf->q0y, qa - prm.qzb, &mbar[0]);
    }
  };
  // a step takes its coefficients by TMA when it has ZS elements of exactly 2 planes each
  for (int i = tid; i * ZS < nez; i += NTHR) {
    bool ok = i * ZS + ZS <= nez;
    for (int ez = 0; ez < ZS && ok; ++ez) ok = sQ0[i * ZS + ez + 1] - sQ0[i * ZS + ez] == 2;
    sStep[i] = ok ? 1 : 0;
  }

  // push one DoF plane (already contracted in y into sA[z]) through the x-contraction into the ring
  auto push_x = [&](int z) {
    if (MFWQ_ABL_MASK & 32) return;
    double vx = 0.0, vy = 0.0, v0 = 0.0;
    const double* a0 = sA + (z * 2 * TQ + ql2) * PV + ex + 1;
    const double* a1 = a0 + TQ * PV;
    const double* b0 = sBx + ql1 * NB;
    const double* b1 = b0 + TQ * NB;
#pragma unroll
    for (int k = 0; k < NB; ++k) {  // only the gradient components the term set uses
      if constexpr (bused<KS>(0)) vx = fma(b1[k], a0[k], vx);
      if constexpr (bused<KS>(2) || bused<KS>(3)) v0 = fma(b0[k], a0[k], v0);
      if constexpr (bused<KS>(1)) vy = fma(b0[k], a1[k], vy);
    }
#pragma unroll
    for (int k = 0; k < R - 1; ++k) {
      hx[k] = hx[k + 1];
      hy[k] = hy[k + 1];
      h0[k] = h0[k + 1];
    }
    hx[R - 1] = vx;
    hy[R - 1] = vy;
    h0[R - 1] = v0;
  };
  // B side, in-plane: DMMA y-contraction of nz planes of sV -> sA
  // By types needed: 0 (By) for the x- and z-gradients, 1 (dBy) for the y-gradient
  constexpr bool kA0 = bused<KS>(0) || bused<KS>(2) || bused<KS>(3), kA1 = bused<KS>(1);
  constexpr int NBY = (kA0 ? 1 : 0) + (kA1 ? 1 : 0);
  auto bside_y = [&](int nz) {
    for (int task = warp; task < ((MFWQ_ABLATE == 2 || (MFWQ_ABL_MASK & 1)) ? 0 : NBY * 2 * NTD); task += NWARP) {  // (b, mt, nt)
      const int bs = task / (2 * NTD), mt = (task / NTD) % 2, nt = task % NTD;
      const int b = NBY == 2 ? bs : (kA0 ? 0 : 1);
      const double* ap = sBy + (b * TQ + mt * 8 + (lane >> 2)) * PKB + (lane & 3);
      double a[KB];
#pragma unroll
      for (int ks = 0; ks < KB; ++ks) a[ks] = ap[ks * 4];  // A fragments shared by the planes
#pragma unroll
      for (int z = 0; z < ZS; ++z) {
        if (z >= nz) break;
        const double* bp = sV + z * VR * PV + (lane & 3) * PV + ((nt * 8 + (lane >> 2)) ^ swz(lane & 3));
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KB; ks += 2) {
          dmma(d0, d1, a[ks], bp[ks * 4 * PV]);
          if (ks + 1 < KB) dmma(e0, e1, a[ks + 1], bp[(ks * 4 + 4) * PV]);
        }
        double* o = sA + ((z * 2 + b) * TQ + mt * 8 + (lane >> 2)) * PV + nt * 8 + 2 * (lane & 3);
        o[0] = d0 + e0;
        o[1] = d1 + e1;
      }
    }
  };

  // W side: retire accumulator slot 0 (complete interior DoF plane) into sT row z and shift the
  // accumulators by one; sT is free during the z-part (its reader, W x, ended before a barrier)
  auto store_row = [&](int z) {
    double* st = sT + ql2 * PK + ql1;
#pragma unroll
    for (int t = 0; t < NT; ++t) st[(z * NT + t) * TQ * PK] = active ? acc[t][0] : 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
#pragma unroll
      for (int k = 0; k < A - 1; ++k) acc[t][k] = acc[t][k + 1];
      acc[t][A - 1] = 0.0;
    }
  };
  auto rows_valid = [&](int ne, int i3s) { return !(i3s + ne - 1 < prm.y_lo || i3s >= prm.y_hi); };  // CTA-uniform
  // W x (after the barrier that completes sT): sT -> sS
  auto w_x = [&](auto NEc) {
    constexpr int ne = decltype(NEc)::value;
    // x-contraction per (row, y-factor group): S_g(q2, c) = sum_{t in g} sum_ql T_t(q2, ql) Wx_t^T(ql, c);
    // the terms sharing a y-factor accumulate in one DMMA chain
    {
      constexpr int NY = L::NY, NTASK = ne * NY * 2 * NTD;
      // round r hands warp w task r*8 + ((w + 4r) & 7): groups differ in chain length (a y-group
      // holds 1..3 terms), and the rotation pairs long and short chains per warp
      for (int r = 0; r * NWARP < NTASK; ++r) {
        const int task = r * NWARP + ((warp + 4 * r) & (NWARP - 1));
        if (task >= NTASK) continue;
        const int z = task / (NY * 2 * NTD), ys = (task / (2 * NTD)) % NY, mt = (task / NTD) % 2, nt = task % NTD;
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (yslot<KS>(wtype(T::a(t), T::b(t), 1)) != ys) continue;  // warp-uniform
          const int xs = xslot<KS>(wtype(T::a(t), T::b(t), 0));
          const double* ap = sT + ((z * NT + t) * TQ + mt * 8 + (lane >> 2)) * PK + (lane & 3);
          const double* bp = sWxT + (xs * TQ + (lane & 3)) * PV + ((nt * 8 + (lane >> 2)) ^ swz(lane & 3));
          dmma(d0, d1, ap[0], bp[0]);
          dmma(e0, e1, ap[4], bp[4 * PV]);
          dmma(d0, d1, ap[8], bp[8 * PV]);
          dmma(e0, e1, ap[12], bp[12 * PV]);
        }
        double* o = sS + ((z * NY + ys) * TQ + mt * 8 + (lane >> 2)) * PV + ((nt * 8 + 2 * (lane & 3)) ^ swz(lane >> 2));
        *reinterpret_cast<double2*>(o) = make_double2(d0 + e0, d1 + e1);
      }
    }
  };
  // W y (after the barrier that completes sS): sS -> w with fp64 atomics
  auto w_y = [&](auto NEc, int i3s) {
    constexpr int ne = decltype(NEc)::value;
    for (int task = warp; task < ne * NTD * NTD; task += NWARP) {
      const int z = task / (NTD * NTD), mt = (task / NTD) % NTD, nt = task % NTD;
      const int i3 = i3s + z;
      if (i3 < prm.y_lo || i3 >= prm.y_hi) continue;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      int chain = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        if (!ytype_used<KS>(w)) continue;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int kq = ks * 4 + (lane & 3);
          const double a = sWy[(yslot<KS>(w) * PV + mt * 8 + (lane >> 2)) * PK + kq];
          const double bb = sS[((z * L::NY + yslot<KS>(w)) * TQ + kq) * PV + ((nt * 8 + (lane >> 2)) ^ swz(lane & 3))];
          if (chain++ & 1) dmma(e0, e1, a, bb);
          else dmma(d0, d1, a, bb);
        }
      }
      d0 += e0;
      d1 += e1;
      const int r = mt * 8 + (lane >> 2), c = nt * 8 + 2 * (lane & 3);
      const int n1 = prm.n1, n2 = prm.n2, Dx = sInf->Dx, Dy = sInf->Dy;
      const int g2 = sInf->day + r, g1 = sInf->dax + c;
      const size_t plane = (size_t)(i3 - prm.y_lo) * n2;
      if (MFWQ_ABLATE == 14 && d0 != 1234.5) continue;
      if (prm.det) {  // deterministic: this CTA's box, plain stores (every window cell written once)
        if (r < Dy) {
          const int dm = prm.det_dm;
          double* o = prm.det + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * prm.det_box +
                      ((size_t)(i3 - (sInf->ea3 - 2)) * dm + r) * dm + c;
          if (c < Dx) o[0] = d0;
          if (c + 1 < Dx) o[1] = d1;
        }
        continue;
      }
      if (r < Dy && g2 >= 0 && g2 < n2) {
        if (c < Dx && g1 >= 0 && g1 < n1) atomicAdd(&yv[(plane + g2) * n1 + g1], d0);
        if (c + 1 < Dx && g1 + 1 >= 0 && g1 + 1 < n1) atomicAdd(&yv[(plane + g2) * n1 + g1 + 1], d1);
      }
    }
    PROF(8)
  };

  // z-part for one quadrature plane: ring offset ro, accumulator offset ez.
  // TMAc: coefficients from the TMA stage (cst) or straight from global memory.
  auto zpoint = [&](auto TMAc, int qz, int ro, int ez, const double* zrow, const double* cst) {
    constexpr bool kTMA = decltype(TMAc)::value;
    const double2* zb0 = reinterpret_cast<const double2*>(zrow);
    const double2* zb1 = reinterpret_cast<const double2*>(zrow + NBP);
    const double2* zw = reinterpret_cast<const double2*>(zrow + 2 * NBP);
    double gx = 0.0, gy = 0.0, gz = 0.0, gm = 0.0;
#pragma unroll
    for (int k2 = 0; k2 < NBP / 2; ++k2) {
      const double2 c0 = zb0[k2], c1 = zb1[k2];
      const int k = 2 * k2;
      if constexpr (bused<KS>(0)) gx = fma(c0.x, hx[ro + k], gx);
      if constexpr (bused<KS>(1)) gy = fma(c0.x, hy[ro + k], gy);
      if constexpr (bused<KS>(2)) gz = fma(c1.x, h0[ro + k], gz);
      if constexpr (bused<KS>(3)) gm = fma(c0.x, h0[ro + k], gm);
      if (k + 1 < NB) {
        if constexpr (bused<KS>(0)) gx = fma(c0.y, hx[ro + k + 1], gx);
        if constexpr (bused<KS>(1)) gy = fma(c0.y, hy[ro + k + 1], gy);
        if constexpr (bused<KS>(2)) gz = fma(c1.y, h0[ro + k + 1], gz);
        if constexpr (bused<KS>(3)) gm = fma(c0.y, h0[ro + k + 1], gm);
      }
    }
    if (MFWQ_ABLATE == 3) return;
    // inactive lanes (outside a narrow tile) run the same code with zero coefficients: no
    // divergent exit, so the accumulator registers need no reconciling moves
    double cg[NGRID];
#pragma unroll
    for (int g = 0; g < NGRID; ++g) {
      if (!grid_used<KS>(g)) { cg[g] = 0.0; continue; }
      if constexpr (OTF) cg[g] = active ? sCx[grid_slot<KS>(g) * TQ + ql1] : 0.0;
      else if constexpr (kTMA) cg[g] = active ? cst[grid_slot<KS>(g) * (2 * ZS) * 256] : 0.0;
      else cg[g] = active ? __ldg((g == MASS_GRID ? prm.Cm : prm.C + g * prm.gstride) + ((size_t)(qz - prm.qzb) * prm.m[1] + sInf->q0y + ql2) * prm.m1p + sInf->q0x + ql1) : 0.0;
    }
    double tv[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int b = T::b(t);
      tv[t] = cg[gkey(T::a(t), b)] * (b == 0 ? gx : (b == 1 ? gy : (b == 2 ? gz : gm)));
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      bool used = false;
#pragma unroll
      for (int t = 0; t < NT; ++t) used |= wtype(T::a(t), T::b(t), 2) == w;
      if (!used) continue;
#pragma unroll
      for (int k2 = 0; k2 < NWP / 2; ++k2) {
        const double2 c = zw[w * (NWP / 2) + k2];
        const int k = 2 * k2;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (wtype(T::a(t), T::b(t), 2) != w) continue;
          acc[t][ez + k] = fma(c.x, tv[t], acc[t][ez + k]);
          if (k + 1 < NW) acc[t][ez + k + 1] = fma(c.y, tv[t], acc[t][ez + k + 1]);
        }
      }
    }
  };
  const int cthr = ql2 * TQ + ql1;  // this thread's point inside a TMA coefficient box

  // Regular element (exactly two quadrature planes, coefficients in the TMA stage): the z-part of
  // both planes interleaved, so each thread keeps six independent gradient chains and then
  // eighteen-odd two-deep accumulator chains in flight instead of one plane's dependent sequence.
  // zr: the plane-0 row of the z table (plane 1 follows at zs doubles).
  auto zelem = [&](const double* zr, int zs, const double* cst) {
    double g[2][4];
#pragma unroll
    for (int pl = 0; pl < 2; ++pl) g[pl][0] = g[pl][1] = g[pl][2] = g[pl][3] = 0.0;
#pragma unroll
    for (int k2 = 0; k2 < NBP / 2; ++k2)
#pragma unroll
      for (int pl = 0; pl < 2; ++pl) {
        const double2 c0 = reinterpret_cast<const double2*>(zr + pl * zs)[k2];
        const double2 c1 = reinterpret_cast<const double2*>(zr + pl * zs + NBP)[k2];
        const int k = 2 * k2;
        if constexpr (bused<KS>(0)) g[pl][0] = fma(c0.x, hx[k], g[pl][0]);
        if constexpr (bused<KS>(1)) g[pl][1] = fma(c0.x, hy[k], g[pl][1]);
        if constexpr (bused<KS>(2)) g[pl][2] = fma(c1.x, h0[k], g[pl][2]);
        if constexpr (bused<KS>(3)) g[pl][3] = fma(c0.x, h0[k], g[pl][3]);
        if (k + 1 < NB) {
          if constexpr (bused<KS>(0)) g[pl][0] = fma(c0.y, hx[k + 1], g[pl][0]);
          if constexpr (bused<KS>(1)) g[pl][1] = fma(c0.y, hy[k + 1], g[pl][1]);
          if constexpr (bused<KS>(2)) g[pl][2] = fma(c1.y, h0[k + 1], g[pl][2]);
          if constexpr (bused<KS>(3)) g[pl][3] = fma(c0.y, h0[k + 1], g[pl][3]);
        }
      }
    double tv[2][NT];
#pragma unroll
    for (int pl = 0; pl < 2; ++pl) {
      double cg[NGRID];
#pragma unroll
      for (int gg = 0; gg < NGRID; ++gg) {
        if (!grid_used<KS>(gg)) { cg[gg] = 0.0; continue; }
        if constexpr (OTF) cg[gg] = active ? sCx[grid_slot<KS>(gg) * TQ + ql1] : 0.0;
        else cg[gg] = active ? cst[pl * 256 + grid_slot<KS>(gg) * (2 * ZS) * 256] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int b = T::b(t);
        tv[pl][t] = cg[gkey(T::a(t), b)] * g[pl][b];
      }
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if (!ztype_used<KS>(w)) continue;
      const double* w0 = zr + 2 * NBP + w * NWP;
#pragma unroll
      for (int k2 = 0; k2 < NWP / 2; ++k2) {
        const double2 c0 = reinterpret_cast<const double2*>(w0)[k2];
        const double2 c1 = reinterpret_cast<const double2*>(w0 + zs)[k2];
        const int k = 2 * k2;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (wtype(T::a(t), T::b(t), 2) != w) continue;
          acc[t][k] = fma(c1.x, tv[1][t], fma(c0.x, tv[0][t], acc[t][k]));
          if (k + 1 < NW) acc[t][k + 1] = fma(c1.y, tv[1][t], fma(c0.y, tv[0][t], acc[t][k + 1]));
        }
      }
    }
  };

  // ---- prologue: fill the ring with planes ea-1 .. ea+p-2 ----------------------
  for (int k = 0; k < P; ++k) {
    fetch_plane(tz.ea - 1 + k, 0);
    cp_commit();
    cp_wait_all();
    __syncthreads();
    bside_y(1);
    __syncthreads();
    push_x(0);
  }
  // first step: its DoF planes (y-contracted here) and its stage (z rows, coefficient planes)
  {
    const int nz0 = nez >= ZS ? ZS : 1;
    for (int z = 0; z < nz0; ++z) fetch_plane(tz.ea + P - 1 + z, z);
    cp_commit();
    arm_stage(0, nz0);
    __syncthreads();  // armed before any copy of the phase lands
    issue_stage(0, nz0);
    cp_wait_all();
    __syncthreads();
    bside_y(nz0);
  }
  // everything above reads only x, the operand blocks and the coefficient stage; the output w is
  // zeroed by the preceding grid (programmatic dependent launch): wait for it before any atomic
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  unsigned parity = 0u;  // phase of the stage mbarrier

  // One step over NZ (compile-time) z-elements starting at chunk element el. Phases between the
  // three barriers:  [B2] next v planes, z-part  [B3] next stage, W x  [B4] W y || next B-side y
  // Two CTA barriers per step:  [B2] next v planes, W y of the previous step, z-part
  // [B3] next stage, W x, next B-side y.  (w_y(k-1) | z(k) and w_x(k) | bside_y(k+1) are independent.)
  auto do_step = [&](auto NZc, int el) {
    constexpr int nz = decltype(NZc)::value;
    const int e3 = sInf->ea3 + el, nez = sInf->nez;
    const int eln = el + nz;
    const int nzn = (nez - eln) >= ZS ? ZS : 1;
    __syncthreads();  // B2: sA of this step and sS of the previous one complete, sV / sT free
    PROF(0)
    if (eln < nez)
      for (int z = 0; z < nzn; ++z) fetch_plane(e3 + nz + P - 1 + z, z);  // next step's planes
    cp_commit();
    PROF(2)
    // the previous step's W y-contraction (DMMA + atomics) shares this phase with the z-part:
    // independent work, and the stage copies get longer to land
    if (MFWQ_ABLATE != 12 && !(MFWQ_ABL_MASK & 8)) {
      const int pend_nz = sInf->pend_nz;
      if (pend_nz == 2) w_y(std::integral_constant<int, 2>{}, sInf->pend_i3);
      else if (pend_nz == 1) w_y(std::integral_constant<int, 1>{}, sInf->pend_i3);
    }
    PROF(7)
    mbar_wait(&mbar[0], parity);  // z rows (and TMA coefficient planes) landed
    parity ^= 1u;
    PROF(4)
    if (nz == ZS && sStep[el / ZS]) {
      const double* cst = sC + cthr;
#pragma unroll
      for (int ez = 0; ez < nz; ++ez) {
        push_x(ez);  // ring: planes e3+ez-1 .. e3+ez+p-1, exactly the support of element e3+ez
        if (MFWQ_ABLATE == 13 || (MFWQ_ABL_MASK & 2)) {
        } else if constexpr (P <= 4) {
          zelem(sZ + 2 * ez * ZT, ZT, cst + ez * 2 * 256);
        } else {  // high degree: one plane at a time keeps the live state inside 128 registers
#pragma unroll
          for (int pl = 0; pl < 2; ++pl)
            zpoint(std::true_type{}, 0, 0, 0, sZ + (2 * ez + pl) * ZT, cst + (ez * 2 + pl) * 256);
        }
        store_row(ez);  // row e3+ez-2 complete
      }
    } else {  // boundary z-elements (extra planes) or the odd tail: C straight from global
#pragma unroll
      for (int ez = 0; ez < nz; ++ez) {
        push_x(ez);
        const int qa = sQ0[el + ez], nq = sQ0[el + ez + 1] - qa;
        for (int zl = 0; zl < nq; ++zl)
          zpoint(std::false_type{}, qa + zl, 0, 0, sZ + (qa - sQ0[el] + zl) * ZT, nullptr);
        store_row(ez);
      }
    }
    PROF(5)
    if (eln < nez) arm_stage(eln, nzn);  // next phase (this one completed above); copies follow B3
    cp_wait_all();
    __syncthreads();  // B3: sT complete, all reads of sC / sZ done, next v planes landed
    PROF(6)
    if (eln < nez) issue_stage(eln, nzn);
    const bool rv = rows_valid(nz, e3 - 2);
    if (rv && MFWQ_ABLATE != 11 && !(MFWQ_ABL_MASK & 4)) w_x(std::integral_constant<int, nz>{});
    PROF(3)
    if (tid == 0) {  // its W y runs in the next z phase (or after the loop); read after the next barrier
      sInf->pend_nz = rv ? nz : 0;
      sInf->pend_i3 = e3 - 2;
    }
    if (eln < nez) {
      if (nzn == ZS) bside_y(ZS);
      else bside_y(1);
    }
    PROF(1)
  };

  int el = 0;
  for (; el + ZS <= sInf->nez; el += ZS) do_step(std::integral_constant<int, ZS>{}, el);
  if (el < sInf->nez) do_step(std::integral_constant<int, 1>{}, el);  // odd tail
  __syncthreads();  // sS of the last step complete, its W x done with sT
  if (sInf->pend_nz == 2) w_y(std::integral_constant<int, 2>{}, sInf->pend_i3);
  else if (sInf->pend_nz == 1) w_y(std::integral_constant<int, 1>{}, sInf->pend_i3);
  // flush the open planes (partial; neighbours add theirs): slot k holds interior row eb-2+k
  for (int k = 0; k < NW - 1; ++k) {
    const int i3 = sInf->ea3 + sInf->nez - 2 + k;
    store_row(0);
    __syncthreads();
    const bool rv = rows_valid(1, i3);
    if (rv) w_x(std::integral_constant<int, 1>{});
    __syncthreads();
    if (rv) w_y(std::integral_constant<int, 1>{}, i3);
  }
  PROF_DUMP
}

// one term set per launch (blockIdx.x: in-plane tile, blockIdx.y: z-chunk)
template <int P, int KS, int ZS, bool OTF>
__global__ void __launch_bounds__(NTHR, Occ<P, KS>::MINB)
    k_fused(const __grid_constant__ Params prm, const __grid_constant__ Maps maps) {
  fused_body<P, KS, ZS, OTF>(prm, maps);
}

// Deterministic mode: y(i3, i2, i1) = the sum, in a fixed (z-chunk, y-tile, x-tile) order, of the
// window cells of every CTA box covering the DoF; candidate tables per direction: (tile, local
// index) pairs, -1 padded, KX / KY / KZ per DoF
struct GatherTabs {
  const int2* cx;
  const int2* cy;
  const int2* cz;
  int kx, ky, kz;
};
static __global__ void __launch_bounds__(256) f2_gather(double* __restrict__ y, const double* __restrict__ det,
                                                 const __grid_constant__ GatherTabs T, int n1, int n2, int y_lo,
                                                 int y_hi, int ntx, int nty, long long box, int dm) {
  const long long n = (long long)(y_hi - y_lo) * n2 * n1;
  for (long long o = blockIdx.x * 256LL + threadIdx.x; o < n; o += (long long)gridDim.x * 256) {
    const int i1 = int(o % n1);
    const long long r = o / n1;
    const int i2 = int(r % n2), i3 = int(r / n2) + y_lo;
    double sum = 0.0;
    for (int a = 0; a < T.kz; ++a) {
      const int2 z = T.cz[(size_t)i3 * T.kz + a];
      if (z.x < 0) break;
      for (int b = 0; b < T.ky; ++b) {
        const int2 yy = T.cy[(size_t)i2 * T.ky + b];
        if (yy.x < 0) break;
        const double* rowp = det + ((size_t)z.x * nty + yy.x) * ntx * box + ((size_t)z.y * dm + yy.y) * dm;
        for (int c = 0; c < T.kx; ++c) {
          const int2 xx = T.cx[(size_t)i1 * T.kx + c];
          if (xx.x < 0) break;
          sum += rowp[(size_t)xx.x * box + xx.y];
        }
      }
    }
    y[o] = sum;
  }
}

}  // namespace f2

// ---------------------------------------------------------------------------
// host: plan (element-blocked tables, tiles, tensor maps), dispatch
// ---------------------------------------------------------------------------
// The warp-specialised kernel (fused3.cu, one CTA per SM) runs the cases it measured faster in
// (tools/f3_sweep.sh, profiles/f3_sweep_r02.txt): the three-term kernel from p = 2 (stored and on the
// fly), the five-term kernel at p = 1, 2, 4, 6.  MFWQ_F3=0 keeps the phased kernel everywhere, MFWQ_F3=2
// takes the warp-specialised one wherever it exists (p <= 6).
inline bool f3_wanted(int p, int ks) {
  static const int on = [] { const char* e = getenv("MFWQ_F3"); return e ? atoi(e) : 1; }();
  if (!on || p < 1 || p > 6 || (ks != 0x111 && ks != 0x11B)) return false;
  if (on == 2) return true;
  return ks == 0x111 ? p >= 2 : (p == 1 || p == 2 || p == 4 || p == 6);
}

struct Fused2Plan {
  bool ok = false;
  int p = 0;
  DevBuf<double> B[3], W[3];
  DevBuf<int> eq[3], q0z, exy;
  DevBuf<double> xblk, yblk, ztab;  // host-prepared per-tile operand blocks, flat z table
  int xblk_sz = 0, yblk_sz = 0;
  DevBuf<f2::Tile> tiles[3];
  int ntile[3] = {0, 0, 0};
  int max_nqz = 0, qe = 0, max_chunk = 0;
  const double* maps_for = nullptr;  // coefficient buffer the maps were encoded for
  const double* maps_for_mass = nullptr;  // mass grid the mass maps were encoded for
  f2::Maps maps;  // 16 x 16 x 4 / x 2 boxes: the ZS x 2 planes of a regular step
  // deterministic mode: candidate tables of the gather, box geometry
  std::vector<f2::Tile> htiles[3];
  DevBuf<int2> cand[3];
  int kc[3] = {0, 0, 0};
  long long det_box = 0;
  int det_dm = 0;
  bool det_ready = false;
};

#ifndef MFWQ_F2_OTF_UNIT  // plan + tensor maps: defined once (fused2.cu), not in fused2_otf.cu
// Element-blocked 1D tables from the operator's banded factors (every non-zero of the reference's
// CSR factors must fall inside the element block; false = the rule is outside this structure)
bool build_elem_tables(const Dir1D& d, std::vector<double>& B, std::vector<double>& W, std::vector<int>& eq) {
  const int p = d.p, NB = p + 1, NW = p + 2, m = d.m;
  eq.assign(m, 0);
  for (int e = 0; e < d.n_el; ++e)
    for (int q = d.elem_q0[e]; q < d.elem_q0[e + 1]; ++q) eq[q] = e;
  B.assign(size_t(2) * m * NB, 0.0);
  W.assign(size_t(4) * m * NW, 0.0);
  // B band: interior column c <-> full j = c+1 ; k = j - e(q)
  for (int b = 0; b < 2; ++b) {
    const BandHost& h = d.B[b].h;
    for (int q = 0; q < m; ++q)
      for (int u = 0; u < h.width; ++u) {
        double v = h.vals[size_t(q) * h.width + u];
        if (v == 0.0) continue;
        int j = h.start[q] + u + 1, k = j - eq[q];
        if (k < 0 || k >= NB) return false;
        B[(size_t(b) * m + q) * NB + k] = v;
      }
  }
  // W band: interior row i <-> full j = i+1 ; k = j - e(q) + 1
  for (int w = 0; w < 4; ++w) {
    const BandHost& h = d.W[w].h;
    for (int i = 0; i < h.rows; ++i)
      for (int u = 0; u < h.width; ++u) {
        double v = h.vals[size_t(i) * h.width + u];
        if (v == 0.0) continue;
        int q = h.start[i] + u, j = i + 1, k = j - eq[q] + 1;
        if (k < 0 || k >= NW) return false;
        W[(size_t(w) * m + q) * NW + k] = v;
      }
  }
  return true;
}

static std::vector<f2::Tile> f2_tiles_inplane(const Dir1D& d) {
  // greedy element-aligned tiles of <= 16 quadrature points from element 0: with an even
  // number of boundary extras every tile but the last is exactly 16 points wide, so the
  // boundary elements ride along with their neighbours instead of forming thin strips
  std::vector<f2::Tile> t;
  const int n = d.n_el;
  auto nq = [&](int a, int b) { return d.elem_q0[b] - d.elem_q0[a]; };
  int e = 0;
  while (e < n) {
    int b = e + 1;
    while (b < n && nq(e, b + 1) <= f2::TQ) ++b;
    t.push_back({e, b, d.elem_q0[e], nq(e, b)});
    e = b;
  }
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
  std::vector<double> HB[3], HW[3];
  std::vector<int> Heq[3];
  std::vector<f2::Tile> T[3];
  for (int l = 0; l < 3 && ok; ++l) {
    std::vector<double>& B = HB[l];
    std::vector<double>& W = HW[l];
    std::vector<int>& eq = Heq[l];
    ok = build_elem_tables(S.dir[l], B, W, eq);
    if (!ok) break;
    F->B[l].upload(B.data(), B.size());
    F->W[l].upload(W.data(), W.size());
    F->eq[l].upload(eq.data(), eq.size());
    for (int e = 0; e < S.dir[l].n_el; ++e) maxe = std::max(maxe, S.dir[l].elem_q0[e + 1] - S.dir[l].elem_q0[e]);
    std::vector<f2::Tile>& t = T[l];
    if (l < 2) {
      t = f2_tiles_inplane(S.dir[l]);
      for (auto& tt : t)
        if (tt.nq > f2::TQ) ok = false;
    } else {
      // z-chunks: minimise waves x (chunk + ring prologue + setup) over the CTA slots of the
      // occupancy the kernel gets (2 or 1 CTAs per SM)
      const long long inplane = (long long)F->ntile[0] * F->ntile[1];
      const int mask = S.term_mask();
      const int ks = (mask & ~0x111) == 0 ? 0x111 : ((mask & ~0x11B) == 0 ? 0x11B : 0x1FF);
      const int occ = f3_wanted(p, ks) ? 1 : f2::occ_for(p, ks);
      int dev = 0, nsm = 148;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const long long slots = (long long)occ * nsm;
      const int E = S.e_hi - S.e_lo;
      int chunk = E + (E & 1);
      double best = 1e300;
      for (int nch = 1; nch <= std::max(1, E / 2); ++nch) {
        int len = (E + nch - 1) / nch;
        len += len & 1;
        const long long ctas = inplane * ((E + len - 1) / len);
        const double cost = double((ctas + slots - 1) / slots) * (len + p + 4);
        if (cost < best - 1e-9) { best = cost; chunk = len; }
      }
      if (const char* ev = getenv("MFWQ_CHUNK")) chunk = std::max(2, atoi(ev));  // tuning experiments
      chunk += chunk & 1;  // even chunks: steps of two z-elements
      for (int e = S.e_lo; e < S.e_hi; e += chunk) {
        const int b = std::min(S.e_hi, e + chunk);
        t.push_back({e, b, S.dir[2].elem_q0[e], S.dir[2].elem_q0[b] - S.dir[2].elem_q0[e]});
        F->max_nqz = std::max(F->max_nqz, t.back().nq);
        F->max_chunk = std::max(F->max_chunk, b - e);
      }
      F->q0z.upload(S.dir[2].elem_q0.data(), S.dir[2].elem_q0.size());
    }
    F->ntile[l] = int(t.size());
    F->htiles[l] = t;
    F->tiles[l].upload(t.data(), t.size());
  }
  if (ok) {  // dense per-tile operand blocks (the band matrices of one tile, zero padded)
    using namespace f2;
    const int NB = p + 1, NW = p + 2, NBP = (NB + 1) & ~1, NWP = (NW + 1) & ~1, ZT = 2 * NBP + 4 * NWP;
    const int m1 = S.dir[0].m, m2 = S.dir[1].m, m3 = S.dir[2].m;
    F->xblk_sz = 4 * TQ * PV + 2 * TQ * NB;
    F->yblk_sz = 2 * TQ * PKB + 4 * PV * PK;
    std::vector<double> xb((size_t)F->ntile[0] * F->xblk_sz, 0.0), yb((size_t)F->ntile[1] * F->yblk_sz, 0.0);
    std::vector<int> exy((size_t)(F->ntile[0] + F->ntile[1]) * TQ, 0);
    for (int i = 0; i < F->ntile[0]; ++i) {
      const Tile& t = T[0][i];
      double* o = xb.data() + (size_t)i * F->xblk_sz;
      for (int q = 0; q < t.nq; ++q) {
        const int ex = Heq[0][t.q0 + q] - t.ea;
        exy[i * TQ + q] = ex;
        for (int w = 0; w < 4; ++w)  // Wx^T(ql, c) = Wt[w][ql][c - e(ql)]
          for (int c = 0; c < PV; ++c) {
            const int k = c - ex;
            if (k >= 0 && k < NW) o[(w * TQ + q) * PV + (c ^ swz(q))] = HW[0][((size_t)w * m1 + t.q0 + q) * NW + k];
          }
        for (int b = 0; b < 2; ++b)
          for (int k = 0; k < NB; ++k) o[4 * TQ * PV + (b * TQ + q) * NB + k] = HB[0][((size_t)b * m1 + t.q0 + q) * NB + k];
      }
    }
    for (int i = 0; i < F->ntile[1]; ++i) {
      const Tile& t = T[1][i];
      double* o = yb.data() + (size_t)i * F->yblk_sz;
      for (int q = 0; q < t.nq; ++q) {
        const int ey = Heq[1][t.q0 + q] - t.ea;
        exy[(F->ntile[0] + i) * TQ + q] = ey;
        for (int b = 0; b < 2; ++b)  // By(q2, r) = Bt[b][q2][r - e(q2) - 1]
          for (int r = 0; r < PKB; ++r) {
            const int k = r - ey - 1;
            if (k >= 0 && k < NB) o[(b * TQ + q) * PKB + r] = HB[1][((size_t)b * m2 + t.q0 + q) * NB + k];
          }
        for (int w = 0; w < 4; ++w)  // Wy(r, q2) = Wt[w][q2][r - e(q2)]
          for (int r = 0; r < PV; ++r) {
            const int k = r - ey;
            if (k >= 0 && k < NW) o[2 * TQ * PKB + (w * PV + r) * PK + q] = HW[1][((size_t)w * m2 + t.q0 + q) * NW + k];
          }
      }
    }
    std::vector<double> zt((size_t)m3 * ZT, 0.0);  // z rows: B0 | B1 | W00 W01 W10 W11, sub-tables padded to even
    for (int q = 0; q < m3; ++q) {
      for (int b = 0; b < 2; ++b)
        for (int k = 0; k < NB; ++k) zt[(size_t)q * ZT + b * NBP + k] = HB[2][((size_t)b * m3 + q) * NB + k];
      for (int w = 0; w < 4; ++w)
        for (int k = 0; k < NW; ++k) zt[(size_t)q * ZT + 2 * NBP + w * NWP + k] = HW[2][((size_t)w * m3 + q) * NW + k];
    }
    F->xblk.upload(xb.data(), xb.size());
    F->yblk.upload(yb.data(), yb.size());
    F->exy.upload(exy.data(), exy.size());
    F->ztab.upload(zt.data(), zt.size());
  }
  F->qe = maxe;
  F->p = p;
  // the v-window fetch packs (in-plane DoF offset << 10 | window cell) into an int
  const bool plane_fits = (long long)S.dir[0].n * S.dir[1].n < (1ll << 21);
  F->ok = ok && maxe <= f2::TQ && plane_fits;
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

void encode_maps(Stiffness& S, Fused2Plan& F) {
  if (F.maps_for == S.coeff.ptr && F.maps_for_mass == S.mass_grid.ptr) return;
  auto enc = get_encode();
  const size_t G = S.grid_elems();
  for (int mi = 0; mi < 2 * f2::NGRID; ++mi) {
    const int g = mi % f2::NGRID;
    const double* base = g == f2::MASS_GRID ? S.mass_grid.ptr : (S.coeff.ptr ? S.coeff.ptr + g * G : nullptr);
    if (!base) continue;  // a grid this operator does not hold is never read
    cuuint64_t dims[3] = {(cuuint64_t)S.dir[0].m, (cuuint64_t)S.dir[1].m, (cuuint64_t)(S.q_hi - S.q_lo)};
    cuuint64_t strides[2] = {(cuuint64_t)S.m1p * 8, (cuuint64_t)S.m1p * S.dir[1].m * 8};
    cuuint32_t box[3] = {(cuuint32_t)f2::TQ, (cuuint32_t)f2::TQ, mi < f2::NGRID ? 4u : 2u};  // the ZS x 2 planes of a step
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&F.maps.m[mi], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaErr("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  }
  F.maps_for = S.coeff.ptr;
  F.maps_for_mass = S.mass_grid.ptr;
}

#endif

void encode_maps(Stiffness& S, Fused2Plan& F);

#ifndef MFWQ_F2_OTF_UNIT
// w = 0 ahead of the fused kernel's atomics; lets the fused kernel launch at once (its prologue
// overlaps this pass and it waits with griddepcontrol.wait before the first atomic)
__global__ void __launch_bounds__(256) f2_zero_out(double* __restrict__ y, long long n) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) y[i] = 0.0;
}
void f2_zero_and_chain(double* y, long long n, cudaStream_t s) {
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  f2_zero_out<<<nsm * 4, 256, 0, s>>>(y, n); note_launch();
}
#else
void f2_zero_and_chain(double* y, long long n, cudaStream_t s);
#endif

static void fill_params(Stiffness& S, Fused2Plan& F, const double* x, double* y, f2::Params& prm) {
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
  prm.C = S.coeff.ptr;
  prm.Cm = S.mass_grid.ptr;
  prm.gstride = S.grid_elems();
  prm.m1p = S.m1p;
  prm.x = x;
  prm.y = y;
  prm.xblk = F.xblk.ptr;
  prm.yblk = F.yblk.ptr;
  prm.exy = F.exy.ptr;
  prm.ztab = F.ztab.ptr;
  prm.xblk_sz = F.xblk_sz;
  prm.yblk_sz = F.yblk_sz;
  prm.v_lo = S.v_lo;
  prm.v_hi = S.v_hi;
  prm.y_lo = S.y_lo;
  prm.y_hi = S.y_hi;
  prm.qzb = S.q_lo;
  prm.n1 = S.dir[0].n;
  prm.n2 = S.dir[1].n;
  prm.n3 = S.dir[2].n;
  prm.qe = F.qe;
  prm.cx = S.cx.ptr;
}

// deterministic mode: the gather's candidate tables (which CTA boxes cover each DoF, in a fixed
// order) and the box geometry, built once per plan
static void det_prepare(Stiffness& S, Fused2Plan& F, int dm) {
  if (F.det_ready && F.det_dm == dm) return;
  const int p = F.p;
  auto build = [&](int l, int n, const std::vector<f2::Tile>& t, bool rows) {
    std::vector<std::vector<int2>> c(n);
    for (int k = 0; k < (int)t.size(); ++k) {
      const int lo = t[k].ea - 2, len = rows ? (t[k].eb - t[k].ea) + p + 1 : (t[k].eb - t[k].ea) + p + 1;
      for (int i = std::max(lo, 0); i < std::min(lo + len, n); ++i) c[i].push_back(make_int2(k, i - lo));
    }
    int kmax = 1;
    for (auto& v : c) kmax = std::max(kmax, (int)v.size());
    std::vector<int2> flat((size_t)n * kmax, make_int2(-1, -1));
    for (int i = 0; i < n; ++i)
      for (size_t a = 0; a < c[i].size(); ++a) flat[(size_t)i * kmax + a] = c[i][a];
    F.cand[l].upload(flat.data(), flat.size());
    F.kc[l] = kmax;
  };
  build(0, S.dir[0].n, F.htiles[0], false);
  build(1, S.dir[1].n, F.htiles[1], false);
  build(2, S.dir[2].n, F.htiles[2], true);
  F.det_dm = dm;
  F.det_box = (long long)(F.max_chunk + p + 1) * dm * dm;
  F.det_ready = true;
}

// zero w (releasing the fused kernel early), then the fused kernel with programmatic stream
// serialisation: grid (in-plane tiles, z-chunks, term subsets).  Deterministic mode: no zero pass
// (every output cell is stored, not added), the fused kernel fully stream-ordered (it reads x in
// its prologue), then the fixed-order gather into y.
template <typename K>
static void launch_chained(Stiffness& S, Fused2Plan& F, K kern, size_t smem, int nsub, f2::Params prm,
                           double* y, cudaStream_t s, int dm = 0, int nthr = f2::NTHR) {
  MFWQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const bool det = S.deterministic && dm > 0;
  const long long nctas = (long long)F.ntile[0] * F.ntile[1] * F.ntile[2];
  if (det) {
    det_prepare(S, F, dm);
    S.det_scratch.alloc_at_least((size_t)(nctas * F.det_box));
    prm.det = S.det_scratch.ptr;
    prm.det_box = F.det_box;
    prm.det_dm = F.det_dm;
  } else {
    prm.det = nullptr;
    f2_zero_and_chain(y, (long long)S.out_elems(), s);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(F.ntile[0] * F.ntile[1], F.ntile[2], nsub);
  cfg.blockDim = dim3(nthr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = det ? 0 : 1;
  MFWQ_CUDA(cudaLaunchKernelEx(&cfg, kern, prm, F.maps));
  note_launch();
  MFWQ_CUDA(cudaGetLastError());
  if (det) {
    f2::GatherTabs T{F.cand[0].ptr, F.cand[1].ptr, F.cand[2].ptr, F.kc[0], F.kc[1], F.kc[2]};
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    f2::f2_gather<<<nsm * 8, 256, 0, s>>>(y, prm.det, T, S.dir[0].n, S.dir[1].n, S.y_lo, S.y_hi, F.ntile[0],
                                          F.ntile[1], F.det_box, F.det_dm);
    note_launch();
    MFWQ_CUDA(cudaGetLastError());
  }
}

template <int P, int KS, bool OTF>
static void launch2(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
  constexpr int ZS = f2::zs_for(P, KS);
  using namespace f2;
  if constexpr (!OTF) encode_maps(S, F);
  Params prm;
  fill_params(S, F, x, y, prm);
  launch_chained(S, F, k_fused<P, KS, ZS, OTF>, Smem<P, KS, ZS, OTF>::bytes(F.qe, F.max_chunk), 1, prm, y, s,
                 Smem<P, KS, ZS, OTF>::DMAX);
}

template <int P, bool OTF>
static void dispatch2(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
  const int mask = S.term_mask();
  if ((mask & ~0x111) == 0) launch2<P, 0x111, OTF>(S, F, x, y, s);
  else if ((mask & ~0x11B) == 0) launch2<P, 0x11B, OTF>(S, F, x, y, s);
  else launch2<P, 0x1FF, OTF>(S, F, x, y, s);
}

template <bool OTF>
static bool dispatch_p(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
#ifdef MFWQ_ONLY_P  // static-analysis / experiment builds of one degree (tools/sass_stats.sh); never in the product
  if (F.p != MFWQ_ONLY_P) return false;
  dispatch2<MFWQ_ONLY_P, OTF>(S, F, x, y, s);
  return true;
#else
  switch (F.p) {
    case 1: dispatch2<1, OTF>(S, F, x, y, s); break;
    case 2: dispatch2<2, OTF>(S, F, x, y, s); break;
    case 3: dispatch2<3, OTF>(S, F, x, y, s); break;
    case 4: dispatch2<4, OTF>(S, F, x, y, s); break;
    case 5: dispatch2<5, OTF>(S, F, x, y, s); break;
    case 6: dispatch2<6, OTF>(S, F, x, y, s); break;
    case 7: dispatch2<7, OTF>(S, F, x, y, s); break;
    case 8: dispatch2<8, OTF>(S, F, x, y, s); break;
    case 9: dispatch2<9, OTF>(S, F, x, y, s); break;
    case 10: dispatch2<10, OTF>(S, F, x, y, s); break;
    default: return false;
  }
  return true;
#endif
}

#ifndef MFWQ_F2_OTF_UNIT
bool fused2_apply_otf(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s);  // fused2_otf.cu
bool fused3_apply(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s);      // fused3.cu

bool fused2_apply(Stiffness& S, const double* x, double* y, cudaStream_t s) {
  Fused2Plan* F = fused2_plan(S);
  if (!F->ok) return false;
  if (fused3_apply(S, *F, x, y, s)) return true;  // warp-specialised kernel (fused3.cu) where it applies
  if (S.otf) return fused2_apply_otf(S, *F, x, y, s);
  return dispatch_p<false>(S, *F, x, y, s);
}

bool fused2_accepts(Stiffness& S) { return fused2_plan(S)->ok; }

// the mass operator (operators.py:87-132) as the fused kernel's one-term case: B0 / W00 in every
// direction, the stored alpha det J grid; false when the rule is outside the element-blocked
// structure (the composed K1 path then runs)
template <int P>
static void launch_mass(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
  launch2<P, f2::MASS_TERM, false>(S, F, x, y, s);
}
bool fused2_apply_mass(Stiffness& S, const double* x, double* y, cudaStream_t s) {
  Fused2Plan* F = fused2_plan(S);
  if (!F->ok || !S.mass_grid.ptr) return false;
  switch (F->p) {
    case 1: launch_mass<1>(S, *F, x, y, s); break;
    case 2: launch_mass<2>(S, *F, x, y, s); break;
    case 3: launch_mass<3>(S, *F, x, y, s); break;
    case 4: launch_mass<4>(S, *F, x, y, s); break;
    case 5: launch_mass<5>(S, *F, x, y, s); break;
    case 6: launch_mass<6>(S, *F, x, y, s); break;
    case 7: launch_mass<7>(S, *F, x, y, s); break;
    case 8: launch_mass<8>(S, *F, x, y, s); break;
    case 9: launch_mass<9>(S, *F, x, y, s); break;
    case 10: launch_mass<10>(S, *F, x, y, s); break;
    default: return false;
  }
  return true;
}

void Stiffness::apply_fused(const double* x, double* y, cudaStream_t s) {
  if (fused2_apply(*this, x, y, s)) return;
  if (is_slab()) throw NotImplErr("slab operators need the element-blocked fused kernel (p <= 10, n_el >= 2)");
  apply_generic(x, y, s);  // rule outside the element-blocked structure: composed K1 path (still GPU)
}
#elif !defined(MFWQ_F3_UNIT)
bool fused2_apply_otf(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
  return dispatch_p<true>(S, F, x, y, s);
}
#endif

}  // namespace mfwq
