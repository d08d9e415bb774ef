// Fused MF-WQ stiffness matvec, v3: the warp-specialised form of fused2.cu (operators.py:185-204).
//
// Same decomposition (one CTA = one element-aligned 16 x 16 in-plane tile of quadrature columns
// streaming a chunk of z-elements), same operand blocks, tiles, tensor maps and arithmetic per
// output as fused2.cu; what changes is who does what.  fused2 runs every phase on all eight warps
// with two CTA barriers per step, so its per-thread (DFMA) z-part and its in-plane DMMA phases
// add up.  Here the roles are separate warps of one CTA per SM, coupled only by mbarrier rings:
//
//   warps 0-7   column warps: one quadrature column per thread.  x-contraction of the B-side plane
//               (ring push), z-contraction of the ring -> grad v, t_ab = C_ab g_b, z-contraction of
//               the W side into the register accumulators, retire one row per element.
//   warps 8,9   W x-contraction (DMMA): retired rows sT -> sS, the Wx^T band fragments of the tile
//               stationary in registers (m-tile 0 / 1).
//   warps 10,11 B-side y-contraction (DMMA): DoF plane window sV -> sA, the By band fragments
//               stationary in registers (n-tile 0 / 1).
//   warp 12     loader: cp.async of the v windows, TMA boxes of the coefficient planes and the bulk
//               copy of the z rows, several elements ahead.
//   warps 14,15 W y-contraction (DMMA, Wy band fragments stationary) and the fp64 atomics into w.
//
// Rings (full / empty mbarriers per stage): V loader -> B y;  A B y -> columns;  C loader -> columns;
// T columns -> W x;  S W x -> W y.  The column warps signal one barrier per step ("row retired"), which
// W x, the loader and B y all wait on.  No CTA barrier after the setup.
#define MFWQ_F2_OTF_UNIT 1
#define MFWQ_F3_UNIT 1
#include "fused2.cu"

#ifndef MFWQ_F3_ABL
#define MFWQ_F3_ABL 0  // timing experiments only (wrong results): 1 = z rows from immediates, 2 = Bx from immediates,
                       // 4 = helpers skip their DMMAs, 8 = column warps skip their arithmetic,
                       // 16 = column warps alone: helpers exit after the setup, no ring waits or arrivals
#endif
namespace mfwq {
namespace f3 {
using namespace f2;

constexpr int NTHR3 = 512;
// Roles by warp: warps 0-7 (two warpgroups) are the column warps, warps 8-15 the helpers.
// setmaxnreg moves registers from the helper warpgroups to the column warpgroups.
#ifndef MFWQ_F3_REG_COL
#define MFWQ_F3_REG_COL 160
#define MFWQ_F3_REG_HELP 96
#endif
constexpr int REG_COL = MFWQ_F3_REG_COL, REG_HELP = MFWQ_F3_REG_HELP;  // 256 x 160 + 256 x 96 = 65536
// helper index h = warp - 8.  W x alone on schedulers 0, 1 (with the loader), B y and W y share 2, 3:
// the DMMA counts per scheduler come out about even
constexpr int H_WX = 0, H_BY = 2, H_LOAD = 4, H_WY = 6;
#ifndef MFWQ_F3_SC
#define MFWQ_F3_SC 4
#endif
#ifndef MFWQ_F3_SV
#define MFWQ_F3_SV 4
#endif
#ifndef MFWQ_F3_ST
#define MFWQ_F3_ST 2
#endif
constexpr int SV = MFWQ_F3_SV, SA = 4, SC = MFWQ_F3_SC, ST = MFWQ_F3_ST, SS = MFWQ_F3_ST;  // ring depths (powers of two)
// "Row j retired" (B_FT, one arrival per column warp) is the only barrier the column warps signal per
// step: W x waits on it for the row, the loader for the coefficient stage of element j (free again)
// and B y for the A plane element j consumed.  It has NFT barriers (row j -> j mod NFT) although the
// T data ring has ST slots; no waiter is ever NFT rows behind the column warps.
constexpr int NFT = 4;
static_assert(SC <= NFT && SA <= NFT && ST <= NFT, "a waiter must see the phase it waits for");
enum {
  B_FV = 0, B_EV = B_FV + SV, B_FA = B_EV + SV, B_EA = B_FA + SA, B_FC = B_EA + SA,
  B_FT = B_FC + SC, B_ET = B_FT + NFT, B_FS = B_ET + ST, B_ES = B_FS + SS, NBAR = B_ES + SS
};

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  if (MFWQ_F3_ABL & 16) return;
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
#ifdef MFWQ_F3_PROF  // timing experiment: cycles each warp spends waiting per ring (one CTA prints)
#define WAITP(slot, b, par) { long long t0_ = clock64(); mbar_wait_acq(b, par); pw[slot] += clock64() - t0_; }
#define PROF3_DECL long long pw[7] = {0, 0, 0, 0, 0, 0, 0}; const long long pstart = clock64();
#define SECT(slot) { long long n_ = clock64(); pw[slot] += n_ - plast; plast = n_; }
#define SECT0 long long plast = clock64();
#define SECTR plast = clock64();
#define PROF3_DUMP(name) if (blockIdx.x == 40 && blockIdx.y == 0 && lane == 0) printf("F3PROF %s w%d total %lld wait0 %lld wait1 %lld wait2 %lld | s3 %lld s4 %lld s5 %lld s6 %lld\n", name, warp, clock64() - pstart, pw[0], pw[1], pw[2], pw[3], pw[4], pw[5], pw[6]);
#else
#define WAITP(slot, b, par) { if (!(MFWQ_F3_ABL & 16)) mbar_wait_acq(b, par); }
#define PROF3_DECL
#define SECT(slot)
#define SECT0
#define SECTR
#define PROF3_DUMP(name)
#endif
// coefficient boxes are read once: evict-first in L2, so the stream does not push v and w out
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d_hint(double* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], "
      "[%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}
// one arrival per warp, after every lane's accesses of the stage
__device__ __forceinline__ void warp_arrive(uint64_t* b, int lane) {
  __syncwarp();
  if (lane == 0) mbar_arrive(b);
}

template <int P, int KS, bool OTF>
struct Smem3 {
  static constexpr int NT = Terms<KS>::N;
  static constexpr int NB = P + 1, NW = P + 2;
  static constexpr int NBP = (NB + 1) & ~1, NWP = (NW + 1) & ~1;
  static constexpr int ZT = 2 * NBP + 4 * NWP;
  static constexpr int G = n_grids<KS>(), NX = n_xtypes<KS>(), NY = n_ytypes<KS>();
  static constexpr int DMAX = TQ / 2 + P + 1;
  static constexpr int KB = (DMAX + 3) / 4, VR = 4 * KB;
  static constexpr int CSZ = OTF ? 0 : G * 2 * 256;  // one coefficient stage: G boxes of 16 x 16 x 2
  static constexpr int TSZ = NT * TQ * PK, ASZ = 2 * TQ * PV, SSZ = NY * TQ * PV, VSZ = VR * PV;
  static constexpr int oC = 0, oT = oC + SC * CSZ, oBy = oT + ST * TSZ, oWx = oBy + 2 * TQ * PKB,
                       oWy = oWx + NX * TQ * PV, oV = oWy + NY * PV * PK, oA = oV + SV * VSZ, oS = oA + SA * ASZ,
                       oBx = oS + SS * SSZ, oCx = oBx + 2 * TQ * NB, oZ = oCx + (OTF ? G * TQ : 0);
  static constexpr int FPL = (DMAX * DMAX + 31) / 32;  // v-window cells per loader lane
  static size_t bytes(int qe, int max_chunk) {
    return sizeof(double) * (size_t)(oZ + SC * qe * ZT) + sizeof(uint64_t) * NBAR + sizeof(int) * 2 * TQ +
           sizeof(int) * (max_chunk + 2) + 64;
  }
};

template <int P, int KS, bool OTF>
__global__ void __launch_bounds__(NTHR3, 1) k_ws(const __grid_constant__ Params prm, const __grid_constant__ Maps maps) {
  static_assert(P <= 6, "two 8-wide tiles over the DoF window");
  using L = Smem3<P, KS, OTF>;
  using T = Terms<KS>;
  constexpr int NT = T::N;
  constexpr int NB = L::NB, NW = L::NW, NBP = L::NBP, NWP = L::NWP, ZT = L::ZT, G = L::G;
  constexpr int R = NB, A = NW, KB = L::KB;
  constexpr int NX = L::NX, NY = L::NY;
  static_assert(L::DMAX <= 16, "window wider than two n-tiles");

  const int QE = prm.qe;
  extern __shared__ __align__(128) double sm[];
  double* sC = sm + L::oC;      // [SC][G][2][256]
  double* sT = sm + L::oT;      // [ST][NT][16][PK]
  double* sBy = sm + L::oBy;    // [2][16][PKB]
  double* sWxT = sm + L::oWx;   // [NX][16][PV]
  double* sWy = sm + L::oWy;    // [NY][PV][PK]
  double* sV = sm + L::oV;      // [SV][VR][PV]
  double* sA = sm + L::oA;      // [SA][2][16][PV]
  double* sS = sm + L::oS;      // [SS][NY][16][PV]
  double* sBx = sm + L::oBx;    // [2][16][NB]
  double* sCx = sm + L::oCx;    // [G][16]
  double* sZ = sm + L::oZ;      // [SC][QE][ZT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sZ + SC * QE * ZT);
  int* sEx = reinterpret_cast<int*>(bar + NBAR);
  int* sEy = sEx + TQ;
  int* sQ0 = sEy + TQ;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool colw = warp < 8;
  const int cw = warp;       // column warp 0..7
  const int hw = warp - 8;   // helper 0..7
  const int tid = threadIdx.x;
  const int bxi = blockIdx.x % prm.ntx, byi = blockIdx.x / prm.ntx;
  const Tile tx = prm.tx[bxi], ty = prm.ty[byi], tz = prm.tz[blockIdx.y];
  const int Dx = tx.eb - tx.ea + P + 1, Dy = ty.eb - ty.ea + P + 1;
  const int dax = tx.ea - 2, day = ty.ea - 2;
  const int nez = tz.eb - tz.ea, ea3 = tz.ea;
  const int nplanes = nez + P;      // DoF planes ea3-1 .. ea3+nez+p-2 through the B side
  const int nrows = nez + NW - 1;   // output rows ea3-2 .. ea3+nez+p-2 through the W side

  // ---- one-time staging (all warps): operand blocks, element offsets, barriers ----
  {
    const double* xb = prm.xblk + (size_t)bxi * prm.xblk_sz;
    const double* yb = prm.yblk + (size_t)byi * prm.yblk_sz;
    auto copy16 = [&](double* dst, const double* src, int n) {
      for (int i = 2 * tid; i < n; i += 2 * NTHR3) cp_async16(dst + i, src + i);
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
    for (int i = tid; i <= nez; i += NTHR3) sQ0[i] = prm.q0z[ea3 + i];
    if (tid == 0) {
      for (int i = 0; i < SV; ++i) { mbar_init(&bar[B_FV + i], 32); mbar_init(&bar[B_EV + i], 2); }
      for (int i = 0; i < SA; ++i) { mbar_init(&bar[B_FA + i], 2); mbar_init(&bar[B_EA + i], 8); }
      for (int i = 0; i < SC; ++i) mbar_init(&bar[B_FC + i], 1);
      for (int i = 0; i < NFT; ++i) mbar_init(&bar[B_FT + i], 8);
      for (int i = 0; i < ST; ++i) mbar_init(&bar[B_ET + i], 2);
      for (int i = 0; i < SS; ++i) { mbar_init(&bar[B_FS + i], 2); mbar_init(&bar[B_ES + i], 2); }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    for (int i = tid; i < SV * L::VSZ; i += NTHR3) sV[i] = 0.0;
    if constexpr (OTF) {
#pragma unroll
      for (int g = 0; g < 6; ++g)
        if (grid_used<KS>(g) && tid < TQ)
          sCx[grid_slot<KS>(g) * TQ + tid] = tid < tx.nq ? prm.cx[(size_t)g * prm.m[0] + tx.q0 + tid] : 0.0;
    }
    cp_wait_all();
  }
  __syncthreads();

#ifndef MFWQ_F3_NOSETREG
  if (!colw) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_HELP));
#endif
  if ((MFWQ_F3_ABL & 16) && !colw) return;
  if (colw) {
    // =========================== column warps ===========================
#ifndef MFWQ_F3_NOSETREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_COL));
#endif
    const int ctid = cw * 32 + lane;
    const int ql1 = ctid & 15, ql2 = ctid >> 4;
    const bool active = ql1 < tx.nq && ql2 < ty.nq;
    const int ex = sEx[ql1];
    const int q0x = tx.q0, q0y = ty.q0;
    // Register windows without moves: the B-side ring (p + 1 live planes) and the W-side
    // accumulators (p + 2 open rows) live in U = p + 2 physical slots each; element i sees logical
    // slot k at physical slot (i + k) mod U.  The element loop is unrolled U-fold, so every slot
    // index is a compile-time constant (no register shifts per element).
    constexpr int U = P + 2;
    double hx[U], hy[U], h0[U];
    double acc[NT][U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      hx[k] = hy[k] = h0[k] = 0.0;
#pragma unroll
      for (int t = 0; t < NT; ++t) acc[t][k] = 0.0;
    }
    const double* const a0base = sA + ql2 * PV + ex + 1;
    const double* const bxp = sBx + ql1 * NB;
    const double* const cbase = sC + ql2 * TQ + ql1;
    double* const tbase = sT + ql2 * PK + ql1;

    // x-contraction of one y-contracted DoF plane (stage sa of the A ring) at this thread's column
    auto xcontract = [&](int sa, double& vx, double& vy, double& v0) {
      vx = vy = v0 = 0.0;
      double wx = 0.0, wy = 0.0, w0 = 0.0;  // odd-k partial sums: half the dependent chain length
      const double* a0 = a0base + sa * L::ASZ;
      const double* a1 = a0 + TQ * PV;
      const double* b0 = bxp;
      const double* b1 = b0 + TQ * NB;
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const double c0 = (MFWQ_F3_ABL & 2) ? 1.25 + k : b0[k], c1 = (MFWQ_F3_ABL & 2) ? 0.75 + k : b1[k];
        if (k & 1) {
          if constexpr (bused<KS>(0)) wx = fma(c1, a0[k], wx);
          if constexpr (bused<KS>(2) || bused<KS>(3)) w0 = fma(c0, a0[k], w0);
          if constexpr (bused<KS>(1)) wy = fma(c0, a1[k], wy);
        } else {
          if constexpr (bused<KS>(0)) vx = fma(c1, a0[k], vx);
          if constexpr (bused<KS>(2) || bused<KS>(3)) v0 = fma(c0, a0[k], v0);
          if constexpr (bused<KS>(1)) vy = fma(c0, a1[k], vy);
        }
      }
      vx += wx;
      vy += wy;
      v0 += w0;
    };
    // z-part of nq quadrature planes of one element: ring rotation RO (compile time).
    // kPair: a regular element, both planes interleaved, coefficients from the TMA stage;
    // otherwise plane by plane with the coefficients straight from global memory.
    auto zpart = [&](auto ROc, auto PAIRc, int nq, int qa, const double* zr, const double* cst) {
      constexpr int RO = decltype(ROc)::value;
      constexpr bool kPair = decltype(PAIRc)::value;
      constexpr int NPL = kPair ? 2 : 1;
      for (int zl = 0; zl < (kPair ? 1 : nq); ++zl) {
        const double* zrow = zr + zl * ZT;
        double g[NPL][4];
#pragma unroll
        for (int pl = 0; pl < NPL; ++pl) g[pl][0] = g[pl][1] = g[pl][2] = g[pl][3] = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < NBP / 2; ++k2)
#pragma unroll
          for (int pl = 0; pl < NPL; ++pl) {
            const double2 c0 = (MFWQ_F3_ABL & 1) ? make_double2(1.25 + k2, 0.75 + pl)
                                                 : reinterpret_cast<const double2*>(zrow + pl * ZT)[k2];
            const double2 c1 = (MFWQ_F3_ABL & 1) ? make_double2(1.5 + k2, 0.35 + pl)
                                                 : reinterpret_cast<const double2*>(zrow + pl * ZT + NBP)[k2];
            const int k = 2 * k2, s0 = (RO + k) % U, s1 = (RO + k + 1) % U;
            if constexpr (bused<KS>(0)) g[pl][0] = fma(c0.x, hx[s0], g[pl][0]);
            if constexpr (bused<KS>(1)) g[pl][1] = fma(c0.x, hy[s0], g[pl][1]);
            if constexpr (bused<KS>(2)) g[pl][2] = fma(c1.x, h0[s0], g[pl][2]);
            if constexpr (bused<KS>(3)) g[pl][3] = fma(c0.x, h0[s0], g[pl][3]);
            if (k + 1 < NB) {
              if constexpr (bused<KS>(0)) g[pl][0] = fma(c0.y, hx[s1], g[pl][0]);
              if constexpr (bused<KS>(1)) g[pl][1] = fma(c0.y, hy[s1], g[pl][1]);
              if constexpr (bused<KS>(2)) g[pl][2] = fma(c1.y, h0[s1], g[pl][2]);
              if constexpr (bused<KS>(3)) g[pl][3] = fma(c0.y, h0[s1], g[pl][3]);
            }
          }
        double tv[NPL][NT];
#pragma unroll
        for (int pl = 0; pl < NPL; ++pl) {
          double cg[NGRID];
#pragma unroll
          for (int gg = 0; gg < NGRID; ++gg) {
            if (!grid_used<KS>(gg)) { cg[gg] = 0.0; continue; }
            if constexpr (OTF) cg[gg] = active ? sCx[grid_slot<KS>(gg) * TQ + ql1] : 0.0;
            else if constexpr (kPair) cg[gg] = active ? cst[pl * 256 + grid_slot<KS>(gg) * 2 * 256] : 0.0;
            else cg[gg] = active ? __ldg((gg == MASS_GRID ? prm.Cm : prm.C + gg * prm.gstride) +
                                         ((size_t)(qa + zl - prm.qzb) * prm.m[1] + q0y + ql2) * prm.m1p + q0x + ql1)
                                 : 0.0;
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
          const double* w0 = zrow + 2 * NBP + w * NWP;
#pragma unroll
          for (int k2 = 0; k2 < NWP / 2; ++k2) {
            double2 c[NPL];
#pragma unroll
            for (int pl = 0; pl < NPL; ++pl)
              c[pl] = (MFWQ_F3_ABL & 1) ? make_double2(1.125 + k2, 0.7 + w + pl)
                                        : reinterpret_cast<const double2*>(w0 + pl * ZT)[k2];
            const int k = 2 * k2, s0 = (RO + k) % U, s1 = (RO + k + 1) % U;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              if (wtype(T::a(t), T::b(t), 2) != w) continue;
#pragma unroll
              for (int pl = 0; pl < NPL; ++pl) {
                acc[t][s0] = fma(c[pl].x, tv[pl][t], acc[t][s0]);
                if (k + 1 < NW) acc[t][s1] = fma(c[pl].y, tv[pl][t], acc[t][s1]);
              }
            }
          }
        }
      }
    };

    PROF3_DECL
    // prologue: planes 0 .. P fill ring slots 0 .. P (element 0 sees slots 0 .. P)
    static_for<0, P + 1>([&](auto Kc) {
      constexpr int k = decltype(Kc)::value;
      constexpr int sa = k & (SA - 1);
      WAITP(0, &bar[B_FA + sa], (k / SA) & 1);
      xcontract(sa, hx[k], hy[k], h0[k]);
      warp_arrive(&bar[B_EA + sa], lane);
    });
    // rows j = 0 .. nrows-1: elements j < nez contribute first; row j retires accumulator slot j mod U
    for (int j0 = 0; j0 < nrows; j0 += U) {
      static_for<0, U>([&](auto Uc) {
        constexpr int u = decltype(Uc)::value;
        const int j = j0 + u;
        if (j >= nrows) return;
        if (j < nez) {
          const int sc = j & (SC - 1);
          const int kn = P + j + 1, san = kn & (SA - 1);
          const bool more = j + 1 < nez;
          WAITP(1, &bar[B_FC + sc], (j / SC) & 1);
          if (more) WAITP(0, &bar[B_FA + san], (kn / SA) & 1);
          SECT0
          const int qa = sQ0[j], nq = sQ0[j + 1] - qa;
          const double* zr = sZ + sc * QE * ZT;
          // the next plane's x-contraction (into the ring slot that is free during this element)
          // shares a basic block with the z-part; after the last element it contracts an older
          // plane into a slot nobody reads
          constexpr int SN = (u + P + 1) % U;
          if (MFWQ_F3_ABL & 8) {
          } else if (nq == 2) {
            xcontract(san, hx[SN], hy[SN], h0[SN]);
            SECT(3)
            zpart(Uc, std::true_type{}, 2, qa, zr, cbase + sc * L::CSZ);
          } else {
            xcontract(san, hx[SN], hy[SN], h0[SN]);
            zpart(Uc, std::false_type{}, nq, qa, zr, nullptr);
          }
          SECT(4)
        }
        SECT0
        const int st = j & (ST - 1);
        WAITP(2, &bar[B_ET + st], ((j / ST) & 1) ^ 1);
        double* o = tbase + st * L::TSZ;
#pragma unroll
        for (int t = 0; t < NT; ++t) {  // inactive lanes hold exact zeros (their coefficients are 0)
          o[t * TQ * PK] = acc[t][u];
          acc[t][u] = 0.0;
        }
        warp_arrive(&bar[B_FT + (j & (NFT - 1))], lane);  // row j retired: also frees its coefficient stage and A plane
        SECT(6)
      });
    }
    PROF3_DUMP("col")
  } else if (hw == H_WX || hw == H_WX + 1) {
    // =========================== W x-contraction ===========================
    // S_g(q2, c) = sum_{t in g} sum_ql T_t(q2, ql) Wx_t^T(ql, c), m-tile mt, both n-tiles
    const int mt = hw - H_WX;
    // the Wx^T band fragments stay in registers when they fit next to the row fragments (up to two
    // x-types); with three x-types (the five-term kernel) they are re-read from shared memory
    constexpr bool kBwReg = NX <= 2;
    auto bwld = [&](int xs, int ks, int nt) {
      return sWxT[(xs * TQ + ks * 4 + (lane & 3)) * PV + ((nt * 8 + (lane >> 2)) ^ swz(lane & 3))];
    };
    double bw[kBwReg ? NX : 1][4][2];
    // band structure: 4 x 8 blocks of Wx^T that are entirely zero are skipped (warp-uniform masks)
    unsigned nzw = 0u;
#pragma unroll
    for (int xs = 0; xs < NX; ++xs)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const double b = bwld(xs, ks, nt);
          if constexpr (kBwReg) bw[xs][ks][nt] = b;
          if (__any_sync(0xffffffffu, b != 0.0)) nzw |= 1u << ((xs * 4 + ks) * 2 + nt);
        }
    PROF3_DECL
    for (int j = 0; j < nrows; ++j) {
      const int st = j % ST;
      WAITP(0, &bar[B_FT + (j & (NFT - 1))], (j / NFT) & 1);
      double d[NY][2][2];
#pragma unroll
      for (int ys = 0; ys < NY; ++ys)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) d[ys][nt][0] = d[ys][nt][1] = 0.0;
      const double* ap = sT + st * L::TSZ + (mt * 8 + (lane >> 2)) * PK + (lane & 3);
      double at[NT][4];
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) at[t][ks] = ap[t * TQ * PK + ks * 4];
      warp_arrive(&bar[B_ET + st], lane);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int ys = yslot<KS>(wtype(T::a(t), T::b(t), 1)), xs = xslot<KS>(wtype(T::a(t), T::b(t), 0));
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
            if (!(MFWQ_F3_ABL & 4) && (nzw & (1u << ((xs * 4 + ks) * 2 + nt))))
              dmma(d[ys][nt][0], d[ys][nt][1], at[t][ks], kBwReg ? bw[kBwReg ? xs : 0][ks][nt] : bwld(xs, ks, nt));
        }
      const int ss = j % SS;
      WAITP(1, &bar[B_ES + ss], ((j / SS) & 1) ^ 1);
#pragma unroll
      for (int ys = 0; ys < NY; ++ys)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          double* o = sS + ss * L::SSZ + (ys * TQ + mt * 8 + (lane >> 2)) * PV + ((nt * 8 + 2 * (lane & 3)) ^ swz(lane >> 2));
          *reinterpret_cast<double2*>(o) = make_double2(d[ys][nt][0], d[ys][nt][1]);
        }
      warp_arrive(&bar[B_FS + ss], lane);
    }
    PROF3_DUMP("wx")
  } else if (hw == H_BY || hw == H_BY + 1) {
    // =========================== B-side y-contraction ===========================
    // A_b(q2, c) = sum_r By_b(q2, r) V(r, c), n-tile nt, both m-tiles, both By types
    const int nt = hw - H_BY;
    constexpr bool kA0 = bused<KS>(0) || bused<KS>(2) || bused<KS>(3), kA1 = bused<KS>(1);
    constexpr int NBY = (kA0 ? 1 : 0) + (kA1 ? 1 : 0);
    double a[NBY][2][KB];
#pragma unroll
    for (int bs = 0; bs < NBY; ++bs) {
      const int b = NBY == 2 ? bs : (kA0 ? 0 : 1);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int ks = 0; ks < KB; ++ks) a[bs][mt][ks] = sBy[(b * TQ + mt * 8 + (lane >> 2)) * PKB + ks * 4 + (lane & 3)];
    }
    unsigned nzb = 0u;  // zero 8 x 4 blocks of the By band are skipped
#pragma unroll
    for (int bs = 0; bs < NBY; ++bs)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int ks = 0; ks < KB; ++ks)
          if (__any_sync(0xffffffffu, a[bs][mt][ks] != 0.0)) nzb |= 1u << (mt * KB + ks);
    PROF3_DECL
    for (int k = 0; k < nplanes; ++k) {
      const int sv = k % SV;
      WAITP(0, &bar[B_FV + sv], (k / SV) & 1);
      double bv[KB];
      const double* bp = sV + sv * L::VSZ + (lane & 3) * PV + ((nt * 8 + (lane >> 2)) ^ swz(lane & 3));
#pragma unroll
      for (int ks = 0; ks < KB; ++ks) bv[ks] = bp[ks * 4 * PV];
      warp_arrive(&bar[B_EV + sv], lane);
      double d[NBY][2][2];
#pragma unroll
      for (int bs = 0; bs < NBY; ++bs)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) d[bs][mt][0] = d[bs][mt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KB; ++ks)
#pragma unroll
        for (int bs = 0; bs < NBY; ++bs)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
            if (!(MFWQ_F3_ABL & 4) && (nzb & (1u << (mt * KB + ks)))) dmma(d[bs][mt][0], d[bs][mt][1], a[bs][mt][ks], bv[ks]);
      const int sa = k % SA;
      if (k >= SA) {  // the plane that held this stage: x-contracted in the prologue (planes 0 .. P), else by element kp - P - 1
        const int kp = k - SA;
        if (kp <= P) { WAITP(1, &bar[B_EA + (kp & (SA - 1))], (kp / SA) & 1); }
        else { const int r = kp - P - 1; WAITP(1, &bar[B_FT + (r & (NFT - 1))], (r / NFT) & 1); }
      }
#pragma unroll
      for (int bs = 0; bs < NBY; ++bs) {
        const int b = NBY == 2 ? bs : (kA0 ? 0 : 1);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          double* o = sA + sa * L::ASZ + (b * TQ + mt * 8 + (lane >> 2)) * PV + nt * 8 + 2 * (lane & 3);
          *reinterpret_cast<double2*>(o) = make_double2(d[bs][mt][0], d[bs][mt][1]);
        }
      }
      warp_arrive(&bar[B_FA + sa], lane);
    }
    PROF3_DUMP("by")
  } else if (hw == H_LOAD) {
    // =========================== loader ===========================
    int code[L::FPL];  // (global in-plane offset << 10 | window cell), -1 = outside the domain
#pragma unroll
    for (int j = 0; j < L::FPL; ++j) {
      const int e = lane + 32 * j, r = e / Dx, c = e % Dx, g2 = day + r, g1 = dax + c;
      const bool ok = e < Dy * Dx && g2 >= 0 && g2 < prm.n2 && g1 >= 0 && g1 < prm.n1;
      code[j] = ok ? ((g2 * prm.n1 + g1) << 10) | (r * PV + (c ^ swz(r))) : -1;
    }
    const uint64_t pol = l2_evict_first_policy();
    PROF3_DECL
    for (int it = 0; it < nplanes; ++it) {
      const int sv = it % SV;
      WAITP(0, &bar[B_EV + sv], ((it / SV) & 1) ^ 1);
      SECT0
      const int i3 = ea3 - 1 + it;
      const bool vp = i3 >= prm.v_lo && i3 < prm.v_hi;
      double* dst = sV + sv * L::VSZ;
      const double* src = prm.x + (vp ? (size_t)(i3 - prm.v_lo) * prm.n2 * prm.n1 : 0);
#pragma unroll
      for (int j = 0; j < L::FPL; ++j)
        if (code[j] >= 0) cp_async8(dst + (code[j] & 1023), src + (code[j] >> 10), vp);
      SECT(3)
      cp_async_arrive(&bar[B_FV + sv]);
      SECT(4)
      if (it >= P && lane == 0) {  // the stage of element it - P: z rows, coefficient boxes of a regular element
        const int el = it - P, sc = el % SC;
        if (el >= SC) { const int r = el - SC; WAITP(1, &bar[B_FT + (r & (NFT - 1))], (r / NFT) & 1); }
        SECTR
        const int qa = sQ0[el], nq = sQ0[el + 1] - qa;
        const bool tma = !OTF && nq == 2;
        mbar_expect_tx(&bar[B_FC + sc], (unsigned)(nq * ZT * 8) + (tma ? G * 2 * TQ * TQ * 8 : 0));
        bulk_load(sZ + sc * QE * ZT, prm.ztab + (size_t)qa * ZT, (unsigned)(nq * ZT * 8), &bar[B_FC + sc]);
        if (tma) {
#pragma unroll
          for (int h = 0; h < NGRID; ++h)
            if (grid_used<KS>(h))
              tma_load_3d_hint(sC + sc * L::CSZ + grid_slot<KS>(h) * 2 * 256, &maps.m[NGRID + h], tx.q0, ty.q0, qa - prm.qzb,
                               &bar[B_FC + sc], pol);
        }
        SECT(5)
      }
      SECTR
      __syncwarp();
      SECT(6)
    }
    PROF3_DUMP("load")
  } else if (hw == H_WY || hw == H_WY + 1) {
    // =========================== W y-contraction + output ===========================
    // out(r, c) = sum_g sum_q2 Wy_g(r, q2) S_g(q2, c), n-tile nt, both m-tiles
    const int nt = hw - H_WY;
    constexpr bool kAwReg = NY <= 2;  // three y-types: the Wy band fragments are re-read from shared memory
    auto awld = [&](int ys, int mt, int ks) { return sWy[(ys * PV + mt * 8 + (lane >> 2)) * PK + ks * 4 + (lane & 3)]; };
    double aw[kAwReg ? NY : 1][2][4];
    unsigned nzy = 0u;  // zero 8 x 4 blocks of the Wy band are skipped
#pragma unroll
    for (int ys = 0; ys < NY; ++ys)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const double a = awld(ys, mt, ks);
          if constexpr (kAwReg) aw[ys][mt][ks] = a;
          if (__any_sync(0xffffffffu, a != 0.0)) nzy |= 1u << ((ys * 2 + mt) * 4 + ks);
        }
    // w is zeroed by the preceding grid (programmatic dependent launch): wait before any atomic
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const int n1 = prm.n1, n2 = prm.n2;
    const int c = nt * 8 + 2 * (lane & 3), g1 = dax + c;
    PROF3_DECL
    for (int j = 0; j < nrows; ++j) {
      const int ss = j % SS;
      WAITP(0, &bar[B_FS + ss], (j / SS) & 1);
      double bs[NY][4];
      const double* bp = sS + ss * L::SSZ + (lane & 3) * PV + ((nt * 8 + (lane >> 2)) ^ swz(lane & 3));
#pragma unroll
      for (int ys = 0; ys < NY; ++ys)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) bs[ys][ks] = bp[(ys * TQ + ks * 4) * PV];
      warp_arrive(&bar[B_ES + ss], lane);
      const int i3 = ea3 - 2 + j;
      if (i3 < prm.y_lo || i3 >= prm.y_hi) continue;  // warp-uniform
      double d[2][2][2];  // [mt][chain][2]
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) d[mt][0][0] = d[mt][0][1] = d[mt][1][0] = d[mt][1][1] = 0.0;
#pragma unroll
      for (int ys = 0; ys < NY; ++ys)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
            if (!(MFWQ_F3_ABL & 4) && (nzy & (1u << ((ys * 2 + mt) * 4 + ks))))
              dmma(d[mt][ks & 1][0], d[mt][ks & 1][1], kAwReg ? aw[kAwReg ? ys : 0][mt][ks] : awld(ys, mt, ks), bs[ys][ks]);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double d0 = d[mt][0][0] + d[mt][1][0], d1 = d[mt][0][1] + d[mt][1][1];
        const int r = mt * 8 + (lane >> 2), g2 = day + r;
        if (prm.det) {  // deterministic: this CTA's box, plain stores
          if (r < Dy) {
            const int dm = prm.det_dm;
            double* o = prm.det + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * prm.det_box + ((size_t)j * dm + r) * dm + c;
            if (c < Dx) o[0] = d0;
            if (c + 1 < Dx) o[1] = d1;
          }
          continue;
        }
        if (r < Dy && g2 >= 0 && g2 < n2) {
          double* row = prm.y + ((size_t)(i3 - prm.y_lo) * n2 + g2) * n1;
          if (c < Dx && g1 >= 0 && g1 < n1) atomicAdd(row + g1, d0);
          if (c + 1 < Dx && g1 + 1 >= 0 && g1 + 1 < n1) atomicAdd(row + g1 + 1, d1);
        }
      }
    }
    PROF3_DUMP("wy")
  }
}

}  // namespace f3

template <int P, int KS, bool OTF>
static void launch3(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
  using namespace f2;
  if constexpr (!OTF) encode_maps(S, F);
  Params prm;
  fill_params(S, F, x, y, prm);
  using L = f3::Smem3<P, KS, OTF>;
  launch_chained(S, F, f3::k_ws<P, KS, OTF>, L::bytes(F.qe, F.max_chunk), 1, prm, y, s, L::DMAX, f3::NTHR3);
}

template <int P>
static void dispatch3(Stiffness& S, Fused2Plan& F, int ks, const double* x, double* y, cudaStream_t s) {
  if (S.otf) {
    if (ks == 0x111) launch3<P, 0x111, true>(S, F, x, y, s);
    else launch3<P, 0x11B, true>(S, F, x, y, s);
  } else {
    if (ks == 0x111) launch3<P, 0x111, false>(S, F, x, y, s);
    else launch3<P, 0x11B, false>(S, F, x, y, s);
  }
}

bool fused3_apply(Stiffness& S, Fused2Plan& F, const double* x, double* y, cudaStream_t s) {
  const int mask = S.term_mask();
  const int ks = (mask & ~0x111) == 0 ? 0x111 : ((mask & ~0x11B) == 0 ? 0x11B : 0x1FF);
  if (!f3_wanted(F.p, ks)) return false;
#ifdef MFWQ_F3_ONLY_P  // experiment builds: one degree only
  if (F.p != MFWQ_F3_ONLY_P) return false;
  dispatch3<MFWQ_F3_ONLY_P>(S, F, ks, x, y, s);
#else
  switch (F.p) {
    case 1: dispatch3<1>(S, F, ks, x, y, s); break;
    case 2: dispatch3<2>(S, F, ks, x, y, s); break;
    case 3: dispatch3<3>(S, F, ks, x, y, s); break;
    case 4: dispatch3<4>(S, F, ks, x, y, s); break;
    case 5: dispatch3<5>(S, F, ks, x, y, s); break;
    case 6: dispatch3<6>(S, F, ks, x, y, s); break;
    default: return false;
  }
#endif
  return true;
}

}  // namespace mfwq
