// Device-resident preconditioned CG (solvers.py:137-173) with fused
// reduction/update kernels.  All vectors stay in HBM; per iteration the host
// reads back two scalars (p.Ap and ||r||^2) for the indefiniteness and
// stopping tests, exactly where the reference takes those decisions.
#include <cmath>
#include <functional>
#include <cstdint>

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
// 16-byte accesses, two pairs per thread per trip (all vectors 16-byte aligned; the odd tail
// element, if any, is done by the last thread of block 0).  Summation order of the partials is
// fixed by the grid, so the result is deterministic.
__global__ void __launch_bounds__(RB) update_xr(double* __restrict__ x, double* __restrict__ r,
                                                const double* __restrict__ p, const double* __restrict__ Ap,
                                                long long N, const double* __restrict__ rz,
                                                const double* __restrict__ pAp, double* __restrict__ partial) {
  const double alpha = *rz / *pAp;
  double s = 0.0;
  const long long N2 = N >> 1, stride = (long long)gridDim.x * RB;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* a2 = reinterpret_cast<const double2*>(Ap);
  long long i = blockIdx.x * (long long)RB + threadIdx.x;
  for (; i + stride < N2; i += 2 * stride) {
    const double2 xa = x2[i], xb = x2[i + stride], pa = p2[i], pb = p2[i + stride];
    const double2 ra = r2[i], rb = r2[i + stride], aa = a2[i], ab = a2[i + stride];
    x2[i] = make_double2(xa.x + alpha * pa.x, xa.y + alpha * pa.y);
    x2[i + stride] = make_double2(xb.x + alpha * pb.x, xb.y + alpha * pb.y);
    const double2 na = make_double2(ra.x - alpha * aa.x, ra.y - alpha * aa.y);
    const double2 nb = make_double2(rb.x - alpha * ab.x, rb.y - alpha * ab.y);
    r2[i] = na;
    r2[i + stride] = nb;
    s += na.x * na.x;
    s += na.y * na.y;
    s += nb.x * nb.x;
    s += nb.y * nb.y;
  }
  for (; i < N2; i += stride) {
    const double2 xa = x2[i], pa = p2[i], ra = r2[i], aa = a2[i];
    x2[i] = make_double2(xa.x + alpha * pa.x, xa.y + alpha * pa.y);
    const double2 na = make_double2(ra.x - alpha * aa.x, ra.y - alpha * aa.y);
    r2[i] = na;
    s += na.x * na.x;
    s += na.y * na.y;
  }
  if ((N & 1) && blockIdx.x == 0 && threadIdx.x == RB - 1) {
    x[N - 1] += alpha * p[N - 1];
    const double ri = r[N - 1] - alpha * Ap[N - 1];
    r[N - 1] = ri;
    s += ri * ri;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// p = z + (rz_new / rz) p ; rz = rz_new
__global__ void __launch_bounds__(RB) update_p(double* __restrict__ p, const double* __restrict__ z, long long N,
                                               const double* __restrict__ rz_new, const double* __restrict__ rz) {
  const double beta = *rz_new / *rz;
  const long long N2 = N >> 1, stride = (long long)gridDim.x * RB;
  double2* p2 = reinterpret_cast<double2*>(p);
  const double2* z2 = reinterpret_cast<const double2*>(z);
  long long i = blockIdx.x * (long long)RB + threadIdx.x;
  for (; i + stride < N2; i += 2 * stride) {
    const double2 pa = p2[i], pb = p2[i + stride], za = z2[i], zb = z2[i + stride];
    p2[i] = make_double2(za.x + beta * pa.x, za.y + beta * pa.y);
    p2[i + stride] = make_double2(zb.x + beta * pb.x, zb.y + beta * pb.y);
  }
  for (; i < N2; i += stride) {
    const double2 pa = p2[i], za = z2[i];
    p2[i] = make_double2(za.x + beta * pa.x, za.y + beta * pa.y);
  }
  if ((N & 1) && blockIdx.x == 0 && threadIdx.x == RB - 1) p[N - 1] = z[N - 1] + beta * p[N - 1];
}

__global__ void copy_scalar(const double* src, double* dst) { *dst = *src; }

static void dot_to(const double* a, const double* b, long long N, double* partial, double* out, cudaStream_t s) {
  dot_partial<<<RGRID, RB, 0, s>>>(a, b, N, partial); note_launch();
  finish_sum<<<1, RB, 0, s>>>(partial, RGRID, out); note_launch();
}

// building blocks shared with the slab-distributed solver (dist.cu)
void vec_dot_to(const double* a, const double* b, long long N, double* partial, double* out, cudaStream_t s) {
  dot_to(a, b, N, partial, out, s);
}
void vec_update_xr(double* x, double* r, const double* p, const double* Ap, long long N, const double* rz,
                   const double* pAp, double* partial, double* rr, cudaStream_t s) {
  update_xr<<<RGRID, RB, 0, s>>>(x, r, p, Ap, N, rz, pAp, partial); note_launch();
  finish_sum<<<1, RB, 0, s>>>(partial, RGRID, rr); note_launch();
}
void vec_update_p(double* p, const double* z, long long N, const double* rz_new, double* rz, cudaStream_t s) {
  update_p<<<RGRID, RB, 0, s>>>(p, z, N, rz_new, rz); note_launch();
  copy_scalar<<<1, 1, 0, s>>>(rz_new, rz); note_launch();
}
int vec_partials() { return RGRID; }

double dev_dot(const double* a, const double* b, long long N, cudaStream_t s) {
  DevBuf<double> part(RGRID), out(1);
  dot_to(a, b, N, part.ptr, out.ptr, s);
  double h;
  MFWQ_CUDA(cudaMemcpyAsync(&h, out.ptr, sizeof h, cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
  return h;
}

// Graph cache of one (operator, preconditioner) pair: the PCG iteration bodies captured once and
// replayed, so a solve issues a handful of graph launches instead of ~20 kernel launches per
// iteration (the small-problem solve is launch-latency bound: cfg 1).  Captured after a first
// eager solve has created every plan, scratch buffer and tensor map the bodies touch.
struct PcgGraphs {
  FastDiag* P = nullptr;
  long long N = 0;
  const double* ws = nullptr;
  const double* hslot = nullptr;
  int device = -1;
  cudaStream_t cs = nullptr;  // capture stream (the caller's may be the legacy default stream)
  cudaGraphExec_t init = nullptr, full = nullptr, aonly = nullptr, ponly = nullptr;
  long long nk_init = 0, nk_full = 0, nk_a = 0, nk_p = 0;
  bool ready = false;
  ~PcgGraphs() {
    for (cudaGraphExec_t g : {init, full, aonly, ponly})
      if (g) cudaGraphExecDestroy(g);
    if (cs) cudaStreamDestroy(cs);
  }
};

static cudaGraphExec_t capture(cudaStream_t cs, long long& nk, const std::function<void()>& body) {
  const long long c0 = __atomic_load_n(&g_launches, __ATOMIC_RELAXED);
  MFWQ_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(cs, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  cudaGraph_t g = nullptr;
  MFWQ_CUDA(cudaStreamEndCapture(cs, &g));
  nk = __atomic_load_n(&g_launches, __ATOMIC_RELAXED) - c0;
  __atomic_sub_fetch(&g_launches, nk, __ATOMIC_RELAXED);  // captured, not launched
  cudaGraphExec_t e = nullptr;
  const cudaError_t err = cudaGraphInstantiate(&e, g, 0);
  cudaGraphDestroy(g);
  MFWQ_CUDA(err);
  return e;
}

static void replay(cudaGraphExec_t g, long long nk, cudaStream_t s) {
  MFWQ_CUDA(cudaGraphLaunch(g, s));
  __atomic_add_fetch(&g_launches, nk, __ATOMIC_RELAXED);
}

void pcg_solve(Stiffness& A, FastDiag* P, const double* b, double* x, long long N, double tol, int maxit,
               std::vector<double>& hist, KrylovOut& out, cudaStream_t s) {
  hist.clear();
  out = KrylovOut{};
  // persistent workspace on the operator (no cudaMalloc/cudaFree inside the solve), work vectors at
  // a 32-double pitch (256-byte aligned for the 16-byte update kernels); the iterate x lives in the
  // workspace too and is copied to the caller's buffer at the end, so the captured bodies never see
  // a caller pointer
  const long long NP = (N + 31) & ~31LL;
  A.pcg_ws.alloc_at_least(5 * NP + RGRID + 32);
  double* r = A.pcg_ws.ptr;
  double* z = r + NP;
  double* p = z + NP;
  double* Ap = p + NP;
  double* xw = Ap + NP;
  double* part = xw + NP;
  double* sc = part + RGRID;  // 0 rz, 1 pAp, 2 rr, 3 rz_new
  double* rz = sc;
  double* pAp = sc + 1;
  double* rr = sc + 2;
  double* rzn = sc + 3;
  // pinned landing slot for the scalars and the event marking their arrival: created once per host
  // thread; the event belongs to a device, so there is one per device the thread solves on
  constexpr int MAXDEV = 64;
  struct ScalarSlot {
    cudaEvent_t ev[64] = {};
    double* h = nullptr;
    ~ScalarSlot() {
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
      if (h) cudaFreeHost(h);
    }
  };
  static thread_local ScalarSlot slot;
  int cur_dev = 0;
  MFWQ_CUDA(cudaGetDevice(&cur_dev));
  if (cur_dev < 0 || cur_dev >= MAXDEV) throw ValueErr("device index out of range");
  if (!slot.h) MFWQ_CUDA(cudaMallocHost(&slot.h, 4 * sizeof(double)));
  if (!slot.ev[cur_dev]) MFWQ_CUDA(cudaEventCreateWithFlags(&slot.ev[cur_dev], cudaEventDisableTiming));
  cudaEvent_t ev = slot.ev[cur_dev];
  double* hsc = slot.h;

  // the host-visible event: an external event node when the body is being captured
  bool capturing = false;
  auto record = [&](cudaStream_t t) {
    if (capturing) MFWQ_CUDA(cudaEventRecordWithFlags(ev, t, cudaEventRecordExternal));
    else MFWQ_CUDA(cudaEventRecord(ev, t));
  };
  // the iteration bodies (each enqueued on stream t)
  auto body_init = [&](cudaStream_t t) {  // z = P r, p = z, rz = r.z  (solvers.py:147-151)
    if (P) P->apply(r, z, t);
    else MFWQ_CUDA(cudaMemcpyAsync(z, r, N * sizeof(double), cudaMemcpyDeviceToDevice, t));
    MFWQ_CUDA(cudaMemcpyAsync(p, z, N * sizeof(double), cudaMemcpyDeviceToDevice, t));
    dot_to(r, z, N, part, rz, t);
    MFWQ_CUDA(cudaMemcpyAsync(hsc + 2, rr, sizeof(double), cudaMemcpyDeviceToHost, t));  // ||b||^2
    record(t);
  };
  auto body_a = [&](cudaStream_t t) {  // Ap, p.Ap, x / r update, ||r||^2 -> host (solvers.py:154-165)
    A.apply(p, Ap, t);
    dot_to(p, Ap, N, part, pAp, t);
    update_xr<<<RGRID, RB, 0, t>>>(xw, r, p, Ap, N, rz, pAp, part); note_launch();
    finish_sum<<<1, RB, 0, t>>>(part, RGRID, rr); note_launch();
    MFWQ_CUDA(cudaGetLastError());
    MFWQ_CUDA(cudaMemcpyAsync(hsc, pAp, 2 * sizeof(double), cudaMemcpyDeviceToHost, t));
    record(t);
  };
  auto body_p = [&](cudaStream_t t) {  // z = P r, p = z + beta p  (solvers.py:168-172)
    if (P) P->apply(r, z, t);
    else MFWQ_CUDA(cudaMemcpyAsync(z, r, N * sizeof(double), cudaMemcpyDeviceToDevice, t));
    dot_to(r, z, N, part, rzn, t);
    update_p<<<RGRID, RB, 0, t>>>(p, z, N, rzn, rz); note_launch();
    copy_scalar<<<1, 1, 0, t>>>(rzn, rz); note_launch();
    MFWQ_CUDA(cudaGetLastError());
  };

  // graphs: built after the first eager solve of this (A, P) pair on this device and host slot
  // a reference keeps the cache alive for this solve even if the operator drops it meanwhile
  const std::shared_ptr<void> Gkeep = A.pcg_graphs;
  auto* G = static_cast<PcgGraphs*>(Gkeep.get());
  const bool graphs_ok = !getenv("MFWQ_NO_PCG_GRAPHS");
  const bool use_graphs = graphs_ok && G && G->ready && G->P == P && G->N == N && G->ws == A.pcg_ws.ptr &&
                          G->hslot == hsc && G->device == cur_dev;

  MFWQ_CUDA(cudaMemsetAsync(xw, 0, N * sizeof(double), s));
  MFWQ_CUDA(cudaMemcpyAsync(r, b, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  dot_to(b, b, N, part, rr, s);
  // the preconditioner of the first step runs before ||b|| is known on the host: if b = 0 it only
  // produces zeros, which are discarded (solvers.py:142-143 returns before P is applied)
  if (use_graphs) replay(G->init, G->nk_init, s);
  else body_init(s);
  MFWQ_CUDA(cudaEventSynchronize(ev));
  const double bnorm = std::sqrt(hsc[2]);
  auto finish = [&]() {
    MFWQ_CUDA(cudaMemcpyAsync(x, xw, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    MFWQ_CUDA(cudaStreamSynchronize(s));
  };
  if (bnorm == 0.0) {
    hist.push_back(0.0);
    out.converged = 1;
    finish();
    return;
  }
  out.precs = 1;
  hist.push_back(1.0);
  // The next preconditioner apply (and its r.z / p update) is enqueued BEFORE the host reads the
  // iteration's scalars whenever the last residual is far above tol: the device then never idles
  // through the host round trip.  The arithmetic and its order are unchanged; on a (rare) wrong
  // guess the extra work is simply dropped (counters count only what the reference would do).
  double last_rel = 1.0;
  bool done = false;
  for (int k = 1; k <= maxit && !done; ++k) {
    // not on the first step: an exact preconditioner (identity geometry: FD inverts the WQ
    // stiffness) converges there, and the speculative apply would be pure waste
    const bool ahead = k > 1 && k < maxit && last_rel > 1e3 * tol;
    if (use_graphs) replay(ahead ? G->full : G->aonly, ahead ? G->nk_full : G->nk_a, s);
    else {
      body_a(s);
      if (ahead) body_p(s);
    }
    out.matvecs++;
    MFWQ_CUDA(cudaEventSynchronize(ev));
    const double pap = hsc[0], rrv = hsc[1];
    if (pap <= 0) {  // solvers.py:156-160
      char m[128];
      snprintf(m, sizeof m, "nonpositive curvature p.Ap = %.3e at iteration %d", pap, k);
      MFWQ_CUDA(cudaStreamSynchronize(s));
      throw IndefiniteErr(m);
    }
    const double rel = std::sqrt(rrv) / bnorm;
    hist.push_back(rel);
    last_rel = rel;
    if (rel <= tol) {
      out.iterations = k;
      out.converged = 1;
      done = true;
      break;
    }
    if (!ahead) {
      if (use_graphs) replay(G->ponly, G->nk_p, s);
      else body_p(s);
    }
    out.precs++;
  }
  if (!done) {
    out.iterations = maxit;
    out.converged = 0;
  }
  finish();
  if (graphs_ok && !use_graphs && !(G && G->N == -1)) {  // capture the bodies for the next solve of this pair
    auto* NG = new PcgGraphs();
    A.pcg_graphs = std::shared_ptr<void>(NG, [](void* q) { delete static_cast<PcgGraphs*>(q); });
    NG->P = P;
    NG->N = N;
    NG->ws = A.pcg_ws.ptr;
    NG->hslot = hsc;
    NG->device = cur_dev;
    try {  // an operator path that cannot be captured keeps solving eagerly (the solve above is done)
      MFWQ_CUDA(cudaStreamCreateWithFlags(&NG->cs, cudaStreamNonBlocking));
      capturing = true;
      NG->init = capture(NG->cs, NG->nk_init, [&] { body_init(NG->cs); });
      NG->aonly = capture(NG->cs, NG->nk_a, [&] { body_a(NG->cs); });
      NG->ponly = capture(NG->cs, NG->nk_p, [&] { body_p(NG->cs); });
      NG->full = capture(NG->cs, NG->nk_full, [&] {
        body_a(NG->cs);
        body_p(NG->cs);
      });
      NG->ready = true;
      capturing = false;
    } catch (const std::exception&) {
      capturing = false;
      cudaGetLastError();  // clear a sticky capture error
      NG->ready = false;
      NG->P = nullptr;
      NG->N = -1;  // never matches: this pair stays eager
    }
  }
}

}  // namespace mfwq
