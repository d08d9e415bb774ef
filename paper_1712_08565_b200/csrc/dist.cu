// Slab-distributed, device-resident FD-preconditioned CG: the `comm` variant of mfwq_pcg_solve
// (solvers.py:137-173 over xi3 slabs).
//
// Partition: rank r owns z-elements [E_r, E_r+1), E_r = r n_el / world, and interior DoF planes
// [lo_r, hi_r) = [E_r - 1, E_r+1 - 1) (first / last rank clipped to [0, n3)); every vector is a
// contiguous slice of the flat (n3, n2, n1) vector.  Per iteration:
//   matvec   p lives in a window buffer [lo, vhi): the p planes above hi (forward halo) are received
//            straight into it, so the slab kernel reads its input window with no copy; it writes
//            rows [ylo, yhi) (1 below, p above the owned rows, zeroed by the kernel's own pre-pass),
//            whose off-slab rows go to their owners and are added there (reverse halo).
//   FD       directions 1, 2 local; an all-to-all to an i2-row partition for direction 3 (U3^T with
//            the fused eigenvalue scale, then U3) and back; directions 2, 1 local.
//   dots     fused update / reduction kernels per rank, the per-rank sums allreduced as scalars;
//            one host read per iteration (p.Ap and ||r||^2, exactly where the reference decides).
// The exchanges go through a Transport: NCCL (one rank per process and GPU, NVLink/NVSwitch), or
// the in-process transport that drives every rank of the partition from one process on one device
// (one cudaMemcpyAsync per message, all ranks on one stream): the same solver code, the same slab
// kernels and messages, checkable 1-vs-P on a single GPU.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "nccl.h"
#include "ops.h"

namespace mfwq {

// ---------------------------------------------------------------------------------------------
// transports
// ---------------------------------------------------------------------------------------------
struct Transport {
  virtual ~Transport() {}
  int world_ = 1, first_ = 0, nlocal_ = 1;
  virtual void begin(cudaStream_t s) = 0;
  virtual void send(int l, const double* buf, size_t n, int peer) = 0;  // from local rank l to global peer
  virtual void recv(int l, double* buf, size_t n, int peer) = 0;        // into local rank l from global peer
  virtual void end() = 0;
  // in-place sum of `count` doubles over all ranks; bufs[l] is local rank l's device buffer
  virtual void allreduce(double* const* bufs, int count, cudaStream_t s) = 0;
};

constexpr int MAX_LOCAL = 16;
struct PtrSet { double* p[MAX_LOCAL]; };
// fixed rank order, so every rank gets the bitwise identical sum
__global__ void allreduce_local_kernel(PtrSet b, int nr, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nr; ++r) s += b.p[r][i];
    for (int r = 0; r < nr; ++r) b.p[r][i] = s;
  }
}

struct LocalTransport : Transport {
  struct Msg { int from, to; const double* src; double* dst; size_t n; };
  std::vector<Msg> sends, recvs;
  cudaStream_t s_ = nullptr;
  explicit LocalTransport(int world) {
    if (world < 1 || world > MAX_LOCAL) throw ValueErr("in-process transport: 1 <= world <= 16");
    world_ = nlocal_ = world;
    first_ = 0;
  }
  void begin(cudaStream_t s) override {
    s_ = s;
    sends.clear();
    recvs.clear();
  }
  void send(int l, const double* buf, size_t n, int peer) override { sends.push_back({l, peer, buf, nullptr, n}); }
  void recv(int l, double* buf, size_t n, int peer) override { recvs.push_back({peer, l, nullptr, buf, n}); }
  void end() override {
    // match in posting order per (from, to) pair, like NCCL's send/recv matching
    std::vector<char> used(sends.size(), 0);
    for (const Msg& r : recvs) {
      size_t k = 0;
      for (; k < sends.size(); ++k)
        if (!used[k] && sends[k].from == r.from && sends[k].to == r.to) break;
      if (k == sends.size()) throw ValueErr("in-process transport: receive without a matching send");
      if (sends[k].n != r.n) throw ValueErr("in-process transport: message size mismatch");
      used[k] = 1;
      if (r.n) MFWQ_CUDA(cudaMemcpyAsync(r.dst, sends[k].src, r.n * sizeof(double), cudaMemcpyDeviceToDevice, s_));
    }
    for (char u : used)
      if (!u) throw ValueErr("in-process transport: send without a matching receive");
  }
  void allreduce(double* const* bufs, int count, cudaStream_t s) override {
    PtrSet b{};
    for (int r = 0; r < nlocal_; ++r) b.p[r] = bufs[r];
    allreduce_local_kernel<<<1, 32, 0, s>>>(b, nlocal_, count); note_launch();
    MFWQ_CUDA(cudaGetLastError());
  }
};

// NCCL, loaded at run time from the library the caller names (torch's bundled NCCL: one NCCL per
// process, no link-time dependency of libmfwq.so)
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  void load(const char* path) {
    if (h) return;
    h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) throw ValueErr(std::string("cannot load NCCL: ") + dlerror());
    auto sym = [&](const char* n) {
      void* f = dlsym(h, n);
      if (!f) throw ValueErr(std::string("NCCL library lacks ") + n);
      return f;
    };
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    Send = reinterpret_cast<decltype(Send)>(sym("ncclSend"));
    Recv = reinterpret_cast<decltype(Recv)>(sym("ncclRecv"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
  }
};
static NcclApi g_nccl;

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw CudaErr(std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "NCCL error"));
}

void nccl_unique_id(const char* lib, unsigned char* id128) {
  g_nccl.load(lib);
  ncclUniqueId id;
  nccl_check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == NCCL_UNIQUE_ID_BYTES, "unique id size");
  std::memcpy(id128, &id, sizeof id);
}

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  cudaStream_t s_ = nullptr;
  NcclTransport(const char* lib, const unsigned char* id128, int world, int rank) {
    g_nccl.load(lib);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    nccl_check(g_nccl.CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
    world_ = world;
    first_ = rank;
    nlocal_ = 1;
  }
  ~NcclTransport() override {
    if (comm) g_nccl.CommDestroy(comm);
  }
  void begin(cudaStream_t s) override {
    s_ = s;
    nccl_check(g_nccl.GroupStart(), "ncclGroupStart");
  }
  void send(int, const double* buf, size_t n, int peer) override {
    nccl_check(g_nccl.Send(buf, n, ncclDouble, peer, comm, s_), "ncclSend");
  }
  void recv(int, double* buf, size_t n, int peer) override {
    nccl_check(g_nccl.Recv(buf, n, ncclDouble, peer, comm, s_), "ncclRecv");
  }
  void end() override { nccl_check(g_nccl.GroupEnd(), "ncclGroupEnd"); }
  void allreduce(double* const* bufs, int count, cudaStream_t s) override {
    nccl_check(g_nccl.AllReduce(bufs[0], bufs[0], count, ncclDouble, ncclSum, comm, s), "ncclAllReduce");
  }
};

Transport* transport_local(int world) { return new LocalTransport(world); }
Transport* transport_nccl(const char* lib, const unsigned char* id128, int world, int rank) {
  return new NcclTransport(lib, id128, world, rank);
}
void transport_destroy(Transport* t) { delete t; }
void transport_info(const Transport* t, int* world, int* nlocal, int* first) {
  *world = t->world_;
  *nlocal = t->nlocal_;
  *first = t->first_;
}

// ---------------------------------------------------------------------------------------------
// partition (same arithmetic as paper_1712_08565_b200.dist.SlabPartition)
// ---------------------------------------------------------------------------------------------
struct Part {
  int n_el, p, n3, n2, world;
  int E(int r) const { return int((long long)r * n_el / world); }
  int lo(int r) const { return r == 0 ? 0 : E(r) - 1; }
  int hi(int r) const { return r == world - 1 ? n3 : E(r + 1) - 1; }
  int vhi(int r) const { return std::min(E(r + 1) + p - 1, n3); }
  int ylo(int r) const { return std::max(E(r) - 2, 0); }
  int yhi(int r) const { return std::min(E(r + 1) + p - 1, n3); }
  int row0(int s) const { return int((long long)s * n2 / world); }
  int row1(int s) const { return int((long long)(s + 1) * n2 / world); }
};

__global__ void add_planes_kernel(double* __restrict__ y, const double* __restrict__ b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] += b[i];
}

// per local rank: slab operator, owned slices and the exchange buffers (one persistent workspace)
struct RankWs {
  Stiffness* A = nullptr;
  int rank = 0, lo = 0, hi = 0, vhi = 0, ylo = 0, yhi = 0;
  long long own = 0;  // owned doubles
  double *x = nullptr, *r = nullptr, *z = nullptr, *pw = nullptr, *p = nullptr, *Apw = nullptr, *Ap = nullptr;
  double *s1 = nullptr, *s2 = nullptr, *t1 = nullptr, *t2 = nullptr, *sendb = nullptr, *recvb = nullptr;
  double *hrecv = nullptr, *part = nullptr, *sc = nullptr;  // sc: 0 rz, 1 pAp, 2 rr, 3 rz_new, 4 bb
};

// planes rank `me` receives in the reverse halo (rows of other ranks' output windows it owns)
static long long reverse_halo_planes(const Part& G, int me) {
  long long n = 0;
  for (int q = 0; q < G.world; ++q) {
    const int segs[2][2] = {{G.ylo(q), G.lo(q)}, {G.hi(q), G.yhi(q)}};
    for (auto& sg : segs) {
      const int s0 = std::max(sg[0], G.lo(me)), s1 = std::min(sg[1], G.hi(me));
      if (s0 < s1 && me != q) n += s1 - s0;
    }
  }
  return n;
}

static size_t pad32(size_t n) { return (n + 31) & ~size_t(31); }

struct DistSolve {
  Transport& T;
  FastDiag& P;
  Part G;
  long long plane;
  int n1;
  std::vector<RankWs*> R;
  cudaStream_t s;

  // forward halo: planes [hi_q, vhi_q) of every rank q come from their owners, straight into q's window
  void halo_forward() {
    T.begin(s);
    for (int l = 0; l < (int)R.size(); ++l) {
      RankWs& W = *R[l];
      const int me = W.rank;
      for (int q = 0; q < G.world; ++q) {
        const int a = G.hi(q), b = G.vhi(q);
        for (int o = 0; o < G.world; ++o) {
          const int s0 = std::max(a, G.lo(o)), s1 = std::min(b, G.hi(o));
          if (s0 >= s1 || o == q) continue;
          if (q == me) T.recv(l, W.pw + (s0 - W.lo) * plane, (s1 - s0) * plane, o);
          if (o == me) T.send(l, W.pw + (s0 - W.lo) * plane, (s1 - s0) * plane, q);
        }
      }
    }
    T.end();
  }
  // reverse halo: rows of rank q's output window outside [lo_q, hi_q) go to their owners, are added
  void halo_reverse() {
    T.begin(s);
    for (int l = 0; l < (int)R.size(); ++l) {
      RankWs& W = *R[l];
      const int me = W.rank;
      long long off = 0;
      for (int q = 0; q < G.world; ++q) {
        const int segs[2][2] = {{G.ylo(q), G.lo(q)}, {G.hi(q), G.yhi(q)}};
        for (auto& sg : segs)
          for (int o = 0; o < G.world; ++o) {
            const int s0 = std::max(sg[0], G.lo(o)), s1 = std::min(sg[1], G.hi(o));
            if (s0 >= s1 || o == q) continue;
            if (q == me) T.send(l, W.Apw + (s0 - W.ylo) * plane, (s1 - s0) * plane, o);
            if (o == me) {
              T.recv(l, W.hrecv + off, (s1 - s0) * plane, q);
              off += (s1 - s0) * plane;
            }
          }
      }
    }
    T.end();
    for (int l = 0; l < (int)R.size(); ++l) {
      RankWs& W = *R[l];
      // owned rows out of the output window (contiguous: the window starts lo - ylo rows earlier)
      MFWQ_CUDA(cudaMemcpyAsync(W.Ap, W.Apw + (W.lo - W.ylo) * plane, W.own * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    // the adds, message by message, in the order the receives were posted
    for (int l = 0; l < (int)R.size(); ++l) {
      RankWs& W = *R[l];
      const int me = W.rank;
      long long off = 0;
      for (int q = 0; q < G.world; ++q) {
        const int segs[2][2] = {{G.ylo(q), G.lo(q)}, {G.hi(q), G.yhi(q)}};
        for (auto& sg : segs)
          for (int o = 0; o < G.world; ++o) {
            const int s0 = std::max(sg[0], G.lo(o)), s1 = std::min(sg[1], G.hi(o));
            if (s0 >= s1 || o == q || o != me) continue;
            const long long n = (s1 - s0) * plane;
            add_planes_kernel<<<148, 256, 0, s>>>(W.Ap + (s0 - W.lo) * plane, W.hrecv + off, n); note_launch();
            off += n;
          }
      }
    }
  }
  void matvec() {  // Ap = A p on every rank (p already in the window buffers)
    halo_forward();
    for (RankWs* W : R) W->A->apply(W->pw, W->Apw, s);
    halo_reverse();
  }

  // z = P^-1 r (solvers.py:107-115) across the slabs
  void precond() {
    const int n2 = G.n2;
    for (RankWs* W : R) {
      const int nz = W->hi - W->lo;
      P.apply_dir(0, 0, 0, W->r, W->s1, nz, n2, 0, s);
      P.apply_dir(1, 0, 0, W->s1, W->s2, nz, n2, 0, s);
      // pack: the block for rank q is rows [row0(q), row1(q)) of every owned plane
      long long off = 0;
      for (int q = 0; q < G.world; ++q) {
        const int rq = G.row1(q) - G.row0(q);
        if (rq > 0 && nz > 0)
          MFWQ_CUDA(cudaMemcpy2DAsync(W->sendb + off, (size_t)rq * n1 * 8, W->s2 + (long long)G.row0(q) * n1, plane * 8,
                                      (size_t)rq * n1 * 8, nz, cudaMemcpyDeviceToDevice, s));
        off += (long long)nz * rq * n1;
      }
    }
    T.begin(s);  // all-to-all: rank r's (nz_r, rows_q) block lands at planes lo_r of rank q's (n3, rows_q)
    for (int l = 0; l < (int)R.size(); ++l) {
      RankWs& W = *R[l];
      const int me = W.rank, nz = W.hi - W.lo;
      const int rm = G.row1(me) - G.row0(me);
      long long off = 0;
      for (int q = 0; q < G.world; ++q) {
        const long long n = (long long)nz * (G.row1(q) - G.row0(q)) * n1;
        if (n) {
          if (q == me) MFWQ_CUDA(cudaMemcpyAsync(W.t1 + (long long)W.lo * rm * n1, W.sendb + off, n * 8, cudaMemcpyDeviceToDevice, s));
          else T.send(l, W.sendb + off, n, q);
        }
        off += n;
        const long long m = (long long)(G.hi(q) - G.lo(q)) * rm * n1;
        if (m && q != me) T.recv(l, W.t1 + (long long)G.lo(q) * rm * n1, m, q);
      }
    }
    T.end();
    for (RankWs* W : R) {
      const int rm = G.row1(W->rank) - G.row0(W->rank);
      if (rm <= 0) continue;
      P.apply_dir(2, 0, 1, W->t1, W->t2, G.n3, rm, G.row0(W->rank), s);
      P.apply_dir(2, 1, 0, W->t2, W->t1, G.n3, rm, G.row0(W->rank), s);
    }
    T.begin(s);  // and back: rank q's planes [lo_r, hi_r) of its rows go to rank r
    for (int l = 0; l < (int)R.size(); ++l) {
      RankWs& W = *R[l];
      const int me = W.rank, nz = W.hi - W.lo;
      const int rm = G.row1(me) - G.row0(me);
      long long off = 0;
      for (int q = 0; q < G.world; ++q) {
        const long long n = (long long)(G.hi(q) - G.lo(q)) * rm * n1;  // my rows of q's planes
        if (n && q != me) T.send(l, W.t1 + (long long)G.lo(q) * rm * n1, n, q);
        const long long m = (long long)nz * (G.row1(q) - G.row0(q)) * n1;
        if (m) {
          if (q == me) MFWQ_CUDA(cudaMemcpyAsync(W.recvb + off, W.t1 + (long long)W.lo * rm * n1, m * 8, cudaMemcpyDeviceToDevice, s));
          else T.recv(l, W.recvb + off, m, q);
        }
        off += m;
      }
    }
    T.end();
    for (RankWs* W : R) {
      const int nz = W->hi - W->lo;
      long long off = 0;
      for (int q = 0; q < G.world; ++q) {  // unpack rank q's rows into (nz, n2, n1)
        const int rq = G.row1(q) - G.row0(q);
        if (rq > 0 && nz > 0)
          MFWQ_CUDA(cudaMemcpy2DAsync(W->s1 + (long long)G.row0(q) * n1, plane * 8, W->recvb + off, (size_t)rq * n1 * 8,
                                      (size_t)rq * n1 * 8, nz, cudaMemcpyDeviceToDevice, s));
        off += (long long)nz * rq * n1;
      }
      P.apply_dir(1, 1, 0, W->s1, W->s2, nz, n2, 0, s);
      P.apply_dir(0, 1, 0, W->s2, W->z, nz, n2, 0, s);
    }
  }

  void allreduce(int slot, int count = 1) {
    double* bufs[MAX_LOCAL];
    for (size_t l = 0; l < R.size(); ++l) bufs[l] = R[l]->sc + slot;
    T.allreduce(bufs, count, s);
  }
};

// The comm variant of pcg_solve: every local rank's owned slice of b in, x out.
void dist_pcg_solve(Transport& T, Stiffness* const* slabs, FastDiag* P, const double* const* b, double* const* x,
                    double tol, int maxit, std::vector<double>& hist, KrylovOut& out, cudaStream_t s) {
  hist.clear();
  out = KrylovOut{};
  if (!P) throw ValueErr("the distributed solver needs the FD preconditioner (identity: use P = NULL single-GPU)");
  const int nl = T.nlocal_;
  Stiffness& A0 = *slabs[0];
  Part G{A0.dir[2].n_el, A0.dir[2].p, A0.dir[2].n, A0.dir[1].n, T.world_};
  const long long plane = (long long)A0.dir[0].n * A0.dir[1].n;
  if (P->n[0] != A0.dir[0].n || P->n[1] != A0.dir[1].n || P->n[2] != A0.dir[2].n)
    throw ValueErr("preconditioner and operator sizes differ");
  for (int r = 0; r < G.world; ++r)
    if (G.hi(r) <= G.lo(r) || G.E(r + 1) <= G.E(r))
      throw ValueErr("a rank owns no DoF plane: too many ranks for the mesh");
  DistSolve D{T, *P, G, plane, A0.dir[0].n, {}, s};
  const int parts = vec_partials();
  for (int l = 0; l < nl; ++l) {
    Stiffness& A = *slabs[l];
    const int rank = T.first_ + l;
    if (A.e_lo != G.E(rank) || A.e_hi != G.E(rank + 1))
      throw ValueErr("slab handle " + std::to_string(l) + " does not hold rank " + std::to_string(rank) +
                     "'s z-elements [E_r, E_r+1), E_r = r n_el / world");
    if (A.v_lo != G.lo(rank) || A.v_hi != G.vhi(rank) || A.y_lo != G.ylo(rank) || A.y_hi != G.yhi(rank))
      throw ValueErr("slab windows disagree with the partition");
    auto* W = new RankWs();  // owned by A's dist workspace slot below
    W->A = &A;
    W->rank = rank;
    W->lo = G.lo(rank);
    W->hi = G.hi(rank);
    W->vhi = G.vhi(rank);
    W->ylo = G.ylo(rank);
    W->yhi = G.yhi(rank);
    W->own = (W->hi - W->lo) * plane;
    const int rm = G.row1(rank) - G.row0(rank);
    const size_t own = pad32(W->own), win = pad32((W->vhi - W->lo) * plane), ywin = pad32((W->yhi - W->ylo) * plane);
    const size_t tsz = pad32((size_t)G.n3 * rm * A.dir[0].n), halo = pad32(reverse_halo_planes(G, rank) * plane);
    const size_t need = 5 * own + win + ywin + 2 * tsz + 2 * own + halo + pad32(parts) + 32;
    A.dist_ws.alloc_at_least(need);
    double* q = A.dist_ws.ptr;
    auto take = [&](size_t n) { double* o = q; q += n; return o; };
    W->x = take(own);
    W->r = take(own);
    W->z = take(own);
    W->Ap = take(own);
    W->s1 = take(own);
    W->pw = take(win);
    W->p = W->pw;  // the owned slice of p starts the window (v_lo == lo)
    W->Apw = take(ywin);
    W->t1 = take(tsz);
    W->t2 = take(tsz);
    W->s2 = take(own);
    W->sendb = take(own);
    W->hrecv = take(halo);
    W->part = take(pad32(parts));
    W->sc = take(32);
    W->recvb = W->Ap;  // the all-to-all return lands in Ap's space (free during the preconditioner)
    D.R.push_back(W);
  }
  struct Cleanup {
    std::vector<RankWs*>& R;
    ~Cleanup() {
      for (RankWs* w : R) delete w;
    }
  } cleanup{D.R};
  // ||b|| (solvers.py:141-143)
  for (int l = 0; l < nl; ++l) {
    RankWs& W = *D.R[l];
    MFWQ_CUDA(cudaMemsetAsync(W.x, 0, W.own * sizeof(double), s));
    MFWQ_CUDA(cudaMemcpyAsync(W.r, b[l], W.own * sizeof(double), cudaMemcpyDeviceToDevice, s));
    vec_dot_to(W.r, W.r, W.own, W.part, W.sc + 4, s);
  }
  D.allreduce(4);
  double hsc[3];
  MFWQ_CUDA(cudaMemcpyAsync(hsc, D.R[0]->sc + 4, sizeof(double), cudaMemcpyDeviceToHost, s));
  MFWQ_CUDA(cudaStreamSynchronize(s));
  const double bnorm = std::sqrt(hsc[0]);
  auto copy_out = [&]() {
    for (int l = 0; l < nl; ++l)
      MFWQ_CUDA(cudaMemcpyAsync(x[l], D.R[l]->x, D.R[l]->own * sizeof(double), cudaMemcpyDeviceToDevice, s));
    MFWQ_CUDA(cudaStreamSynchronize(s));
  };
  if (bnorm == 0.0) {
    hist.push_back(0.0);
    out.converged = 1;
    copy_out();
    return;
  }
  D.precond();  // z = P r, p = z, rz = r.z
  out.precs = 1;
  for (RankWs* W : D.R) {
    MFWQ_CUDA(cudaMemcpyAsync(W->p, W->z, W->own * sizeof(double), cudaMemcpyDeviceToDevice, s));
    vec_dot_to(W->r, W->z, W->own, W->part, W->sc + 0, s);
  }
  D.allreduce(0);
  hist.push_back(1.0);
  for (int k = 1; k <= maxit; ++k) {
    D.matvec();
    out.matvecs++;
    for (RankWs* W : D.R) vec_dot_to(W->p, W->Ap, W->own, W->part, W->sc + 1, s);
    D.allreduce(1);
    for (RankWs* W : D.R) vec_update_xr(W->x, W->r, W->p, W->Ap, W->own, W->sc + 0, W->sc + 1, W->part, W->sc + 2, s);
    D.allreduce(2);
    MFWQ_CUDA(cudaMemcpyAsync(hsc, D.R[0]->sc + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    MFWQ_CUDA(cudaStreamSynchronize(s));  // the one host read of the iteration
    if (hsc[0] <= 0) {  // solvers.py:156-160
      char m[128];
      snprintf(m, sizeof m, "nonpositive curvature p.Ap = %.3e at iteration %d", hsc[0], k);
      throw IndefiniteErr(m);
    }
    const double rel = std::sqrt(hsc[1]) / bnorm;
    hist.push_back(rel);
    if (rel <= tol) {
      out.iterations = k;
      out.converged = 1;
      copy_out();
      return;
    }
    D.precond();
    out.precs++;
    for (RankWs* W : D.R) vec_dot_to(W->r, W->z, W->own, W->part, W->sc + 3, s);
    D.allreduce(3);
    for (RankWs* W : D.R) vec_update_p(W->p, W->z, W->own, W->sc + 3, W->sc + 0, s);
  }
  out.iterations = maxit;
  out.converged = 0;
  copy_out();
}

}  // namespace mfwq
