// extern "C" boundary of libmfwq.so (declared in include/mfwq.h).
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mfwq.h"
#include "ops.h"

using namespace mfwq;

struct mfwq_rule1d_s { Rule1D r; int nfun; };
// host-buffer pipeline state (mfwq_stiffness_apply_host): two device staging pairs, one H2D and one
// D2H stream, and the events that order staging reuse; created on first use
struct HostPipe {
  bool ready = false;
  int i = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  DevBuf<double> x[2], y[2];
  cudaEvent_t landed[2] = {}, freed[2] = {}, read[2] = {};
  bool freed_set[2] = {false, false}, read_set[2] = {false, false};
  ~HostPipe() {
    if (!ready) return;
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(landed[k]);
      cudaEventDestroy(freed[k]);
      cudaEventDestroy(read[k]);
    }
    cudaStreamDestroy(h2d);
    cudaStreamDestroy(d2h);
  }
};
// Pageable host memory (a numpy array): the driver stages such copies through its own pinned
// buffer on one thread (~12 GB/s).  Here the host side of each chunk is copied by a small pool of
// threads into a pinned slot while the previous chunk's DMA runs.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  // dst <- src (bytes), split across the pool's threads and the caller
  void copy(void* dst, const void* src, size_t bytes) {
    const int parts = int(workers_.size()) + 1;
    if (bytes < (size_t(1) << 20)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const size_t per = (bytes / parts + 63) & ~size_t(63);
    size_t mine = 0;  // tasks of this call (other host threads may be copying concurrently)
    {
      std::unique_lock<std::mutex> lk(m_);
      for (int k = 1; k < parts; ++k) {
        const size_t o = per * k;
        if (o < bytes) {
          tasks_.push_back({static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                            std::min(per, bytes - o), &mine});
          ++mine;
        }
      }
    }
    cv_.notify_all();
    std::memcpy(dst, src, std::min(per, bytes));
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return mine == 0; });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  struct Task { char* dst; const char* src; size_t n; size_t* left; };  // left: the caller's count
  CopyPool() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    const int n = int(std::min(7u, hw / 2));  // + the caller
    for (int k = 0; k < n; ++k) workers_.emplace_back([this] { run(); });
  }
  void run() {
    for (;;) {
      Task t;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || !tasks_.empty(); });
        if (stop_ && tasks_.empty()) return;
        t = tasks_.back();
        tasks_.pop_back();
      }
      std::memcpy(t.dst, t.src, t.n);
      std::lock_guard<std::mutex> lk(m_);
      if (--*t.left == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::vector<Task> tasks_;
  bool stop_ = false;
  std::mutex m_;
  std::condition_variable cv_, done_;
};

// synchronous apply on pageable host buffers: chunked H2D through two pinned slots, the kernel,
// chunked D2H through two pinned slots; host copies of chunk k overlap the DMA of chunk k -+ 1
struct PageablePipe {
  static constexpr size_t CHUNK = size_t(4) << 20;  // bytes per slot
  bool ready = false;
  cudaStream_t cs = nullptr;  // copy stream
  double* pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {}, kdone = nullptr;
  DevBuf<double> x, y;
  ~PageablePipe() {
    if (!ready) return;
    for (int k = 0; k < 2; ++k) {
      cudaFreeHost(pin[k]);
      cudaEventDestroy(ev[k]);
    }
    cudaEventDestroy(kdone);
    cudaStreamDestroy(cs);
  }
  void init() {
    if (ready) return;
    MFWQ_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      MFWQ_CUDA(cudaMallocHost(&pin[k], CHUNK));
      MFWQ_CUDA(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    }
    MFWQ_CUDA(cudaEventCreateWithFlags(&kdone, cudaEventDisableTiming));
    ready = true;
  }
  void run(Stiffness& S, const double* xh, double* yh, cudaStream_t s) {
    init();
    const size_t nin = S.in_elems(), nout = S.out_elems();
    x.alloc_at_least(nin);
    y.alloc_at_least(nout);
    CopyPool& pool = CopyPool::get();
    const size_t cd = CHUNK / sizeof(double);
    bool used[2] = {false, false};
    for (size_t off = 0, k = 0; off < nin; off += cd, ++k) {  // H2D
      const int sl = int(k & 1);
      const size_t n = std::min(cd, nin - off);
      if (used[sl]) MFWQ_CUDA(cudaEventSynchronize(ev[sl]));  // its previous DMA has read it
      pool.copy(pin[sl], xh + off, n * sizeof(double));
      MFWQ_CUDA(cudaMemcpyAsync(x.ptr + off, pin[sl], n * sizeof(double), cudaMemcpyHostToDevice, cs));
      MFWQ_CUDA(cudaEventRecord(ev[sl], cs));
      used[sl] = true;
    }
    MFWQ_CUDA(cudaEventRecord(kdone, cs));
    MFWQ_CUDA(cudaStreamWaitEvent(s, kdone, 0));
    S.apply(x.ptr, y.ptr, s);
    MFWQ_CUDA(cudaEventRecord(kdone, s));
    MFWQ_CUDA(cudaStreamWaitEvent(cs, kdone, 0));
    const size_t nch = (nout + cd - 1) / cd;
    auto issue = [&](size_t k) {
      const int sl = int(k & 1);
      const size_t off = k * cd, n = std::min(cd, nout - off);
      MFWQ_CUDA(cudaMemcpyAsync(pin[sl], y.ptr + off, n * sizeof(double), cudaMemcpyDeviceToHost, cs));
      MFWQ_CUDA(cudaEventRecord(ev[sl], cs));
    };
    for (size_t k = 0; k < std::min<size_t>(2, nch); ++k) issue(k);
    for (size_t k = 0; k < nch; ++k) {  // D2H
      const int sl = int(k & 1);
      const size_t off = k * cd, n = std::min(cd, nout - off);
      MFWQ_CUDA(cudaEventSynchronize(ev[sl]));
      pool.copy(yh + off, pin[sl], n * sizeof(double));
      if (k + 2 < nch) issue(k + 2);
    }
  }
};

struct mfwq_stiffness_s {
  Stiffness op;
  HostPipe pipe;
  PageablePipe pageable;
};
struct mfwq_fd_s { FastDiag fd; };
struct mfwq_quad_s { Quadrature q; };

static thread_local std::string g_err;
long long mfwq::g_launches = 0;

template <class F>
static int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return MFWQ_OK;
  } catch (const ValueErr& e) {
    g_err = e.what();
    return MFWQ_E_VALUE;
  } catch (const WQErr& e) {
    g_err = e.what();
    return MFWQ_E_WQ;
  } catch (const DegenerateErr& e) {
    g_err = e.what();
    return MFWQ_E_DEGENERATE;
  } catch (const EigenErr& e) {
    g_err = e.what();
    return MFWQ_E_EIGEN;
  } catch (const IndefiniteErr& e) {
    g_err = e.what();
    return MFWQ_E_INDEFINITE;
  } catch (const CudaErr& e) {
    g_err = e.what();
    return MFWQ_E_CUDA;
  } catch (const NotImplErr& e) {
    g_err = e.what();
    return MFWQ_E_NOTIMPL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MFWQ_E_INTERNAL;
  }
}

extern "C" {

const char* mfwq_last_error(void) { return g_err.c_str(); }
int mfwq_version(void) { return 1; }
long long mfwq_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int mfwq_set_lapack(const char* lib_path, const char* symbol) {
  return guard([&] {
    if (!lib_path || !symbol) throw ValueErr("mfwq_set_lapack: library path and symbol required");
    void* h = dlopen(lib_path, RTLD_NOW | RTLD_LOCAL);  // kept open for the life of the process
    if (!h) throw ValueErr(std::string("cannot load LAPACK library: ") + dlerror());
    void* fn = dlsym(h, symbol);
    if (!fn) throw ValueErr(std::string("LAPACK library has no symbol ") + symbol);
    // the companion dsyevd (np.linalg.eigvalsh, behind numpy's Gauss-Legendre rule): same naming
    std::string ev(symbol);
    const size_t at = ev.find("gelsd");
    if (at == std::string::npos) throw ValueErr("symbol must name a dgelsd (e.g. scipy_dgelsd_64_)");
    ev.replace(at, 5, "syevd");
    void* fe = dlsym(h, ev.c_str());
    if (!fe) throw ValueErr("LAPACK library has no symbol " + ev);
    set_lapack(reinterpret_cast<dgelsd64_t>(fn), reinterpret_cast<dsyevd64_t>(fe));
  });
}

int mfwq_lapack_active(void) { return have_dgelsd() ? 1 : 0; }

int mfwq_rule1d_build(int p, int nknots, const double* knots, mfwq_rule1d_t* out) {
  return guard([&] {
    Knots kv(p, knots, nknots);
    auto* h = new mfwq_rule1d_s{build_rule(kv), kv.nfun()};
    *out = h;
  });
}

int mfwq_rule1d_sizes(mfwq_rule1d_t r, int* npts, int* nfun, int* extra, int* nnz6) {
  return guard([&] {
    *npts = int(r->r.pts.size());
    *nfun = r->nfun;
    *extra = r->r.extra;
    for (int k = 0; k < 4; ++k) nnz6[k] = int(r->r.W[k].data.size());
    for (int k = 0; k < 2; ++k) nnz6[4 + k] = int(r->r.B[k].data.size());
  });
}

int mfwq_rule1d_export(mfwq_rule1d_t r, double* pts, int* const* indptr6, int* const* indices6, double* const* data6) {
  return guard([&] {
    std::memcpy(pts, r->r.pts.data(), r->r.pts.size() * sizeof(double));
    for (int k = 0; k < 6; ++k) {
      const Csr& c = k < 4 ? r->r.W[k] : r->r.B[k - 4];
      std::memcpy(indptr6[k], c.indptr.data(), c.indptr.size() * sizeof(int));
      std::memcpy(indices6[k], c.indices.data(), c.indices.size() * sizeof(int));
      std::memcpy(data6[k], c.data.data(), c.data.size() * sizeof(double));
    }
  });
}

void mfwq_rule1d_destroy(mfwq_rule1d_t r) { delete r; }

int mfwq_univariate_km(int p, int nknots, const double* knots, double* K, double* M) {
  return guard([&] {
    Knots kv(p, knots, nknots);
    std::vector<double> k, m;
    univariate_km(kv, k, m);
    std::memcpy(K, k.data(), k.size() * sizeof(double));
    std::memcpy(M, m.data(), m.size() * sizeof(double));
  });
}

int mfwq_stiffness_create(const mfwq_stiffness_desc* d, mfwq_stiffness_t* out) {
  return guard([&] {
    auto* h = new mfwq_stiffness_s();
    try {
      h->op.init(d->p, d->nknots, d->knots, d->npts, d->pts, d->indptr, d->indices, d->data);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int mfwq_stiffness_set_geometry(mfwq_stiffness_t h, int kind, const double* affine9, const double* K9,
                                const double* J_dev, const double* Kfield_dev, void* stream) {
  return guard([&] {
    if (kind < 0 || kind > 3) throw ValueErr("unknown geometry kind");
    if (kind == MFWQ_GEOM_JACOBIAN && !J_dev) throw ValueErr("JACOBIAN geometry needs J_dev");
    h->op.set_geometry(kind, affine9, K9, J_dev, Kfield_dev, (cudaStream_t)stream);
  });
}

int mfwq_stiffness_set_on_the_fly(mfwq_stiffness_t h, int kind, const double* affine9, const double* K9,
                                  void* stream) {
  return guard([&] {
    if (kind < 0 || kind > 3) throw ValueErr("unknown geometry kind");
    h->op.set_on_the_fly(kind, affine9, K9, (cudaStream_t)stream);
  });
}

int mfwq_mass_set(mfwq_stiffness_t h, int kind, const double* affine9, const double* J_dev, double alpha,
                  const double* alpha_field_dev, int on_the_fly, void* stream) {
  return guard([&] {
    if (kind < 0 || kind > 3) throw ValueErr("unknown geometry kind");
    if (kind == MFWQ_GEOM_JACOBIAN && !J_dev) throw ValueErr("JACOBIAN geometry needs J_dev");
    h->op.set_mass(kind, affine9, J_dev, alpha, alpha_field_dev, on_the_fly, (cudaStream_t)stream);
  });
}

int mfwq_mass_apply(mfwq_stiffness_t h, const double* x, double* y, void* stream) {
  return guard([&] { h->op.apply_mass(x, y, (cudaStream_t)stream); });
}

int mfwq_mass_flops(mfwq_stiffness_t h, long long* flops) {
  return guard([&] { *flops = h->op.mass_flops(); });
}

int mfwq_stiffness_set_coeffs(mfwq_stiffness_t h, const double* const* grids, void* stream) {
  return guard([&] { h->op.set_coeffs(grids, (cudaStream_t)stream); });
}

int mfwq_stiffness_get_coeff(mfwq_stiffness_t h, int key, double* out, void* stream) {
  return guard([&] {
    if (key < 0 || key > 5) throw ValueErr("coefficient key out of range");
    if (!h->op.coeffs_ready) throw ValueErr("coefficient grids not set");
    h->op.get_coeffs(key, out, (cudaStream_t)stream);
  });
}

int mfwq_stiffness_sizes(mfwq_stiffness_t h, int* n3, int* m3, long long* N, long long* Nq) {
  return guard([&] {
    for (int l = 0; l < 3; ++l) {
      n3[l] = h->op.dir[l].n;
      m3[l] = h->op.dir[l].m;
    }
    *N = h->op.N;
    *Nq = h->op.Nq;
  });
}

int mfwq_stiffness_apply(mfwq_stiffness_t h, const double* x, double* y, void* stream) {
  return guard([&] {
    // the output is zeroed before the kernel reads x: an overlapping (in-place) call is rejected
    const double *x1 = x + h->op.in_elems(), *y1 = y + h->op.out_elems();
    if (x < y1 && y < x1) throw ValueErr("x and y must not overlap (y is overwritten before x is read)");
    h->op.apply(x, y, (cudaStream_t)stream);
  });
}

int mfwq_stiffness_apply_host(mfwq_stiffness_t h, const double* x_host, double* y_host, void* stream) {
  return guard([&] {
    HostPipe& P = h->pipe;
    Stiffness& S = h->op;
    const size_t nin = S.in_elems(), nout = S.out_elems();
    if (!P.ready) {
      MFWQ_CUDA(cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking));
      MFWQ_CUDA(cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking));
      for (int k = 0; k < 2; ++k) {
        P.x[k].alloc(nin);
        P.y[k].alloc(nout);
        MFWQ_CUDA(cudaEventCreateWithFlags(&P.landed[k], cudaEventDisableTiming));
        MFWQ_CUDA(cudaEventCreateWithFlags(&P.freed[k], cudaEventDisableTiming));
        MFWQ_CUDA(cudaEventCreateWithFlags(&P.read[k], cudaEventDisableTiming));
      }
      P.ready = true;
    }
    if (P.x[0].n < nin || P.y[0].n < nout) {
      // the slab window grew since the staging pairs were sized (mfwq_stiffness_set_slab): drain the
      // pipe, then resize both pairs
      for (int k = 0; k < 2; ++k) {
        if (P.read_set[k]) MFWQ_CUDA(cudaEventSynchronize(P.read[k]));
        if (P.freed_set[k]) MFWQ_CUDA(cudaEventSynchronize(P.freed[k]));
        P.x[k].alloc(nin);
        P.y[k].alloc(nout);
      }
    }
    const cudaStream_t s = (cudaStream_t)stream;
    const int i = P.i;
    P.i ^= 1;
    // H2D into staging pair i once the kernel that last read it is done
    if (P.freed_set[i]) MFWQ_CUDA(cudaStreamWaitEvent(P.h2d, P.freed[i], 0));
    MFWQ_CUDA(cudaMemcpyAsync(P.x[i].ptr, x_host, nin * sizeof(double), cudaMemcpyHostToDevice, P.h2d));
    MFWQ_CUDA(cudaEventRecord(P.landed[i], P.h2d));
    // the kernel on the caller's stream: after its input landed and the D2H that last read y[i]
    MFWQ_CUDA(cudaStreamWaitEvent(s, P.landed[i], 0));
    if (P.read_set[i]) MFWQ_CUDA(cudaStreamWaitEvent(s, P.read[i], 0));
    S.apply(P.x[i].ptr, P.y[i].ptr, s);
    MFWQ_CUDA(cudaEventRecord(P.freed[i], s));
    P.freed_set[i] = true;
    // D2H of the result on the D2H stream
    MFWQ_CUDA(cudaStreamWaitEvent(P.d2h, P.freed[i], 0));
    MFWQ_CUDA(cudaMemcpyAsync(y_host, P.y[i].ptr, nout * sizeof(double), cudaMemcpyDeviceToHost, P.d2h));
    MFWQ_CUDA(cudaEventRecord(P.read[i], P.d2h));
    P.read_set[i] = true;
  });
}

int mfwq_stiffness_apply_pageable(mfwq_stiffness_t h, const double* x_host, double* y_host, void* stream) {
  return guard([&] {
    if (x_host == y_host) throw ValueErr("x and y must not be the same buffer");
    h->pageable.run(h->op, x_host, y_host, (cudaStream_t)stream);
  });
}

int mfwq_stiffness_host_join(mfwq_stiffness_t h, void* stream) {
  return guard([&] {
    HostPipe& P = h->pipe;
    for (int k = 0; k < 2; ++k)
      if (P.read_set[k]) MFWQ_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, P.read[k], 0));
  });
}

int mfwq_stiffness_set_slab(mfwq_stiffness_t h, int e_lo, int e_hi) {
  return guard([&] { h->op.set_slab(e_lo, e_hi); });
}

int mfwq_stiffness_slab_info(mfwq_stiffness_t h, int* info6) {
  return guard([&] {
    const Stiffness& S = h->op;
    const int v[6] = {S.e_lo, S.e_hi, S.v_lo, S.v_hi, S.y_lo, S.y_hi};
    std::memcpy(info6, v, sizeof v);
  });
}

int mfwq_stiffness_set_path(mfwq_stiffness_t h, int path) {
  return guard([&] {
    if (path < 0 || path > 2) throw ValueErr("path must be 0..2");
    h->op.path = path;
    h->op.pcg_graphs.reset();
  });
}

int mfwq_stiffness_set_deterministic(mfwq_stiffness_t h, int on) {
  return guard([&] {
    h->op.deterministic = on != 0;
    h->op.pcg_graphs.reset();  // captured PCG iterations hold the other accumulation scheme
  });
}

int mfwq_stiffness_info(mfwq_stiffness_t h, int* term_mask, int* fused_ok, int* kernel_terms) {
  return guard([&] {
    const int tm = h->op.term_mask();
    *term_mask = tm;
    *fused_ok = fused2_accepts(h->op) ? 1 : 0;
    *kernel_terms = (tm & ~0x111) == 0 ? 3 : ((tm & ~0x11B) == 0 ? 5 : 9);
  });
}

int mfwq_stiffness_flops(mfwq_stiffness_t h, long long* flops) {
  return guard([&] { *flops = h->op.flops; });
}

int mfwq_stiffness_flops_active(mfwq_stiffness_t h, long long* flops) {
  return guard([&] { *flops = h->op.flops_for(h->op.term_mask()); });
}

void mfwq_stiffness_destroy(mfwq_stiffness_t h) { delete h; }

int mfwq_fd_create(const int* n3, const double* const* K3, const double* const* M3, double sigma, mfwq_fd_t* out) {
  return guard([&] {
    auto* h = new mfwq_fd_s();
    try {
      h->fd.init(n3, K3, M3, sigma);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int mfwq_fd_apply(mfwq_fd_t h, const double* r, double* z, void* stream) {
  return guard([&] { h->fd.apply(r, z, (cudaStream_t)stream); });
}

int mfwq_fd_apply_dir(mfwq_fd_t h, int dir, int inverse, int scale, const double* x, double* y, int nz, int ny,
                      int row_lo, void* stream) {
  return guard([&] { h->fd.apply_dir(dir, inverse, scale, x, y, nz, ny, row_lo, (cudaStream_t)stream); });
}

int mfwq_fd_eigen(mfwq_fd_t h, int dir, double* lam, double* U) {
  return guard([&] {
    if (dir < 0 || dir > 2) throw ValueErr("direction out of range");
    std::memcpy(lam, h->fd.lam_h[dir].data(), h->fd.lam_h[dir].size() * sizeof(double));
    std::memcpy(U, h->fd.U_h[dir].data(), h->fd.U_h[dir].size() * sizeof(double));
  });
}

void mfwq_fd_destroy(mfwq_fd_t h) { delete h; }

int mfwq_pcg_solve(mfwq_stiffness_t A, mfwq_fd_t P, const double* b, double* x, double tol, int maxit,
                   double* residuals, mfwq_krylov_report* rep, void* stream) {
  return guard([&] {
    if (A->op.is_slab()) throw ValueErr("mfwq_pcg_solve takes a whole-domain operator (slab handles: mfwq_pcg_solve_comm)");
    std::vector<double> hist;
    KrylovOut o;
    pcg_solve(A->op, P ? &P->fd : nullptr, b, x, A->op.N, tol, maxit, hist, o, (cudaStream_t)stream);
    rep->iterations = o.iterations;
    rep->converged = o.converged;
    rep->matvecs = o.matvecs;
    rep->precond_applies = o.precs;
    rep->n_residuals = int(hist.size());
    std::memcpy(residuals, hist.data(), hist.size() * sizeof(double));
  });
}

struct mfwq_comm_s {
  Transport* t = nullptr;
  ~mfwq_comm_s() { transport_destroy(t); }
};

int mfwq_nccl_unique_id(const char* nccl_lib, unsigned char* id128) {
  return guard([&] { nccl_unique_id(nccl_lib, id128); });
}

int mfwq_comm_create_nccl(const char* nccl_lib, const unsigned char* id128, int world, int rank, mfwq_comm_t* out) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) throw ValueErr("rank out of range");
    auto* c = new mfwq_comm_s();
    c->t = transport_nccl(nccl_lib, id128, world, rank);
    *out = c;
  });
}

int mfwq_comm_create_local(int world, mfwq_comm_t* out) {
  return guard([&] {
    auto* c = new mfwq_comm_s();
    c->t = transport_local(world);
    *out = c;
  });
}

int mfwq_comm_info(mfwq_comm_t c, int* world, int* nlocal, int* first_rank) {
  return guard([&] { transport_info(c->t, world, nlocal, first_rank); });
}

void mfwq_comm_destroy(mfwq_comm_t c) { delete c; }

int mfwq_pcg_solve_comm(mfwq_comm_t comm, const mfwq_stiffness_t* slabs, mfwq_fd_t P, const double* const* b,
                        double* const* x, double tol, int maxit, double* residuals, mfwq_krylov_report* rep,
                        void* stream) {
  return guard([&] {
    int world, nl, first;
    transport_info(comm->t, &world, &nl, &first);
    std::vector<Stiffness*> ops(nl);
    for (int l = 0; l < nl; ++l) ops[l] = &slabs[l]->op;
    std::vector<double> hist;
    KrylovOut o;
    dist_pcg_solve(*comm->t, ops.data(), P ? &P->fd : nullptr, b, x, tol, maxit, hist, o, (cudaStream_t)stream);
    rep->iterations = o.iterations;
    rep->converged = o.converged;
    rep->matvecs = o.matvecs;
    rep->precond_applies = o.precs;
    rep->n_residuals = int(hist.size());
    std::memcpy(residuals, hist.data(), hist.size() * sizeof(double));
  });
}

int mfwq_kron_apply(int d, const int* rows, const int* cols, const double* const* A, const double* x, double* y,
                    int accumulate, void* stream) {
  return guard([&] { kron_apply_dense(d, rows, cols, A, x, y, accumulate, (cudaStream_t)stream); });
}

int mfwq_dot(const double* a, const double* b, long long n, double* out, void* stream) {
  return guard([&] { *out = dot_fast(a, b, n, (cudaStream_t)stream); });
}

int mfwq_dot2(const double* a, const double* b, long long n, double* aa_ab, void* stream) {
  return guard([&] { dot2(a, b, n, aa_ab, (cudaStream_t)stream); });
}

int mfwq_axpy(double* y, const double* x, long long n, double a, void* stream) {
  return guard([&] { axpy(y, x, n, a, (cudaStream_t)stream); });
}

int mfwq_bicg_p(double* p, const double* r, const double* v, long long n, double beta, double omega, void* stream) {
  return guard([&] { bicg_p(p, r, v, n, beta, omega, (cudaStream_t)stream); });
}

int mfwq_bicg_s(double* s, const double* r, const double* v, long long n, double alpha, double* ss, void* stream) {
  return guard([&] { *ss = bicg_s(s, r, v, n, alpha, (cudaStream_t)stream); });
}

int mfwq_bicg_xr(double* x, double* r, const double* phat, const double* shat, const double* s, const double* t,
                 long long n, double alpha, double omega, double* rr, void* stream) {
  return guard([&] { *rr = bicg_xr(x, r, phat, shat, s, t, n, alpha, omega, (cudaStream_t)stream); });
}


int mfwq_quad_create(const int* p3, const int* nknots3, const double* const* knots3, int gpts, mfwq_quad_t* out) {
  return guard([&] { *out = new mfwq_quad_s{Quadrature(p3, nknots3, knots3, gpts)}; });
}

int mfwq_quad_sizes(mfwq_quad_t h, int* ng3, long long* npts, long long* ndofs) {
  return guard([&] {
    for (int l = 0; l < 3; ++l) ng3[l] = h->q.dir[l].n_el * h->q.g;
    *npts = h->q.n_points();
    *ndofs = h->q.n_dofs();
  });
}

int mfwq_quad_points(mfwq_quad_t h, int dir, double* x, double* w) {
  return guard([&] {
    if (dir < 0 || dir > 2) throw ValueErr("direction must be 0, 1 or 2");
    std::memcpy(x, h->q.dir[dir].x.data(), h->q.dir[dir].x.size() * sizeof(double));
    std::memcpy(w, h->q.dir[dir].w.data(), h->q.dir[dir].w.size() * sizeof(double));
  });
}

int mfwq_quad_rhs(mfwq_quad_t h, int kind, const double* affine12, const double* J_dev, int case_id,
                  const double* fvals_dev, double* rhs_dev, void* stream) {
  return guard([&] { h->q.rhs(kind, affine12, J_dev, case_id, fvals_dev, rhs_dev, (cudaStream_t)stream); });
}

int mfwq_quad_errors(mfwq_quad_t h, int kind, const double* affine12, const double* J_dev, int case_id,
                     const double* uvals_dev, const double* gvals_dev, const double* u_dev, int with_grad,
                     double* err_ref, void* stream) {
  return guard([&] {
    h->q.errors(kind, affine12, J_dev, case_id, uvals_dev, gvals_dev, u_dev, with_grad, err_ref, (cudaStream_t)stream);
  });
}

void mfwq_quad_destroy(mfwq_quad_t h) { delete h; }
}  // extern "C"
