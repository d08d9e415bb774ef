// Shared device-side definitions for the MF-WQ B200 library.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "rule1d.h"

namespace mfwq {

#define MFWQ_CUDA(call)                                                                 \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::mfwq::CudaErr(std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

// Owned device allocation (RAII).
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) MFWQ_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
  }
  void alloc_at_least(size_t count) {
    if (count > n) alloc(count);
  }
  void upload(const T* host, size_t count, cudaStream_t s = 0) {
    if (count > n) alloc(count);
    if (count) MFWQ_CUDA(cudaMemcpyAsync(ptr, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Banded 1D factor on the device: row r holds `width` consecutive entries
// starting at column start[r] (zero padded).  Built from the reference's CSR
// factors after the Dirichlet interior restriction of operators.py:146-160.
struct BandView {
  int rows, cols, width;
  const int* start;
  const double* vals;
};

struct BandHost {
  int rows = 0, cols = 0, width = 0;
  std::vector<int> start;
  std::vector<double> vals;
};

struct Band {
  BandHost h;
  DevBuf<int> start;
  DevBuf<double> vals;
  BandView view() const { return BandView{h.rows, h.cols, h.width, start.ptr, vals.ptr}; }
  void upload() {
    start.upload(h.start.data(), h.start.size());
    vals.upload(h.vals.data(), h.vals.size());
  }
};

// CSR (rows x cols) restricted to row range [r0, r1) and column range [c0, c1)
// (shifted to 0) -> band.
BandHost csr_to_band(const Csr& A, int r0, int r1, int c0, int c1);

inline int ceil_div(long long a, long long b) { return int((a + b - 1) / b); }

}  // namespace mfwq

namespace mfwq {
// Count of this library's kernel launches (reported by bench.py as gpu_launches).
extern long long g_launches;
inline void note_launch() { __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED); }
}  // namespace mfwq
