// Probe: can DFMA (fp64 pipe) and DMMA (tensor pipe) run concurrently on B200?
// Runs DFMA-only, DMMA-only and mixed kernels (each thread issues both) and prints TF/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int NF, int NM>
__global__ void mix(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-9;
  double av = a + threadIdx.x * 1e-12, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NF; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
#pragma unroll
    for (int k = 0; k < NM; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void lat(double* out, long long* cyc, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double c0 = 0, c1 = 0;
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; }
  out[threadIdx.x] = x + c0 + c1;
}

template <int NF, int NM>
double run(double* out, int sms, int bps) {
  const int iters = 2048;
  dim3 grid(sms * bps), block(256);
  mix<NF, NM><<<grid, block>>>(out, 8, 1.0000001, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<NF, NM><<<grid, block>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double thr = (double)grid.x * block.x;
  const double f = 2.0 * NF * 8 * iters * thr + 2.0 * 256 * NM * 8 * iters * thr / 32;
  return f / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8 * 1024);
  cudaMalloc(&cyc, 16);
  for (int bps : {2, 4}) {
    printf("bps=%d dfma-only(16): %.2f TF\n", bps, run<16, 0>(out, sms, bps));
    printf("bps=%d dmma-only(4): %.2f TF\n", bps, run<0, 4>(out, sms, bps));
    printf("bps=%d mix 16 dfma x8 + 4 dmma x8: %.2f TF (pure-time sum would be ~%.2f)\n", bps, run<16, 4>(out, sms, bps), 0.0);
    printf("bps=%d mix 32 dfma x8 + 4 dmma x8: %.2f TF\n", bps, run<32, 4>(out, sms, bps));
    printf("bps=%d mix 8 dfma x8 + 4 dmma x8: %.2f TF\n", bps, run<8, 4>(out, sms, bps));
  }
  lat<<<1, 32>>>(out, cyc, 1.0000001, 1e-9);
  long long h[2];
  cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  printf("dependent DFMA latency %.1f clk, dependent DMMA latency %.1f clk\n", h[0] / 1024.0, h[1] / 1024.0);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
