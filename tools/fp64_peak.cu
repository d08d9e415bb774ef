// fp64 peak microbenchmark for the roofline denominators (DFMA vs DMMA).
// Prints one JSON line: {"dfma_tflops":..,"dmma_tflops":..,"sm_count":..}
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-9;
  double av = a + threadIdx.x * 1e-12, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  double best_f = 0, best_m = 0;
  for (int blocksPerSM : {4, 8}) {
    int iters = 4096;
    dim3 grid(sms * blocksPerSM), block(256);
    dfma_kernel<<<grid, block>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * iters * (double)grid.x * block.x;
    best_f = fmax(best_f, flops / (ms * 1e-3) / 1e12);
    dmma_kernel<<<grid, block>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dmma_kernel<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double mflops = 2.0 * 256 * 4 * 8 * iters * (double)grid.x * (block.x / 32);
    best_m = fmax(best_m, mflops / (ms * 1e-3) / 1e12);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sm_count\": %d, \"err\": \"%s\"}\n", best_f, best_m, sms,
         cudaGetErrorString(err));
  return err != cudaSuccess;
}
