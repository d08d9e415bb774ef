// DMMA throughput vs resident warps per SM and independent accumulator chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-9;
  double av = a + threadIdx.x * 1e-12, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}
template <int CH>
void run(int sms, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wps : {4, 8, 16, 32, 64}) {  // warps per SM
    int threads = 128, blocks = sms * wps / 4;
    int iters = 2048;
    k<CH><<<blocks, threads>>>(out, 8, 1.0, 1e-9);
    cudaEventRecord(e0);
    k<CH><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * CH * (double)iters * blocks * (threads / 32);
    printf("chains=%2d warps/SM=%2d  %.2f TF\n", CH, wps, fl / (ms * 1e-3) / 1e12);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  run<1>(sms, out); run<2>(sms, out); run<4>(sms, out); run<8>(sms, out); run<16>(sms, out);
  return 0;
}
