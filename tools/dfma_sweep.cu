// DFMA throughput vs resident warps per SM and independent chains per thread (issue-rate probe).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  double av = a + threadIdx.x * 1e-12, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}
template <int CH>
void run(int sms, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wps : {4, 8, 16, 32}) {  // warps per SM
    int threads = wps * 32, blocks = sms;
    int iters = 4096;
    k<CH><<<blocks, threads>>>(out, 8, 1.0, 1e-9);
    cudaEventRecord(e0);
    k<CH><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double inst = (double)CH * iters * wps;  // warp-DFMAs per SM
    double cyc = ms * 1e-3 * 1.965e9;
    printf("chains=%2d warps/SM=%2d  %.2f TF  %.2f clk per warp-DFMA per scheduler (warps/sched %d)\n", CH, wps,
           2.0 * 32 * inst * sms / (ms * 1e-3) / 1e12, cyc / (inst / 4), wps / 4);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  run<1>(sms, out); run<2>(sms, out); run<4>(sms, out); run<8>(sms, out); run<16>(sms, out);
  return 0;
}
