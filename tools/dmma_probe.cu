// Microbenchmark: sustained FP64 tensor (DMMA m8n8k4) throughput and
// dependent-chain latency on this GPU (diagnostic only).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(double* d, int sms, cudaEvent_t e0, cudaEvent_t e1, int threads, int bps) {
  int blocks = sms * bps, iters = 2048;
  dmma_kernel<CH><<<blocks, threads>>>(d, 16, 0.999, 1e-6);
  cudaEventRecord(e0);
  dmma_kernel<CH><<<blocks, threads>>>(d, iters, 0.999, 1e-6);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * CH * iters * (double)blocks * (threads / 32);
  printf("DMMA chains=%d warps/SM=%d: %.2f TFLOP/s  (%.2f SM-cycles per DMMA at 1.9 GHz)\n", CH,
         threads / 32 * bps, flops / ms / 1e9,
         1.9e9 * sms / (flops / 512 / (ms * 1e-3)));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  run<1>(d, sms, e0, e1, 32, 1);
  run<1>(d, sms, e0, e1, 128, 1);
  run<4>(d, sms, e0, e1, 128, 1);
  run<8>(d, sms, e0, e1, 128, 1);
  run<4>(d, sms, e0, e1, 256, 1);
  run<5>(d, sms, e0, e1, 512, 1);
  run<8>(d, sms, e0, e1, 512, 1);
  run<8>(d, sms, e0, e1, 1024, 1);
  return 0;
}
