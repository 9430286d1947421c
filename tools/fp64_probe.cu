// Microbenchmark: sustained DFMA throughput on this GPU (diagnostic only).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * 2, iters = 4096;
    dfma_kernel<<<blocks, threads>>>(d, 16, 0.999, 1e-6);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 0.999, 1e-6);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
    ffma_kernel<<<blocks, threads>>>((float*)d, iters, 0.999f, 1e-6f);
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>((float*)d, iters, 0.999f, 1e-6f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  return 0;
}
