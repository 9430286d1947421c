// Microbenchmark: dependent-chain latency of DFMA, DADD, fp64 exp and div,
// FFMA and expf on one warp (diagnostic only).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double x0, int steps, long long* out, double* sink) {
  double x = x0 + threadIdx.x * 1e-9;
  float f = (float)x;
  long long t0, t1;
  t0 = clock64();
  for (int k = 0; k < steps; ++k) x = fma(x, 0.9999999, 1e-9);
  t1 = clock64(); out[0] = (t1 - t0) / steps;
  t0 = clock64();
  for (int k = 0; k < steps; ++k) x = exp(x - 1.0);
  t1 = clock64(); out[1] = (t1 - t0) / steps;
  t0 = clock64();
  for (int k = 0; k < steps; ++k) x = 1.0 / (x + 1.5);
  t1 = clock64(); out[2] = (t1 - t0) / steps;
  t0 = clock64();
  for (int k = 0; k < steps; ++k) f = fmaf(f, 0.9999f, 1e-6f);
  t1 = clock64(); out[3] = (t1 - t0) / steps;
  t0 = clock64();
  for (int k = 0; k < steps; ++k) f = __expf(f - 1.0f);
  t1 = clock64(); out[4] = (t1 - t0) / steps;
  t0 = clock64();
  for (int k = 0; k < steps; ++k) x = x + 1e-9;
  t1 = clock64(); out[5] = (t1 - t0) / steps;
  sink[threadIdx.x] = x + f;
}
int main() {
  long long* out; double* sink;
  cudaMalloc(&out, 64); cudaMalloc(&sink, 1024);
  lat<<<1, 32>>>(0.5, 100, out, sink);
  lat<<<1, 32>>>(0.5, 4000, out, sink);
  long long r[6];
  cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
  const char* n[6] = {"DFMA", "exp(double)", "1/x double", "FFMA", "__expf", "DADD"};
  for (int i = 0; i < 6; ++i) printf("%-12s dependent latency: %lld cycles\n", n[i], r[i]);
  return 0;
}
