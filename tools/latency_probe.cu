// Microbenchmark: dependent-load latency (pointer chase) for L2-resident
// global data (ld.cg), L1 hits, and shared memory (diagnostic only).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chase(const int* __restrict__ next, int steps, int mode, long long* out, int* sink) {
  __shared__ int s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = (i * 97 + 13) & 4095;
  __syncthreads();
  if (threadIdx.x != 0) return;
  int j = 0;
  long long t0 = clock64();
  if (mode == 0) {
    for (int k = 0; k < steps; ++k) j = __ldcg(next + j);
  } else if (mode == 1) {
    for (int k = 0; k < steps; ++k) j = __ldca(next + (j & 1023));
  } else {
    for (int k = 0; k < steps; ++k) j = s[j];
  }
  long long t1 = clock64();
  out[blockIdx.x] = (t1 - t0) / steps;
  sink[blockIdx.x] = j;
}
int main() {
  const int n = 1 << 22;  // 16 MB: L2-resident
  int* h = new int[n];
  unsigned x = 1;
  for (int i = 0; i < n; ++i) { x = x * 1664525u + 1013904223u; h[i] = (int)(x % n); }
  int *d, *sink; long long* out;
  cudaMalloc(&d, n * 4); cudaMalloc(&sink, 4096); cudaMalloc(&out, 4096);
  cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
  const char* names[3] = {"L2 (ld.cg, 16 MB random)", "L1 (ld.ca, 4 KB)", "shared"};
  for (int mode = 0; mode < 3; ++mode) {
    chase<<<1, 32>>>(d, 1000, mode, out, sink);  // warm
    chase<<<148, 32>>>(d, 2000, mode, out, sink);
    long long r[148];
    cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
    long long mn = r[0], mx = r[0], sum = 0;
    for (int i = 0; i < 148; ++i) { mn = r[i] < mn ? r[i] : mn; mx = r[i] > mx ? r[i] : mx; sum += r[i]; }
    printf("%-28s cycles per dependent load: min %lld avg %lld max %lld\n", names[mode], mn, sum / 148, mx);
  }
  return 0;
}
