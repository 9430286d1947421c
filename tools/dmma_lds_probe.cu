// Diagnostics (not product code): DMMA m8n8k4 throughput when the fragments
// come from shared memory the way route.cu's tile loop loads them (5 A + 2 B
// LDS.64 per 10 DMMAs per k step), for 4 / 8 / 16 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kLd = 132;
template <int MT, int NT>
__global__ void probe(double* out, int reps, int full_mantissa) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 64 * kLd; i += blockDim.x) sm[i] = full_mantissa ? (double)__sinf(0.37f * i + 0.11f) : 1e-3 * (i % 17);
  __syncthreads();
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  double acc[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  const double* qa = sm + lr * kLd + lc;
  const double* kb = sm + (40 + lr) * kLd + lc;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int s = 0; s < 32; ++s) {
      double a[MT], b[NT];
#pragma unroll
      for (int m = 0; m < MT; ++m) a[m] = qa[m * 8 * kLd + 4 * s];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = kb[(n & 1) * 8 * kLd + 4 * s];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
              : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
              : "d"(a[m]), "d"(b[n]));
    }
  }
  double t = 0;
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) t += acc[m][n][0] + acc[m][n][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int MT, int NT>
void run(double* d, int sms, int warps, int fm) {
  cudaFuncSetAttribute(probe<MT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * kLd * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 64;
  probe<MT, NT><<<sms, 32 * warps, 64 * kLd * 8>>>(d, 2, fm);
  cudaEventRecord(e0);
  probe<MT, NT><<<sms, 32 * warps, 64 * kLd * 8>>>(d, reps, fm);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas = (double)sms * warps * reps * 32 * MT * NT;
  printf("%s MT=%d NT=%d warps/SM=%2d: %.2f TFLOP/s, %.2f SM-cycles per DMMA (1.9 GHz)\n",
         fm ? "random-data" : "simple-data", MT, NT, warps, dmmas * 512 / (ms * 1e-3) / 1e12,
         1.9e9 * (ms * 1e-3) / (dmmas / sms));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 1 << 24);
  for (int fm : {0, 1})
    for (int w : {8, 16}) run<5, 2>(d, sms, w, fm);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
