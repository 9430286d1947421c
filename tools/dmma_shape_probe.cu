// Microbenchmark (diagnostic only): sustained FP64 tensor throughput of the
// mma.sync f64 shapes on this GPU -- m8n8k4 (sm_80) against the sm_90+
// m16n8k4 / m16n8k8 / m16n8k16 -- with non-uniform operands, 8 independent
// accumulator chains per warp, 16 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE, int CH>
__global__ void k(double* out, int iters) {
  const double s = 1.0 + threadIdx.x * 1e-7;
  double a[8], b[4], c[CH][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = s * (0.37 + i * 0.011);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = s * (0.53 - i * 0.017);
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) t += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int SHAPE>
void run(const char* name, double macs, double* d, int sms) {
  constexpr int CH = 8;
  const int threads = 512, iters = 1024;
  k<SHAPE, CH><<<sms, threads>>>(d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<SHAPE, CH><<<sms, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = (double)CH * iters * sms * (threads / 32);
  const double tf = 2.0 * macs * n / (ms * 1e-3) / 1e12;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = (ms * 1e-3) * clk * 1e3 / (n / sms);
  printf("%-9s %.2f TFLOP/s  %.2f SM-cycles per mma  %.2f cycles per 256 MACs\n", name, tf, cyc, cyc * 256.0 / macs);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, sizeof(double) * sms * 512);
  run<0>("m8n8k4", 256, d, sms);
  run<1>("m16n8k4", 512, d, sms);
  run<2>("m16n8k8", 1024, d, sms);
  run<3>("m16n8k16", 2048, d, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
