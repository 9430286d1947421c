// Diagnostics (not product code): cycles per tcgen05.mma kind::f16 (M = 128,
// K = 16, both operands in shared memory, SW128) as a function of N and of
// the operand majorness, issued back to back by one thread and retired
// through one commit.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I paper_2605_19893_b200/csrc tools/mma_probe.cu -o tools/mma_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace sm100;

__global__ void probe(int n, int mn_major, int reps, int nacc, int nmma, int warp_issue, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (tid < 32) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp_issue ? tid < 32 : tid == 0) {
    const uint32_t a = smem_u32(smem), b = a + 65536;
    const uint32_t idesc = idesc_bf16(128, n, mn_major, mn_major);
    long long t0 = 0;
    for (int r = 0; r < reps + 1; ++r) {
      if (r == 1) t0 = clock64();
      if (warp_issue) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = mn_major ? desc_sw128(a + kk * 2048, 16384, 1024) : desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = mn_major ? desc_sw128(b + kk * 2048, 16384, 1024) : desc_sw128(b + (kk >> 2) * 32768 + (kk & 3) * 32, 16, 1024);
          umma_f16_warp(tbase + (kk % nacc) * n, ad, bd, idesc, kk >= nacc);
        }
        umma_commit_warp(&bar);
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = mn_major ? desc_sw128(a + kk * 2048, 16384, 1024) : desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = mn_major ? desc_sw128(b + kk * 2048, 16384, 1024) : desc_sw128(b + (kk >> 2) * 32768 + (kk & 3) * 32, 16, 1024);
          umma_f16(tbase + (kk % nacc) * n, ad, bd, idesc, kk >= nacc);
        }
        umma_commit(&bar);
      }
      mbar_wait(&bar, r & 1);
    }
    if (tid == 0) out[0] = (clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) { tc_fence_after(); tmem_dealloc<512>(tbase); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  auto run = [&](int n, int mn, int reps, int nacc, int w) {
    probe<<<1, 128, 160 * 1024>>>(n, mn, reps, nacc, 8, w, d);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    return h / (double)reps;
  };
  for (int w : {0, 1})
    for (int n : {48, 96, 192})
      for (int nacc : {1, 2, 4})
        if (n * nacc <= 512) printf("%s N=%3d 8 MMAs into %d accumulators: %6.1f cycles (commit->wait round trip)\n",
               w ? "warp-issue  " : "thread-issue", n, nacc, run(n, 0, 32, nacc, w));
  for (int w : {0, 1}) printf("%s MN-major N=96 8 MMAs: %6.1f\n", w ? "warp-issue  " : "thread-issue", run(96, 1, 32, 1, w));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
