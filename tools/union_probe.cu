// Diagnostics (not product code): the attend kernel's union build
// (coop_union) in isolation -- 12 softmax warps, C2-shaped index rows (9
// queries x 16 random selection blocks of 1024, a 512-token window) -- SM
// cycles per step, measured with clock64 on warp 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_19893_b200/csrc -I include \
//     tools/union_probe.cu paper_2605_19893_b200/csrc/policy.cpp -lcuda -o tools/union_probe
#include "attend.cu"
#include <cstdio>

namespace specsv_b200 {
namespace {
__global__ void __launch_bounds__(kThreads, 1) union_probe(const int* qsel, int nqc, int n, int rows, int wlo, int whi,
                                                           long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Misc& m = *reinterpret_cast<Misc*>(smem + kOffMisc);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int rep = 0; rep < 1; ++rep) {
    if (warp == kWarpUnion) {
      if (lane == 0) {
        mbar_init(&m.rows_ready, 32);
        mbar_init(&m.union_ready, 32);
        fence_mbar_init();
      }
      __syncwarp();
      zero_union(m, nqc, n, 64, rows, wlo, whi, lane);
      for (int e = lane; e < nqc * n; e += 32) m.qsel[e] = qsel[e];
      if (lane < nqc) {
        m.qcount[lane] = n;
        m.qbound[lane] = rows;
      }
    }
    __syncthreads();
    if (warp == kWarpUnion) mbar_arrive(&m.rows_ready);
    if (warp < kSoftWarps) {
      const long long c0 = clock64();
      unsigned long long tr[64];
      coop_union(m, tid, nqc, n, 64, rows, wlo, whi, tid == 0 ? tr : nullptr);
      if (tid == 0) {
        out[rep * 8 + 0] = clock64() - c0;
        out[rep * 8 + 1] = tr[57];
        out[rep * 8 + 2] = tr[58];
        out[rep * 8 + 3] = tr[60];
        out[rep * 8 + 4] = tr[47];
        out[rep * 8 + 5] = tr[31];
        out[rep * 8 + 6] = m.n_union;
      }
    }
    __syncthreads();
  }
}
}  // namespace
}  // namespace specsv_b200

int main() {
  using namespace specsv_b200;
  const int nqc = 9, n = 16, rows = 65536;
  int h[nqc * n];
  unsigned s = 12345;
  for (int i = 0; i < nqc * n; ++i) {
    s = s * 1103515245u + 12345u;
    h[i] = (s >> 8) % 1024;
  }
  int* d;
  long long* o;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 64 * sizeof(long long));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const size_t sm = attend_smem_bytes();
  cudaFuncSetAttribute(union_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  union_probe<<<1, kThreads, sm>>>(d, nqc, n, rows, rows - 520, rows + 7, o);
  long long r[64];
  cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int rep = 0; rep < 1; ++rep)
    printf("rep %d: total %lld cycles; rows %lld, bits+bar %lld, scatter %lld, own %lld, bar %lld; n_union %lld\n", rep,
           r[rep * 8], r[rep * 8 + 1], r[rep * 8 + 2], r[rep * 8 + 3], r[rep * 8 + 4], r[rep * 8 + 5], r[rep * 8 + 6]);
  return 0;
}
