// route.cu -- refresh-layer routing on sm_100a: fp64 compressed-block scores
// and Top-n block selection with forced blocks.
//
// Replaces nsa::selection_scores + nsa::select_blocks
// (src/nsa_attention.cpp:38-136) for every query that constructs indices.
//
//  R1 (grid: compressed-block tiles x KV heads x row chunks): per (query, head,
//     block) logit = dot(q_h, ck_i) * 1/sqrt(dh) in fp64 with the reference's
//     lane order (4 interleaved partial sums, (s0+s2)+(s1+s3)); fp32 x fp32
//     products are exact in fp64, so DFMA == the reference's mul-then-add and
//     the logits are bit-identical.  Fused: per-tile max and exp-sum.
//  R2 (grid: block chunks x routed queries): merge tile statistics per head
//     (online-softmax merge), then mass_i = sum_h (ascending) p_hi.
//  R3 (one CTA per routed query): overlap remap to selection blocks in the
//     reference's ascending order, then Top-n: forced {0, avail-2, avail-1}
//     plus the best remaining by (score desc, id asc), written ascending.
#include <cuda_runtime.h>

#include <cstdint>

#include "attend.h"

namespace specsv_b200 {
namespace {

constexpr int kR1Threads = 256;

__global__ void __launch_bounds__(kR1Threads)
    route_logits_kernel(const __grid_constant__ RouteParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int dh = p.dh;
  const int tile = blockIdx.x, kvh = blockIdx.y;
  const int rows_total = p.nr * p.G;
  const int r0 = blockIdx.z * kRouteRows;
  const int nrows = min(kRouteRows, rows_total - r0);
  double* qd = reinterpret_cast<double*>(smem);                    // [nrows][dh]
  float* cks = reinterpret_cast<float*>(smem + (size_t)nrows * dh * 8);  // [64][dh + 4]
  const int ckld = dh + 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // q rows (fp32 -> fp64, exact)
  for (int e = tid; e < nrows * dh; e += kR1Threads) {
    const int r = e / dh, x = e % dh;
    const int rr = r0 + r;
    const int slot = rr / p.G, g = rr % p.G;
    const int q = p.slot_q[slot];
    const int h = kvh * p.G + g;
    qd[e] = (double)p.q[((int64_t)q * p.Hq + h) * dh + x];
  }
  // compressed keys of this tile (zero beyond the cache)
  const int i0 = tile * kRouteTile;
  for (int e = tid; e < kRouteTile * (dh / 4); e += kR1Threads) {
    const int b = e / (dh / 4), x4 = e % (dh / 4);
    const int i = i0 + b;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < p.blocks) {
      v = *reinterpret_cast<const float4*>(p.ck + ((int64_t)i * p.Hkv + kvh) * dh + x4 * 4);
    }
    *reinterpret_cast<float4*>(cks + b * ckld + x4 * 4) = v;
  }
  __syncthreads();

  const float* k0 = cks + lane * ckld;
  const float* k1 = cks + (lane + 32) * ckld;
  for (int rbase = warp; rbase < nrows; rbase += 8 * 4) {
    double acc[4][2][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;
    int rowi[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) rowi[a] = min(rbase + 8 * a, nrows - 1);
    for (int x = 0; x < dh; x += 4) {
      const float4 ka = *reinterpret_cast<const float4*>(k0 + x);
      const float4 kb = *reinterpret_cast<const float4*>(k1 + x);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double2 qa = *reinterpret_cast<const double2*>(qd + (size_t)rowi[a] * dh + x);
        const double2 qb = *reinterpret_cast<const double2*>(qd + (size_t)rowi[a] * dh + x + 2);
        acc[a][0][0] = fma(qa.x, (double)ka.x, acc[a][0][0]);
        acc[a][0][1] = fma(qa.y, (double)ka.y, acc[a][0][1]);
        acc[a][0][2] = fma(qb.x, (double)ka.z, acc[a][0][2]);
        acc[a][0][3] = fma(qb.y, (double)ka.w, acc[a][0][3]);
        acc[a][1][0] = fma(qa.x, (double)kb.x, acc[a][1][0]);
        acc[a][1][1] = fma(qa.y, (double)kb.y, acc[a][1][1]);
        acc[a][1][2] = fma(qb.x, (double)kb.z, acc[a][1][2]);
        acc[a][1][3] = fma(qb.y, (double)kb.w, acc[a][1][3]);
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = rbase + 8 * a;
      if (r >= nrows) continue;  // warp-uniform
      const int rr = r0 + r;
      const int slot = rr / p.G, g = rr % p.G;
      const int h = kvh * p.G + g;
      const int mvis = p.slot_mvis[slot];
      double lg[2];
      bool ok[2];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double dot = __dadd_rn(__dadd_rn(acc[a][b][0], acc[a][b][2]),
                                     __dadd_rn(acc[a][b][1], acc[a][b][3]));
        lg[b] = __dmul_rn(dot, p.scale);
        ok[b] = (i0 + lane + 32 * b) < mvis;
      }
      double mx = -INFINITY;
      if (ok[0]) mx = lg[0];
      if (ok[1]) mx = fmax(mx, lg[1]);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      double e0 = ok[0] ? exp(lg[0] - mx) : 0.0;
      double e1 = ok[1] ? exp(lg[1] - mx) : 0.0;
      double s = e0 + e1;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      double* E = p.E + ((int64_t)slot * p.Hq + h) * p.m_pad;
      E[i0 + lane] = e0;
      E[i0 + lane + 32] = e1;
      if (lane == 0) {
        p.TM[((int64_t)slot * p.Hq + h) * p.ntiles + tile] = mx;
        p.TD[((int64_t)slot * p.Hq + h) * p.ntiles + tile] = s;
      }
    }
  }
}

constexpr int kR2Threads = 256;
constexpr int kR2Blocks = 256;  // compressed blocks per CTA (4 R1 tiles)

__global__ void __launch_bounds__(kR2Threads)
    route_mass_kernel(const __grid_constant__ RouteParams p) {
  __shared__ double sM[128], sD[128];
  __shared__ double sF[128][kR2Blocks / kRouteTile];
  const int slot = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * kR2Blocks;
  const int t0 = i0 / kRouteTile;
  for (int h = warp; h < p.Hq; h += kR2Threads / 32) {
    const double* TM = p.TM + ((int64_t)slot * p.Hq + h) * p.ntiles;
    const double* TD = p.TD + ((int64_t)slot * p.Hq + h) * p.ntiles;
    double mx = -INFINITY;
    for (int t = lane; t < p.ntiles; t += 32) mx = fmax(mx, TM[t]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    double den = 0.0;
    for (int t = lane; t < p.ntiles; t += 32)
      if (TD[t] > 0.0) den += TD[t] * exp(TM[t] - mx);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
    if (lane == 0) {
      sM[h] = mx;
      sD[h] = den;
    }
  }
  __syncthreads();
  for (int e = tid; e < p.Hq * (kR2Blocks / kRouteTile); e += kR2Threads) {
    const int h = e / (kR2Blocks / kRouteTile), tt = e % (kR2Blocks / kRouteTile);
    const int t = t0 + tt;
    double f = 0.0;
    if (t < p.ntiles && sD[h] > 0.0) {
      const double tm = p.TM[((int64_t)slot * p.Hq + h) * p.ntiles + t];
      if (tm != -INFINITY) f = exp(tm - sM[h]) / sD[h];
    }
    sF[h][tt] = f;
  }
  __syncthreads();
  const int i = i0 + tid;
  if (i >= p.m_pad) return;
  const int tt = (i - i0) / kRouteTile;
  double mass = 0.0;
  if (i < p.slot_mvis[slot]) {
    for (int h = 0; h < p.Hq; ++h)
      mass += p.E[((int64_t)slot * p.Hq + h) * p.m_pad + i] * sF[h][tt];
  }
  p.mass[(int64_t)slot * p.m_pad + i] = mass;
}

constexpr int kR3Threads = 1024;

// (score desc, id asc): true when (sa, ia) ranks before (sb, ib)
__device__ __forceinline__ bool ranks_before(double sa, int ia, double sb, int ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// Top-n over sel[0, avail) in shared memory (select_blocks, nsa_attention.cpp:94-136)
__device__ void topn_write(const double* sel, uint8_t* taken, int avail, int n, int32_t* idx_row,
                           int32_t* count, uint32_t* forced_bits) {
  __shared__ double wbest_s[32];
  __shared__ int wbest_i[32];
  __shared__ int picks[64];
  __shared__ int npicks;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int b = tid; b < avail; b += blockDim.x) taken[b] = 0;
  __syncthreads();
  if (tid == 0) {
    npicks = 0;
    if (avail > 0) {
      picks[npicks++] = 0;
      taken[0] = 2;
      if (avail - 2 > 0) { picks[npicks++] = avail - 2; taken[avail - 2] = 2; }
      if (avail - 1 > 0) { picks[npicks++] = avail - 1; taken[avail - 1] = 2; }
    }
  }
  __syncthreads();
  const int target = min(n, avail);
  const int rounds = target - npicks;
  for (int r = 0; r < rounds; ++r) {
    double bs = -1.0;
    int bi = 0x7fffffff;
    for (int b = tid; b < avail; b += blockDim.x)
      if (!taken[b] && ranks_before(sel[b], b, bs, bi)) { bs = sel[b]; bi = b; }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ranks_before(os, oi, bs, bi)) { bs = os; bi = oi; }
    }
    if (lane == 0) { wbest_s[warp] = bs; wbest_i[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      bs = lane < nw ? wbest_s[lane] : -1.0;
      bi = lane < nw ? wbest_i[lane] : 0x7fffffff;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ranks_before(os, oi, bs, bi)) { bs = os; bi = oi; }
      }
      if (lane == 0 && bi != 0x7fffffff) {
        taken[bi] = 1;
        picks[npicks++] = bi;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    const int cnt = npicks;
    // ascending (insertion sort, <= n entries)
    for (int a = 1; a < cnt; ++a) {
      const int v = picks[a];
      int b = a - 1;
      while (b >= 0 && picks[b] > v) { picks[b + 1] = picks[b]; --b; }
      picks[b + 1] = v;
    }
    uint32_t fb = 0u;
    for (int a = 0; a < n; ++a) {
      idx_row[a] = a < cnt ? picks[a] : -1;
      if (a < cnt && taken[picks[a]] == 2) fb |= 1u << a;
    }
    *count = cnt;
    *forced_bits = fb;
  }
}

__global__ void __launch_bounds__(kR3Threads)
    route_select_kernel(const __grid_constant__ RouteParams p, double* scores_out, int only_slot) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int slot = only_slot >= 0 ? only_slot : blockIdx.x;
  const int avail = p.slot_avail[slot];
  const int mvis = p.slot_mvis[slot];
  double* sel = reinterpret_cast<double*>(smem);
  uint8_t* taken = smem + (size_t)kMaxAvail * 8;
  const double inv_heads = 1.0 / (double)p.Hq;
  const double* mass = p.mass + (int64_t)slot * p.m_pad;
  // overlap remap (nsa_attention.cpp:67-78), ascending i per selection block
  for (int b = threadIdx.x; b < avail; b += blockDim.x) {
    const int64_t blo = (int64_t)b * p.l_sel, bhi = blo + p.l_sel;
    int64_t ilo = blo - p.l < 0 ? 0 : (blo - p.l) / p.d + 1;
    if (blo - p.l < 0) ilo = 0;
    double s = 0.0;
    for (int64_t i = ilo; i < mvis && i * p.d < bhi; ++i) {
      const int64_t lo = i * p.d, hi = lo + p.l;
      const int64_t olo = lo > blo ? lo : blo;
      const int64_t ohi = hi < bhi ? hi : bhi;
      if (ohi <= olo) continue;
      s = __dadd_rn(s, __ddiv_rn(__dmul_rn(__dmul_rn(mass[i], inv_heads), (double)(ohi - olo)),
                                 (double)p.l));
    }
    sel[b] = s;
    if (scores_out != nullptr) scores_out[b] = s;
  }
  __syncthreads();
  if (scores_out != nullptr) return;
  if (blockIdx.x == 0) {
    for (int u = threadIdx.x; u < p.n_unrouted; u += blockDim.x) {
      const int q = p.unrouted[u];
      p.idx_count[q] = -1;
      p.idx_forced[q] = 0u;
      for (int a = 0; a < p.n; ++a) p.idx[(int64_t)q * p.n + a] = -1;
    }
  }
  const int q = p.slot_q[slot];
  topn_write(sel, taken, avail, p.n, p.idx + (int64_t)q * p.n, p.idx_count + q, p.idx_forced + q);
}

__global__ void __launch_bounds__(kR3Threads)
    select_only_kernel(const double* scores, int avail, int n, int32_t* idx, int32_t* count,
                       uint32_t* forced) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* sel = reinterpret_cast<double*>(smem);
  uint8_t* taken = smem + (size_t)kMaxAvail * 8;
  for (int b = threadIdx.x; b < avail; b += blockDim.x) sel[b] = scores[b];
  __syncthreads();
  topn_write(sel, taken, avail, n, idx, count, forced);
}

constexpr size_t kR3Smem = (size_t)kMaxAvail * 9;

cudaError_t launch_r1_r2(const RouteParams& p, cudaStream_t s) {
  if (p.ntiles == 0) return cudaSuccess;  // nothing compressed is visible yet: all masses 0
  const int rows_total = p.nr * p.G;
  const int rchunks = (rows_total + kRouteRows - 1) / kRouteRows;
  const int maxrows = rows_total < kRouteRows ? rows_total : kRouteRows;
  const size_t smem1 = (size_t)maxrows * p.dh * 8 + (size_t)kRouteTile * (p.dh + 4) * 4;
  cudaError_t e = cudaFuncSetAttribute(route_logits_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  if (e != cudaSuccess) return e;
  route_logits_kernel<<<dim3(p.ntiles, p.Hkv, rchunks), kR1Threads, smem1, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  route_mass_kernel<<<dim3((p.m_pad + kR2Blocks - 1) / kR2Blocks, p.nr), kR2Threads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_route(const RouteParams& p, cudaStream_t s, bool write_idx) {
  (void)write_idx;
  cudaError_t e = launch_r1_r2(p, s);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(route_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kR3Smem);
  if (e != cudaSuccess) return e;
  route_select_kernel<<<p.nr, kR3Threads, kR3Smem, s>>>(p, nullptr, -1);
  return cudaGetLastError();
}

cudaError_t launch_scores_only(const RouteParams& p, double* scores, int slot, cudaStream_t s) {
  cudaError_t e = launch_r1_r2(p, s);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(route_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kR3Smem);
  if (e != cudaSuccess) return e;
  route_select_kernel<<<1, kR3Threads, kR3Smem, s>>>(p, scores, slot);
  return cudaGetLastError();
}

cudaError_t launch_select(const double* scores, int avail, int n, int32_t* idx, int32_t* count,
                          uint32_t* forced, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(select_only_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kR3Smem);
  if (e != cudaSuccess) return e;
  select_only_kernel<<<1, kR3Threads, kR3Smem, s>>>(scores, avail, n, idx, count, forced);
  return cudaGetLastError();
}

}  // namespace specsv_b200
