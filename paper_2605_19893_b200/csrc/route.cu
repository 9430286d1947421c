// route.cu -- refresh-layer routing on sm_100a: fp64 compressed-block scores
// and Top-n block selection with forced blocks.
//
// Replaces nsa::selection_scores + nsa::select_blocks
// (src/nsa_attention.cpp:38-136) for every query that constructs indices.
//
//  R1 (grid: 64-block tiles x KV heads x row chunks): per (query, head,
//     block) logit = dot(q_h, ck_i) * 1/sqrt(dh) in fp64 with the reference's
//     lane order (4 interleaved partial sums, (s0+s2)+(s1+s3)); fp32 x fp32
//     products are exact in fp64, so DFMA == the reference's mul-then-add and
//     the logits are bit-identical.  Register blocking: 8 query rows x 2
//     blocks per thread (the q rows are warp-broadcast smem reads, the key
//     rows per-lane reads), fused per-tile max and exp-sum.
//  R2 (grid: 128-block chunks x routed queries): merge tile statistics per
//     head (online-softmax merge), then mass_i = sum_h (ascending) p_hi.
//  R3 (one CTA per routed query): overlap remap to selection blocks in the
//     reference's ascending order, then Top-n: forced {0, avail-2, avail-1}
//     plus the best remaining by (score desc, id asc) via an in-smem bitonic
//     sort, written ascending.
#include <cuda_runtime.h>

#include <cstdint>

#include "attend.h"

namespace specsv_b200 {
namespace {

constexpr int kRowsPerWarp = 8;

__global__ void __launch_bounds__(256)
    route_logits_kernel(const __grid_constant__ RouteParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int dh = p.dh;
  const int tile = blockIdx.x, kvh = blockIdx.y;
  const int rows_total = p.nr * p.G;
  const int r0 = blockIdx.z * kRouteRows;
  const int nrows = min(kRouteRows, rows_total - r0);
  double* qd = reinterpret_cast<double*>(smem);                          // [nrows][dh]
  float* cks = reinterpret_cast<float*>(smem + (size_t)nrows * dh * 8);  // [64][dh + 4]
  const int ckld = dh + 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nthr = blockDim.x;

  for (int e = tid; e < nrows * (dh / 4); e += nthr) {  // q rows, fp32 -> fp64 (exact)
    const int r = e / (dh / 4), x4 = e % (dh / 4);
    const int rr = r0 + r;
    const int slot = rr / p.G, g = rr % p.G;
    const int h = kvh * p.G + g;
    const float4 v = *reinterpret_cast<const float4*>(p.q + ((int64_t)p.slot_q[slot] * p.Hq + h) * dh + 4 * x4);
    double* dst = qd + (size_t)r * dh + 4 * x4;
    dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
  }
  const int i0 = tile * kRouteTile;
  for (int e = tid; e < kRouteTile * (dh / 4); e += nthr) {  // key tile (zero beyond the cache)
    const int b = e / (dh / 4), x4 = e % (dh / 4);
    const int i = i0 + b;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < p.blocks) v = *reinterpret_cast<const float4*>(p.ck + ((int64_t)i * p.Hkv + kvh) * dh + x4 * 4);
    *reinterpret_cast<float4*>(cks + b * ckld + x4 * 4) = v;
  }
  __syncthreads();

  const int rbase = warp * kRowsPerWarp;
  if (rbase >= nrows) return;
  const float* k0 = cks + lane * ckld;
  const float* k1 = cks + (lane + 32) * ckld;
  double acc[kRowsPerWarp][2][4];
#pragma unroll
  for (int a = 0; a < kRowsPerWarp; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;
  const double* qrow[kRowsPerWarp];
#pragma unroll
  for (int a = 0; a < kRowsPerWarp; ++a) qrow[a] = qd + (size_t)min(rbase + a, nrows - 1) * dh;
#pragma unroll 1
  for (int x = 0; x < dh; x += 4) {
    const float4 ka = *reinterpret_cast<const float4*>(k0 + x);
    const float4 kb = *reinterpret_cast<const float4*>(k1 + x);
    const double ka0 = ka.x, ka1 = ka.y, ka2 = ka.z, ka3 = ka.w;
    const double kb0 = kb.x, kb1 = kb.y, kb2 = kb.z, kb3 = kb.w;
#pragma unroll
    for (int a = 0; a < kRowsPerWarp; ++a) {
      const double2 qa = *reinterpret_cast<const double2*>(qrow[a] + x);
      const double2 qb = *reinterpret_cast<const double2*>(qrow[a] + x + 2);
      acc[a][0][0] = fma(qa.x, ka0, acc[a][0][0]);
      acc[a][0][1] = fma(qa.y, ka1, acc[a][0][1]);
      acc[a][0][2] = fma(qb.x, ka2, acc[a][0][2]);
      acc[a][0][3] = fma(qb.y, ka3, acc[a][0][3]);
      acc[a][1][0] = fma(qa.x, kb0, acc[a][1][0]);
      acc[a][1][1] = fma(qa.y, kb1, acc[a][1][1]);
      acc[a][1][2] = fma(qb.x, kb2, acc[a][1][2]);
      acc[a][1][3] = fma(qb.y, kb3, acc[a][1][3]);
    }
  }
#pragma unroll
  for (int a = 0; a < kRowsPerWarp; ++a) {
    const int r = rbase + a;
    if (r >= nrows) break;  // warp-uniform
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
    const double e0 = ok[0] ? exp(lg[0] - mx) : 0.0;
    const double e1 = ok[1] ? exp(lg[1] - mx) : 0.0;
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

constexpr int kR2Threads = 128;
constexpr int kR2Blocks = 128;  // compressed blocks per CTA (2 R1 tiles)

__global__ void __launch_bounds__(kR2Threads)
    route_mass_kernel(const __grid_constant__ RouteParams p) {
  __shared__ double sM[128], sD[128];
  __shared__ double sF[128][kR2Blocks / kRouteTile];
  const int slot = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * kR2Blocks;
  const int t0 = i0 / kRouteTile;
  // per-head softmax statistics merged over the tiles (online-softmax merge)
  for (int h = warp; h < p.Hq; h += kR2Threads / 32) {
    const double* TM = p.TM + ((int64_t)slot * p.Hq + h) * p.ntiles;
    const double* TD = p.TD + ((int64_t)slot * p.Hq + h) * p.ntiles;
    double mx = -INFINITY, den = 0.0;
    for (int t0l = 0; t0l < p.ntiles; t0l += 128) {
      double tm[4], td[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = t0l + lane + 32 * k;
        tm[k] = t < p.ntiles ? TM[t] : -INFINITY;
        td[k] = t < p.ntiles ? TD[t] : 0.0;
      }
      double cmx = fmax(fmax(tm[0], tm[1]), fmax(tm[2], tm[3]));
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) cmx = fmax(cmx, __shfl_xor_sync(0xffffffffu, cmx, off));
      double cden = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (td[k] > 0.0) cden += td[k] * exp(tm[k] - cmx);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) cden += __shfl_xor_sync(0xffffffffu, cden, off);
      if (cmx != -INFINITY) {
        const double nm = fmax(mx, cmx);
        den = (mx == -INFINITY ? 0.0 : den * exp(mx - nm)) + cden * exp(cmx - nm);
        mx = nm;
      }
    }
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
  // mass for i in [i0 - halo, i0 + kR2Blocks): the halo covers the compressed
  // blocks that straddle into this chunk's first selection block
  __shared__ double smass[kR2Blocks + 8];
  const int halo = (p.l - 1) / p.d;  // <= 7 (host-checked)
  const int mvis = p.slot_mvis[slot];
  for (int k = tid; k < kR2Blocks + halo; k += kR2Threads) {
    const int i = i0 - halo + k;
    double mass = 0.0;
    if (i >= 0 && i < mvis) {
      const int tt = i / kRouteTile;
      const double* E = p.E + (int64_t)slot * p.Hq * p.m_pad + i;
      for (int h0 = 0; h0 < p.Hq; h0 += 16) {  // loads in flight, then accumulate in head order
        double e[16], f[16];
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) {
          e[k2] = h0 + k2 < p.Hq ? E[(int64_t)(h0 + k2) * p.m_pad] : 0.0;
          f[k2] = 0.0;
        }
        if (tt >= t0 && tt < t0 + kR2Blocks / kRouteTile) {
#pragma unroll
          for (int k2 = 0; k2 < 16; ++k2) f[k2] = h0 + k2 < p.Hq ? sF[h0 + k2][tt - t0] : 0.0;
        } else {  // halo block of the previous chunk: factor from the tile statistics
#pragma unroll
          for (int k2 = 0; k2 < 16; ++k2) {
            const int h = h0 + k2;
            if (h < p.Hq && sD[h] > 0.0) {
              const double tm = p.TM[((int64_t)slot * p.Hq + h) * p.ntiles + tt];
              f[k2] = tm == -INFINITY ? 0.0 : exp(tm - sM[h]) / sD[h];
            }
          }
        }
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2)
          if (h0 + k2 < p.Hq) mass += e[k2] * f[k2];
      }
    }
    smass[k] = mass;
  }
  __syncthreads();
  // selection scores (nsa_attention.cpp:67-78): block b gets, in ascending i,
  // mass_i * (1/Hq) * overlap / l from every compressed block overlapping it
  const double inv_heads = 1.0 / (double)p.Hq;
  const int b_lo = (i0 * p.d + p.l_sel - 1) / p.l_sel;                  // first block starting in chunk
  const int b_hi = ((i0 + kR2Blocks) * p.d + p.l_sel - 1) / p.l_sel;    // exclusive
  const int avail = p.slot_avail[slot];
  for (int b = b_lo + tid; b < b_hi && b < avail; b += kR2Threads) {
    const int64_t blo = (int64_t)b * p.l_sel, bhi = blo + p.l_sel;
    const int64_t ilo = blo - p.l < 0 ? 0 : (blo - p.l) / p.d + 1;
    double sacc = 0.0;
    for (int64_t i = ilo; i < mvis && i * p.d < bhi; ++i) {
      const int64_t lo = i * p.d, hi = lo + p.l;
      const int64_t olo = lo > blo ? lo : blo;
      const int64_t ohi = hi < bhi ? hi : bhi;
      if (ohi <= olo) continue;
      const double mi = (i - (i0 - halo)) < kR2Blocks + halo ? smass[i - (i0 - halo)] : 0.0;
      sacc = __dadd_rn(sacc, __ddiv_rn(__dmul_rn(__dmul_rn(mi, inv_heads), (double)(ohi - olo)),
                                       (double)p.l));
    }
    p.sel[(int64_t)slot * p.sel_pad + b] = sacc;
  }
}

constexpr int kR3Threads = 1024;

// (score desc, id asc): true when (sa, ia) ranks before (sb, ib)
__device__ __forceinline__ bool ranks_before(double sa, int ia, double sb, int ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// Top-n over sel[0, avail) (select_blocks, nsa_attention.cpp:94-136): forced
// blocks first, then the best remaining by (score desc, id asc).  Each
// candidate counts the candidates that rank before it, stopping once it
// cannot be among the winners; a winner's count is its rank.
__device__ void topn_write(const double* sel, int avail, int n, int32_t* idx_row, int32_t* count,
                           uint32_t* forced_bits) {
  __shared__ int picks[64];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int f1 = avail - 2 > 0 ? avail - 2 : -1;
  const int f2 = avail - 1 > 0 ? avail - 1 : -1;
  const int nforced = avail > 0 ? 1 + (f1 > 0) + (f2 > 0 && f2 != f1) : 0;
  const int target = n < avail ? n : avail;
  const int want = target - nforced;  // picks among the non-forced blocks
  if (tid < 64) picks[tid] = -1;
  __syncthreads();
  for (int b = tid; b < avail && want > 0; b += nthr) {
    const bool forced = b == 0 || b == f1 || b == f2;
    int rank = 0;
    if (!forced) {
      const double sb = sel[b];
      for (int c = 0; c < avail && rank < want; ++c) {
        const bool cf = c == 0 || c == f1 || c == f2;
        rank += (!cf && ranks_before(sel[c], c, sb, b)) ? 1 : 0;
      }
      if (rank < want) picks[nforced + rank] = b;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int cnt = 0;
    if (avail > 0) {
      picks[cnt++] = 0;
      if (f1 > 0) picks[cnt++] = f1;
      if (f2 > 0 && f2 != f1) picks[cnt++] = f2;
    }
    cnt = target > 0 ? target : 0;
    for (int a = 1; a < cnt; ++a) {  // ascending
      const int v = picks[a];
      int b = a - 1;
      while (b >= 0 && picks[b] > v) { picks[b + 1] = picks[b]; --b; }
      picks[b + 1] = v;
    }
    uint32_t fb = 0u;
    for (int a = 0; a < n; ++a) {
      idx_row[a] = a < cnt ? picks[a] : -1;
      if (a < cnt && (picks[a] == 0 || picks[a] == f1 || picks[a] == f2)) fb |= 1u << a;
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
  double* sel = reinterpret_cast<double*>(smem);
  for (int b = threadIdx.x; b < avail; b += blockDim.x) {
    const double v = p.ntiles > 0 ? p.sel[(int64_t)slot * p.sel_pad + b] : 0.0;
    sel[b] = v;
    if (scores_out != nullptr) scores_out[b] = v;
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
  topn_write(sel, avail, p.n, p.idx + (int64_t)q * p.n, p.idx_count + q, p.idx_forced + q);
}

__global__ void __launch_bounds__(kR3Threads)
    select_only_kernel(const double* scores, int avail, int n, int32_t* idx, int32_t* count,
                       uint32_t* forced) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* sel = reinterpret_cast<double*>(smem);
  for (int b = threadIdx.x; b < avail; b += blockDim.x) sel[b] = scores[b];
  __syncthreads();
  topn_write(sel, avail, n, idx, count, forced);
}

constexpr size_t kR3Smem = (size_t)kMaxAvail * 8;

cudaError_t launch_r1_r2(const RouteParams& p, cudaStream_t s) {
  if (p.ntiles == 0) return cudaSuccess;  // nothing compressed is visible yet: all masses 0
  const int rows_total = p.nr * p.G;
  const int rchunks = (rows_total + kRouteRows - 1) / kRouteRows;
  const int maxrows = rows_total < kRouteRows ? rows_total : kRouteRows;
  const size_t smem1 = (size_t)maxrows * p.dh * 8 + (size_t)kRouteTile * (p.dh + 4) * 4;
  cudaError_t e = cudaFuncSetAttribute(route_logits_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(route_logits_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  const int warps = (maxrows + kRowsPerWarp - 1) / kRowsPerWarp;
  route_logits_kernel<<<dim3(p.ntiles, p.Hkv, rchunks), 32 * warps, smem1, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // one extra chunk so the selection blocks that start past the last compressed block get written
  route_mass_kernel<<<dim3((p.m_pad + kR2Blocks - 1) / kR2Blocks + 1, p.nr), kR2Threads, 0, s>>>(p);
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
