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

#include <algorithm>
#include <cstdint>

#include "attend.h"

namespace specsv_b200 {
namespace {

constexpr int kR1Threads = 512; // 16 warps: warp w owns compressed blocks [8(w%8), 8(w%8) + 8) of
                                // the tile and the row tiles of parity w/8
constexpr int kDhRoute = 128;   // d_head of this build (host-checked)
constexpr int kR1MaxMt = 8;     // up to 64 query rows (8-row MMA tiles) per CTA

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// fp64 logits on the FP64 tensor pipe: S[row][block] = q_row . ck_block in
// fp64 (fp32 x fp32 products are exact in fp64; the 4-term partial sums are
// accumulated in the MMA's order, within a few ulp of the reference's
// 4-lane order -- contract P3).  Persistent over 64-block tiles, next tile
// prefetched into registers.  Per-tile max / exp-sum fused.
template <int MT>
__global__ void __launch_bounds__(kR1Threads, 1)
    route_logits_kernel(const __grid_constant__ RouteParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ double red_m[8 * MT][8], red_s[8 * MT][8];
  __shared__ int is_last;
  constexpr int kRows = 8 * MT;
  constexpr int dh = kDhRoute;
  constexpr int qld = dh + 4;   // doubles (row stride 1056 B: conflict-light A loads)
  constexpr int ckld = dh + 4;  // floats
  const int kvh = blockIdx.y;
  const int rows_total = p.nr * p.G;
  const int r0 = blockIdx.z * kRows;
  const int nrows = min(kRows, rows_total - r0);
  double* qd = reinterpret_cast<double*>(smem);                             // [kRows][qld]
  float* ckbuf = reinterpret_cast<float*>(smem + (size_t)kRows * qld * 8);  // 2 x [64][ckld]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lr = lane >> 2, lc = lane & 3;  // fragment row / column within the 8x8 tile
  const int nt = warp & 7, mh = warp >> 3;  // block tile, row-tile parity
  constexpr int kKPer = kRouteTile * (dh / 4) / kR1Threads;  // 4 float4 per thread

  auto load_tile = [&](int t, float4 (&kv4)[kKPer]) {
#pragma unroll
    for (int it = 0; it < kKPer; ++it) {
      const int e = tid + it * kR1Threads;
      const int b = e / (dh / 4), x4 = e % (dh / 4);
      const int i = t * kRouteTile + b;
      kv4[it] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < p.ntiles && i < p.blocks)
        kv4[it] = __ldg(reinterpret_cast<const float4*>(p.ck + ((int64_t)i * p.Hkv + kvh) * dh + x4 * 4));
    }
  };
  auto store_tile = [&](float* dst, const float4 (&kv4)[kKPer]) {
#pragma unroll
    for (int it = 0; it < kKPer; ++it) {
      const int e = tid + it * kR1Threads;
      const int b = e / (dh / 4), x4 = e % (dh / 4);
      *reinterpret_cast<float4*>(dst + b * ckld + x4 * 4) = kv4[it];
    }
  };
  {  // q rows, fp32 -> fp64 (exact); rows past nrows are zero
    constexpr int kQPer = (kRows * (dh / 4) + kR1Threads - 1) / kR1Threads;
    float4 qv4[kQPer];
#pragma unroll
    for (int it = 0; it < kQPer; ++it) {
      const int e = tid + it * kR1Threads;
      const int r = e / (dh / 4), x4 = e % (dh / 4);
      qv4[it] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nrows) {
        const int rr = r0 + r;
        const int slot = rr / p.G, gg = rr % p.G;
        const int h = kvh * p.G + gg;
        qv4[it] = __ldg(reinterpret_cast<const float4*>(p.q + ((int64_t)p.slot_q[slot] * p.Hq + h) * dh + 4 * x4));
      }
    }
#pragma unroll
    for (int it = 0; it < kQPer; ++it) {
      const int e = tid + it * kR1Threads;
      const int r = e / (dh / 4), x4 = e % (dh / 4);
      if (r < kRows) {
        double* dst = qd + (size_t)r * qld + 4 * x4;
        dst[0] = qv4[it].x; dst[1] = qv4[it].y; dst[2] = qv4[it].z; dst[3] = qv4[it].w;
      }
    }
  }
  float4 kv4[kKPer];
  int t = blockIdx.x;
  load_tile(t, kv4);
  store_tile(ckbuf, kv4);
  __syncthreads();
  const int nmt = (nrows + 7) >> 3;
  for (int it_t = 0; t < p.ntiles; t += gridDim.x, ++it_t) {
    const float* cks = ckbuf + (it_t & 1) * kRouteTile * ckld;
    load_tile(t + gridDim.x, kv4);  // next tile, lands while this one is multiplied
    const int i0 = t * kRouteTile;
    constexpr int MH = MT / 2;  // row tiles per warp: mt = 2 j + mh
    double acc[MH][2];
#pragma unroll
    for (int j = 0; j < MH; ++j) acc[j][0] = acc[j][1] = 0.0;
    // B fragment: block (8 nt + lr), element 4 s + lc; A: row (8 mt + lr), element 4 s + lc
    const float* kb = cks + (8 * nt + lr) * ckld + lc;
    const double* qa = qd + (size_t)(8 * mh + lr) * qld + lc;
#pragma unroll 4
    for (int s = 0; s < dh / 4; ++s) {
      const double b = kb[4 * s];
#pragma unroll
      for (int j = 0; j < MH; ++j)
        if (2 * j + mh < nmt) dmma_8x8x4(acc[j], qa[(size_t)j * 16 * qld + 4 * s], b);
    }
    // C fragment: row 8 mt + lr, blocks 8 nt + 2 lc + {0, 1}
    const int blk = i0 + 8 * nt + 2 * lc;
#pragma unroll
    for (int j = 0; j < MH; ++j) {
      const int r = 8 * (2 * j + mh) + lr;
      const bool rowok = r < nrows;
      const int mvis = p.slot_mvis[(r0 + (rowok ? r : 0)) / p.G];
      double mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        acc[j][c] = __dmul_rn(acc[j][c], p.scale);
        if (rowok && blk + c < mvis) mx = fmax(mx, acc[j][c]);
      }
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      if (lc == 0 && 2 * j + mh < nmt) red_m[r][nt] = mx;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < MH; ++j) {
      if (2 * j + mh >= nmt) break;
      const int r = 8 * (2 * j + mh) + lr;
      const bool rowok = r < nrows;
      const int rr = r0 + (rowok ? r : 0);
      const int slot = rr / p.G, gg = rr % p.G;
      const int h = kvh * p.G + gg;
      const int mvis = p.slot_mvis[slot];
      double mx = red_m[r][0];
#pragma unroll
      for (int w = 1; w < 8; ++w) mx = fmax(mx, red_m[r][w]);
      double ev[2], sum = 0.0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const bool ok = rowok && blk + c < mvis;
        ev[c] = ok ? exp(acc[j][c] - mx) : 0.0;
        sum += ev[c];
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      if (lc == 0) red_s[r][nt] = sum;
      if (rowok)
        *reinterpret_cast<double2*>(p.E + ((int64_t)slot * p.Hq + h) * p.m_pad + blk) =
            make_double2(ev[0], ev[1]);
    }
    __syncthreads();
    if (tid < nrows) {
      const int rr = r0 + tid;
      const int slot = rr / p.G, gg = rr % p.G;
      const int h = kvh * p.G + gg;
      double mx = red_m[tid][0], sm = 0.0;
#pragma unroll
      for (int w = 1; w < 8; ++w) mx = fmax(mx, red_m[tid][w]);
#pragma unroll
      for (int w = 0; w < 8; ++w) sm += red_s[tid][w];
      p.TM[((int64_t)slot * p.Hq + h) * p.ntiles + t] = mx;
      p.TD[((int64_t)slot * p.Hq + h) * p.ntiles + t] = sm;
    }
    store_tile(ckbuf + ((it_t + 1) & 1) * kRouteTile * ckld, kv4);
    __syncthreads();
  }
  // the last CTA of this (row chunk, KV head) folds the tile statistics into
  // per-tile factors F_t = exp(m_t - M) / DEN (online-softmax merge), written
  // over TD; the counter returns to 0 for the next launch
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int* cnt = p.counters + blockIdx.z * p.Hkv + kvh;
    is_last = atomicAdd(cnt, 1) == (int)gridDim.x - 1;
    if (is_last) atomicExch(cnt, 0);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // row groups of the (rows x tiles) statistics go through shared memory in
  // one coalesced pass each (the q / key buffers are free now), then per-row
  // reductions run there
  constexpr size_t kSmemBytes = (size_t)kRows * qld * 8 + 2 * (size_t)kRouteTile * ckld * 4;
  const int rg = min(nrows, max(1, (int)(kSmemBytes / (16 * (size_t)p.ntiles))));
  double* sTM = reinterpret_cast<double*>(smem);
  double* sTD = sTM + rg * p.ntiles;
  for (int g0 = 0; g0 < nrows; g0 += rg) {
    const int gn = min(rg, nrows - g0);
    __syncthreads();
    for (int e = tid; e < gn * p.ntiles; e += kR1Threads) {
      const int rr = r0 + g0 + e / p.ntiles, tt = e % p.ntiles;
      const int64_t base = ((int64_t)(rr / p.G) * p.Hq + kvh * p.G + rr % p.G) * p.ntiles + tt;
      sTM[e] = __ldcg(p.TM + base);
      sTD[e] = __ldcg(p.TD + base);
    }
    __syncthreads();
    for (int r = warp; r < gn; r += kR1Threads / 32) {
      const double* tm = sTM + r * p.ntiles;
      const double* td = sTD + r * p.ntiles;
      double mx = -INFINITY;
      for (int tt = lane; tt < p.ntiles; tt += 32) mx = fmax(mx, tm[tt]);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      double den = 0.0;
      for (int tt = lane; tt < p.ntiles; tt += 32)
        if (td[tt] > 0.0) den += td[tt] * exp(tm[tt] - mx);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
      const int rr = r0 + g0 + r;
      double* F = p.TD + ((int64_t)(rr / p.G) * p.Hq + kvh * p.G + rr % p.G) * p.ntiles;
      for (int tt = lane; tt < p.ntiles; tt += 32)
        F[tt] = (den > 0.0 && tm[tt] != -INFINITY) ? exp(tm[tt] - mx) / den : 0.0;
    }
  }
}

template <int MT>
cudaError_t launch_r1(const RouteParams& p, cudaStream_t s) {
  constexpr int kRows = 8 * MT;
  const int rows_total = p.nr * p.G;
  const int rchunks = (rows_total + kRows - 1) / kRows;
  const size_t smem1 = (size_t)kRows * (kDhRoute + 4) * 8 + 2 * (size_t)kRouteTile * (kDhRoute + 4) * 4;
  cudaError_t e = cudaFuncSetAttribute(route_logits_kernel<MT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = std::max(1, std::min(p.ntiles, sms / (p.Hkv * rchunks)));
  route_logits_kernel<MT><<<dim3(ctas, p.Hkv, rchunks), kR1Threads, smem1, s>>>(p);
  return cudaGetLastError();
}

constexpr int kR2Threads = 128;
constexpr int kR2Blocks = 128;     // compressed blocks per CTA

// mass_i = sum_h (ascending) E[h][i] * F[h][tile(i)] for i in [i0 - halo,
// i0 + 128), then the selection scores of the blocks starting in this chunk
// (nsa_attention.cpp:67-78: block b gets, in ascending i, mass_i * (1/Hq) *
// overlap / l from every compressed block overlapping it)
__global__ void __launch_bounds__(kR2Threads)
    route_mass_kernel(const __grid_constant__ RouteParams p) {
  __shared__ double smass[kR2Blocks + 8];
  const int slot = blockIdx.y;
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * kR2Blocks;
  const int halo = (p.l - 1) / p.d;  // <= 7 (host-checked)
  const int mvis = p.slot_mvis[slot];
  const double* F = p.TD;  // per-tile factors written by the last R1 CTA
  for (int k = tid; k < kR2Blocks + halo; k += kR2Threads) {
    const int i = i0 - halo + k;
    double mass = 0.0;
    if (i >= 0 && i < mvis) {
      const int t = i / kRouteTile;
      const double* E = p.E + (int64_t)slot * p.Hq * p.m_pad + i;
      const double* Fs = F + (int64_t)slot * p.Hq * p.ntiles + t;
      for (int h0 = 0; h0 < p.Hq; h0 += 16) {
        double ev[16], fv[16];
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) {
          const bool ok = h0 + k2 < p.Hq;
          ev[k2] = ok ? E[(int64_t)(h0 + k2) * p.m_pad] : 0.0;
          fv[k2] = ok ? Fs[(int64_t)(h0 + k2) * p.ntiles] : 0.0;
        }
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2)
          if (h0 + k2 < p.Hq) mass += ev[k2] * fv[k2];
      }
    }
    smass[k] = mass;
  }
  __syncthreads();
  const double inv_heads = 1.0 / (double)p.Hq;
  const int b_lo = (i0 * p.d + p.l_sel - 1) / p.l_sel;
  const int b_hi = ((i0 + kR2Blocks) * p.d + p.l_sel - 1) / p.l_sel;
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
      const int64_t k = i - (i0 - halo);
      const double mi = (k >= 0 && k < kR2Blocks + halo) ? smass[k] : 0.0;
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
// blocks first, then the best remaining by (score desc, id asc).
//  1. every warp's best candidate -> the K-th best of those is a lower bound
//     of the K-th best overall (K = picks needed, <= number of warps);
//  2. candidates ranking at or before that bound survive (typically ~K);
//  3. exact rank among the survivors.
__device__ void topn_write(const double* sel, int* surv, int avail, int n, int32_t* idx_row,
                           int32_t* count, uint32_t* forced_bits) {
  __shared__ double wbest_s[32];
  __shared__ int wbest_i[32];
  __shared__ double lb_s;
  __shared__ int lb_i, nsurv;
  __shared__ int picks[64];
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = nthr >> 5;
  const int f1 = avail - 2 > 0 ? avail - 2 : -1;
  const int f2 = avail - 1 > 0 ? avail - 1 : -1;
  const int nforced = avail > 0 ? 1 + (f1 > 0) + (f2 > 0 && f2 != f1) : 0;
  const int target = n < avail ? n : avail;
  const int want = target - nforced;
  auto cand = [&](int b, double& sc) {
    const bool forced = b == 0 || b == f1 || b == f2;
    sc = (b < avail && !forced) ? sel[b] : -INFINITY;
    return b < avail && !forced;
  };
  if (tid == 0) {
    nsurv = 0;
    lb_s = -INFINITY;  // no bound unless a warp maximum holds rank K-1
    lb_i = 0x7fffffff;
  }
  if (want > 0) {
    // 1. per-warp best over the warp's candidates (b = warp*32 + lane + k*nthr)
    double bs = -INFINITY;
    int bi = 0x7fffffff;
    for (int b = warp * 32 + lane; b < avail; b += nthr) {
      double sc;
      if (cand(b, sc) && ranks_before(sc, b, bs, bi)) { bs = sc; bi = b; }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ranks_before(os, oi, bs, bi)) { bs = os; bi = oi; }
    }
    if (lane == 0) { wbest_s[warp] = bs; wbest_i[warp] = bi; }
    __syncthreads();
    if (warp == 0) {  // K-th best warp maximum (rank counting among <= 32)
      const double ms = lane < nwarps ? wbest_s[lane] : -INFINITY;
      const int mi = lane < nwarps ? wbest_i[lane] : 0x7fffffff;
      int rank = 0;
      for (int o = 0; o < nwarps; ++o) rank += ranks_before(wbest_s[o], wbest_i[o], ms, mi) ? 1 : 0;
      const int kk = want <= nwarps ? want - 1 : -1;
      if (kk >= 0 && lane < nwarps && rank == kk && ms != -INFINITY) { lb_s = ms; lb_i = mi; }
    }
    __syncthreads();
    // 2. survivors: rank at or before the bound
    const double ls = lb_s;
    const int li = lb_i;
    for (int b = tid; b < avail; b += nthr) {
      double sc;
      if (cand(b, sc) && (ranks_before(sc, b, ls, li) || (sc == ls && b == li))) {
        const int slotn = atomicAdd(&nsurv, 1);
        surv[slotn] = b;
      }
    }
    __syncthreads();
    // 3. exact rank among survivors
    const int ns = nsurv;
    for (int k = tid; k < ns; k += nthr) {
      const int b = surv[k];
      const double sb = sel[b];
      int rank = 0;
      for (int o = 0; o < ns; ++o) {
        const int c = surv[o];
        rank += ranks_before(sel[c], c, sb, b) ? 1 : 0;
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
  int* surv = reinterpret_cast<int*>(sel + kMaxAvail);
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
  topn_write(sel, surv, avail, p.n, p.idx + (int64_t)q * p.n, p.idx_count + q, p.idx_forced + q);
}

__global__ void __launch_bounds__(kR3Threads)
    select_only_kernel(const double* scores, int avail, int n, int32_t* idx, int32_t* count,
                       uint32_t* forced) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* sel = reinterpret_cast<double*>(smem);
  int* surv = reinterpret_cast<int*>(sel + kMaxAvail);
  for (int b = threadIdx.x; b < avail; b += blockDim.x) sel[b] = scores[b];
  __syncthreads();
  topn_write(sel, surv, avail, n, idx, count, forced);
}

constexpr size_t kR3Smem = (size_t)kMaxAvail * 8 + (size_t)kMaxAvail * 4;

cudaError_t launch_r1_r2(const RouteParams& p, cudaStream_t s) {
  if (p.ntiles == 0) return cudaSuccess;  // nothing compressed is visible yet: all masses 0
  // rows per thread: 4 for the approx (few representatives) shapes, 12 otherwise
  const int rows = p.nr * p.G;
  const cudaError_t e = rows <= 16 ? launch_r1<2>(p, s) : rows <= 32 ? launch_r1<4>(p, s) : launch_r1<8>(p, s);
  if (e != cudaSuccess) return e;
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
