// route.cu -- refresh-layer routing on sm_100a: fp64 compressed-block scores
// and Top-n block selection with forced blocks.
//
// Replaces nsa::selection_scores + nsa::select_blocks
// (src/nsa_attention.cpp:38-136) for every query that constructs indices.
//
// One cooperative persistent kernel (one 512-thread CTA per SM), two phases
// and a single grid-wide arrival barrier:
//  1. tiles (all CTAs): per (routed query, head, compressed block i) logit =
//     dot(q_h, ck_i) / sqrt(dh) in fp64 on the FP64 tensor pipe (DMMA
//     m8n8k4; fp32 x fp32 products are exact in fp64).  Per 64-block tile t
//     and row: TM = max logit, TD = sum e^(logit - TM), and for every
//     selection block b the tile touches G[t][b] = sum_i overlap(i, b) *
//     e^(logit_i - TM) -- the tile's share of b's score before the softmax
//     normalisation is known, so no per-block probabilities reach HBM.
//  2. tail (one CTA per routed query): per head M = max_t TM, DEN = sum_t TD
//     e^(TM - M), F_t = e^(TM_t - M) / DEN; score_b = sum_t sum_h (ascending)
//     F_ht G_ht[b] / (Hq l)  (= the reference's sum over blocks and heads of
//     p_hi * overlap / l, nsa_attention.cpp:52-78, regrouped -- contract P3);
//     then Top-n: forced {0, avail-2, avail-1} plus the best remaining by
//     (score desc, id asc), written ascending (nsa_attention.cpp:94-136).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "attend.h"
#include "sm100.cuh"

namespace specsv_b200 {
namespace {

constexpr int kR1Threads = 512;  // two groups of 8 warps; warp w of a group owns the
                                 // compressed blocks [8w, 8w + 8) of that group's tile
constexpr int kR1GroupThreads = kR1Threads / 2;
constexpr int kDhRoute = 128;    // d_head of this build (host-checked)
constexpr int kQld = kDhRoute + 4;   // q row stride, doubles (1056 B: conflict-light A loads)
constexpr int kCkld = kDhRoute + 4;  // key row stride, floats (528 B: conflict-free B loads)
constexpr int kW = kRouteSpan;       // selection blocks one warp's 8 compressed blocks touch
constexpr size_t kTopnSmem = (size_t)kMaxAvail * 8 + (size_t)kMaxAvail * 4;

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void tstamp_any(unsigned long long* tr, int k) {
  if (tr != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[k] = t;
  }
}
__device__ __forceinline__ void tstamp(unsigned long long* tr, int k) {
  if (tr != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[k] = t;
  }
}

// tokens shared by compressed block i ([i d, i d + l)) and selection block b
__device__ __forceinline__ int overlap(int i, int b, int d, int l, int l_sel) {
  const int lo = max(i * d, b * l_sel), hi = min(i * d + l, (b + 1) * l_sel);
  return hi > lo ? hi - lo : 0;
}

// dynamic shared memory of phase 1 (MT row tiles)
template <int MT>
struct TileSmem {
  static constexpr int kRows = 8 * MT;
  static constexpr size_t q = 0;                                            // [kRows][kQld] f64
  static constexpr size_t ck = q + (size_t)kRows * kQld * 8;                // [2 grp][2 buf][64][kCkld] f32
  static constexpr size_t red_m = ck + 4 * (size_t)kRouteTile * kCkld * 4;  // [2][kRows][8]
  static constexpr size_t red_s = red_m + 2 * (size_t)kRows * 8 * 8;        // [2][kRows][8]
  static constexpr size_t gpart = red_s + 2 * (size_t)kRows * 8 * 8;        // [2][kRows][8][kW]
  static constexpr size_t bytes = gpart + 2 * (size_t)kRows * 8 * kW * 8;
  static_assert(bytes <= 227 * 1024, "tile-phase shared memory");
};

// Phase 1.  S[row][block] = q_row . ck_block in fp64 on the FP64 tensor pipe;
// the 4-term partial sums are accumulated in the MMA's order, within a few
// ulp of the reference's 4-lane order (contract P3).
//
// The CTA's two warp groups ping-pong over alternate 64-block tiles
// (group-local named barriers), so one group's softmax epilogue overlaps the
// other's MMAs on the shared FP64 pipe.  Each group keeps its next tile in
// registers while the current one is multiplied.  Per-tile statistics go
// through shared buffers guarded by a group barrier at the end of each tile.
template <int MT>
__device__ __forceinline__ void tiles_phase(const RouteParams& p, uint8_t* smem,
                                            unsigned long long* trc) {
  using L = TileSmem<MT>;
  constexpr int kRows = L::kRows;
  constexpr int dh = kDhRoute;
  constexpr int qld = kQld, ckld = kCkld;
  const int kvh = blockIdx.y;
  const int rows_total = p.nr * p.G;
  const int r0 = blockIdx.z * p.chunk_rows;
  const int nrows = min(p.chunk_rows, rows_total - r0);
  const int nmt = (nrows + 7) >> 3;
  double* qd = reinterpret_cast<double*>(smem + L::q);
  float* ckbuf = reinterpret_cast<float*>(smem + L::ck);
  const int tid = threadIdx.x;
  const int grp = tid / kR1GroupThreads, gtid = tid % kR1GroupThreads;
  const int warp = gtid >> 5, lane = tid & 31;
  const int lr = lane >> 2, lc = lane & 3;  // fragment row / column within the 8x8 tile
  const int vstride = 2 * gridDim.x;  // tiles of this group: t = 2 blockIdx.x + grp + k vstride
  float* cks0 = ckbuf + grp * 2 * kRouteTile * ckld;  // this group's two key buffers
  const uint32_t gbar = 1 + grp;
  const int l = p.l, d = p.d, l_sel = p.l_sel;

  // key tile t -> buffer, fire-and-forget (cp.async, blocks past the cache zero-filled)
  auto issue_tile = [&](int t, float* dst) {
    constexpr int kPer = kRouteTile * (dh / 4) / kR1GroupThreads;  // 8 x 16 B per thread
#pragma unroll
    for (int it = 0; it < kPer; ++it) {
      const int e = gtid + it * kR1GroupThreads;
      const int b = e / (dh / 4), x4 = e % (dh / 4);
      const int i = t * kRouteTile + b;
      const bool ok = t < p.ntiles && i < p.blocks;
      sm100::cp_async16_zfill(dst + b * ckld + x4 * 4,
                              p.ck + ((int64_t)(ok ? i : 0) * p.Hkv + kvh) * dh + x4 * 4, ok ? 16u : 0u);
    }
    sm100::cp_async_commit();
  };
  int t = 2 * blockIdx.x + grp;
  issue_tile(t, cks0);  // in flight while the q rows are converted
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
  __syncthreads();
  // diagnostics: group leader stamps [16 + 8 grp + ...]: prologue, then per tile (mma, epilogue)
  unsigned long long* tg = trc != nullptr && gtid == 0 ? trc + 16 + 16 * grp : nullptr;
  tstamp_any(tg, 0);
  // tile-invariant epilogue constants: tile t starts at selection block t d
  // (l_sel == 64 == tile width), so the overlap weights of this thread's two
  // blocks with the warp's kW selection blocks do not depend on t
  const int gshift = __ffs(p.G) - 1;  // G is a power of two (host-checked)
  __shared__ double s_wgt[8][4][2][kW];  // [warp][lane column][block][selection block]
  if (grp == 0)
    for (int e = lane; e < 4 * 2 * kW; e += 32) {
      const int c4 = e / (2 * kW), c = (e / kW) % 2, k = e % kW;
      s_wgt[warp][c4][c][k] = (double)overlap(8 * warp + 2 * c4 + c, (8 * warp * d) / l_sel + k, d, l, l_sel);
    }
  __syncthreads();
  const double (*wgt)[kW] = s_wgt[warp][lc];
  int mvis_mt[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
    mvis_mt[mt] = 8 * mt + lr < nrows ? p.slot_mvis[(r0 + 8 * mt + lr) >> gshift] : 0;
  int tile_no = 0;
  for (int par = 0; t < p.ntiles; t += vstride, par ^= 1, ++tile_no) {
    double (*rm)[8] = reinterpret_cast<double (*)[8]>(smem + L::red_m) + grp * kRows;
    double (*rs)[8] = reinterpret_cast<double (*)[8]>(smem + L::red_s) + grp * kRows;
    double (*gp)[8][kW] =
        reinterpret_cast<double (*)[8][kW]>(smem + L::gpart) + grp * kRows;
    const float* cks = cks0 + (tile_no & 1) * kRouteTile * ckld;
    issue_tile(t + vstride, cks0 + ((tile_no + 1) & 1) * kRouteTile * ckld);  // lands meanwhile
    sm100::cp_async_wait<1>();  // this thread's copies of the current tile are done
    sm100::named_bar_sync(gbar, kR1GroupThreads);  // ... and every thread's
    // stagger: group 1 starts its first MMAs when group 0 is done with its
    // own, so from then on one group's epilogue overlaps the other's MMAs
    if (tile_no == 0 && grp == 1 && 2 * blockIdx.x < p.ntiles) sm100::named_bar_sync(5, kR1Threads);
    const int i0 = t * kRouteTile;
    double acc[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    // B fragment: block (8 warp + lr), element 4 s + lc; A: row (8 mt + lr), element 4 s + lc
    const float* kb = cks + (8 * warp + lr) * ckld + lc;
    const double* qa = qd + (size_t)lr * qld + lc;
    // all MT row tiles unconditionally (rows past nrows are zero in smem and
    // masked in the epilogue): no predicates, so the A loads of a k step are
    // all issued before its MMAs instead of one load-use pair at a time
#pragma unroll 2
    for (int s = 0; s < dh / 4; ++s) {
      const double b = kb[4 * s];
      double a[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = qa[(size_t)mt * 8 * qld + 4 * s];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) dmma_8x8x4(acc[mt], a[mt], b);
    }
    // C fragment: row 8 mt + lr, blocks 8 warp + 2 lc + {0, 1}
    const int blk = i0 + 8 * warp + 2 * lc;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt >= nmt) break;
      const int r = 8 * mt + lr;
      double mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        acc[mt][c] = __dmul_rn(acc[mt][c], p.scale);
        if (blk + c < mvis_mt[mt]) mx = fmax(mx, acc[mt][c]);
      }
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      if (lc == 0) rm[r][warp] = mx;
    }
    if (tile_no == 0 && grp == 0 && 2 * blockIdx.x + 1 < p.ntiles) sm100::named_bar_arrive(5, kR1Threads);
    sm100::named_bar_sync(gbar, kR1GroupThreads);  // also: every warp is done reading cks
    if (tile_no < 3) tstamp_any(tg, 1 + 5 * tile_no);
    if (tile_no < 3) tstamp_any(tg, 2 + 5 * tile_no);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt >= nmt) break;
      const int r = 8 * mt + lr;
      double mx = rm[r][0];
#pragma unroll
      for (int w = 1; w < 8; ++w) mx = fmax(mx, rm[r][w]);
      double sum = 0.0, g[kW];
#pragma unroll
      for (int k = 0; k < kW; ++k) g[k] = 0.0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double ev = blk + c < mvis_mt[mt] ? exp(acc[mt][c] - mx) : 0.0;
        sum += ev;
#pragma unroll
        for (int k = 0; k < kW; ++k) g[k] += ev * wgt[c][k];
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, off);
#pragma unroll
        for (int k = 0; k < kW; ++k) g[k] += __shfl_xor_sync(0xffffffffu, g[k], off);
      }
      if (lc == 0) {
        rs[r][warp] = sum;
#pragma unroll
        for (int k = 0; k < kW; ++k) gp[r][warp][k] = g[k];
      }
    }
    if (tile_no < 3) tstamp_any(tg, 3 + 5 * tile_no);
    sm100::named_bar_sync(gbar, kR1GroupThreads);
    if (gtid < nrows) {
      const int rr = r0 + gtid;
      const int64_t row = (int64_t)(rr >> gshift) * p.Hq + kvh * p.G + (rr & (p.G - 1));
      double mx = rm[gtid][0], sm = 0.0;
#pragma unroll
      for (int w = 1; w < 8; ++w) mx = fmax(mx, rm[gtid][w]);
#pragma unroll
      for (int w = 0; w < 8; ++w) sm += rs[gtid][w];
      p.TM[row * p.ntiles + t] = mx;
      p.TD[row * p.ntiles + t] = sm;
    }
    if (tile_no < 3) tstamp_any(tg, 4 + 5 * tile_no);
    // G[slot][t][h][j] for the selection blocks t d + j the tile touches (lane
    // j < g_stride <= 32), summed over the 8 warps in ascending order
    if (lane < p.g_stride) {
      for (int r = warp; r < nrows; r += 8) {
        const int rr = r0 + r;
        const int slot = rr >> gshift, h = kvh * p.G + (rr & (p.G - 1));
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const int k = lane - (8 * w * d) / l_sel;
          if (k >= 0 && k < kW) v += gp[r][w][k];
        }
        p.gsh[(((int64_t)slot * p.ntiles + t) * p.Hq + h) * p.g_stride + lane] = v;
      }
    }
    if (tile_no < 3) tstamp_any(tg, 5 + 5 * tile_no);
    sm100::named_bar_sync(gbar, kR1GroupThreads);  // red_* / gpart are rewritten by the next tile
  }
}

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
                           int32_t* count, uint32_t* forced_bits, unsigned long long* tr = nullptr) {
  __shared__ double wbest_s[32];
  __shared__ int wbest_i[32];
  __shared__ double lb_s;
  __shared__ int lb_i, nsurv;
  __shared__ int picks[64];
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;  // whole CTA
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
    tstamp(tr, 9);
    if (warp == 0) {  // K-th best warp maximum (rank counting among <= 32)
      const double ms = lane < nwarps ? wbest_s[lane] : -INFINITY;
      const int mi = lane < nwarps ? wbest_i[lane] : 0x7fffffff;
      int rank = 0;
      for (int o = 0; o < nwarps; ++o) rank += ranks_before(wbest_s[o], wbest_i[o], ms, mi) ? 1 : 0;
      const int kk = want <= nwarps ? want - 1 : -1;
      if (kk >= 0 && lane < nwarps && rank == kk && ms != -INFINITY) { lb_s = ms; lb_i = mi; }
    }
    __syncthreads();
    tstamp(tr, 10);
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
    tstamp(tr, 11);
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
  tstamp(tr, 12);
  if (warp == 0) {  // ascending order by a parallel rank-and-scatter (block ids are distinct)
    __shared__ uint32_t fbits;
    const int cnt = target > 0 ? target : 0;
    if (lane == 0) {
      fbits = 0u;
      if (avail > 0) {
        int c = 0;
        picks[c++] = 0;
        if (f1 > 0) picks[c++] = f1;
        if (f2 > 0 && f2 != f1) picks[c++] = f2;
      }
    }
    __syncwarp();
    for (int a = lane; a < cnt; a += 32) {
      const int v = picks[a];
      int rank = 0;
      for (int o = 0; o < cnt; ++o) rank += picks[o] < v ? 1 : 0;
      idx_row[rank] = v;
      if ((v == 0 || v == f1 || v == f2) && rank < 32) atomicOr(&fbits, 1u << rank);
    }
    for (int a = cnt + lane; a < n; a += 32) idx_row[a] = -1;
    __syncwarp();
    if (lane == 0) {
      *count = cnt;
      *forced_bits = fbits;
    }
  }
}



// Phase 2 (every CTA, after all tile statistics are out).  For each of the
// CTA's rows: M = max_t TM, DEN = sum_t TD e^(TM - M) (warp per row, the
// row's statistics in registers) and F_t = e^(TM_t - M) / DEN for the CTA's
// own tiles.  Then for each (slot of the chunk, own tile, j):
// part[slot][kvh][t][j] = sum_g (ascending) F[slot, g][t] G[slot][t][g][j] --
// the KV head's share of the tile's selection-block scores.
__device__ __noinline__ void shares_phase(const RouteParams& p, uint8_t* smem, unsigned long long* tr) {
  // Runs once per launch, so it is bound by instruction fetch unless small:
  // every global read is a fire-and-forget cp.async into shared memory
  // (one round trip per stage), the arithmetic runs from there.
  const int kvh = blockIdx.y;
  const int r0 = blockIdx.z * p.chunk_rows;
  const int nrows = min(p.chunk_rows, p.nr * p.G - r0);
  const int tid = threadIdx.x;
  const int vstride = 2 * gridDim.x;
  const int t0 = 2 * blockIdx.x;  // own tiles: t0 + {0, 1} + m vstride
  const int nt = p.ntiles, G = p.G, gs = p.g_stride;
  const int ct = nt > t0 ? 2 * ((nt - t0 + vstride - 1) / vstride) : 0;
  double* sF = reinterpret_cast<double*>(smem);  // [chunk_rows][ct]
  double* sMD = sF + p.chunk_rows * ct;          // [chunk_rows][2]: M, DEN
  double* sT = sMD + 2 * p.chunk_rows;           // staging
  // statistics, rg rows at a time: M, DEN per row (8 lanes per row), F for own tiles
  const int rg = min(nrows, p.shares_rows);
  for (int g0 = 0; g0 < nrows; g0 += rg) {
    const int gn = min(rg, nrows - g0);
    __syncthreads();
    for (int e = tid; e < gn * nt; e += kR1Threads) {
      const int rr = r0 + g0 + e / nt;
      const int64_t src = ((int64_t)(rr / G) * p.Hq + kvh * G + rr % G) * nt + e % nt;
      sm100::cp_async8(sT + 2 * e, p.TM + src);
      sm100::cp_async8(sT + 2 * e + 1, p.TD + src);
    }
    sm100::cp_async_wait_all();
    __syncthreads();
    constexpr int kL = 8;
    for (int rb = 0; rb < gn; rb += kR1Threads / kL) {  // CTA-uniform rounds
      const int r = min(rb + tid / kL, gn - 1), l8 = tid % kL;
      const double* st = sT + 2 * r * nt;
      double mx = -INFINITY, den = 0.0;
      for (int t = l8; t < nt; t += kL) mx = fmax(mx, st[2 * t]);
#pragma unroll
      for (int off = kL / 2; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      for (int t = l8; t < nt; t += kL)
        if (st[2 * t + 1] > 0.0) den += st[2 * t + 1] * exp(st[2 * t] - mx);
#pragma unroll
      for (int off = kL / 2; off >= 1; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
      if (l8 == 0) {
        sMD[2 * (g0 + r)] = mx;
        sMD[2 * (g0 + r) + 1] = den;
      }
    }
    __syncthreads();
    for (int e = tid; e < gn * ct; e += kR1Threads) {
      const int r = e / ct, k = e % ct;
      const int t = t0 + (k >> 1) * vstride + (k & 1);
      const double mx = sMD[2 * (g0 + r)], den = sMD[2 * (g0 + r) + 1];
      const double tm = t < nt ? sT[2 * (r * nt + t)] : -INFINITY;
      sF[(g0 + r) * ct + k] = (den > 0.0 && tm != -INFINITY) ? exp(tm - mx) / den : 0.0;
    }
  }
  tstamp(tr, 13);
  // shares of the KV group for own tiles, kc own tiles at a time:
  // part[slot][kvh][t][j] = sum_g (ascending) F[slot, g][t] G[slot][t][kvh G + g][j]
  const int nslots = nrows / G;
  const int kc = max(1, min(ct, p.shares_rows * 2 * nt / max(1, nslots * G * gs)));
  for (int k0 = 0; k0 < ct; k0 += kc) {
    const int kn = min(kc, ct - k0);
    __syncthreads();
    for (int e = tid; e < nslots * kn * G * gs; e += kR1Threads) {
      const int sk = e / (G * gs), rem = e % (G * gs);
      const int sl = sk / kn, k = k0 + sk % kn;
      const int t = min(t0 + (k >> 1) * vstride + (k & 1), nt - 1);
      sm100::cp_async8(sT + e, p.gsh + (((int64_t)(r0 / G + sl) * nt + t) * p.Hq + kvh * G) * gs + rem);
    }
    sm100::cp_async_wait_all();
    __syncthreads();
    for (int e = tid; e < nslots * kn * gs; e += kR1Threads) {
      const int sk = e / gs, j = e % gs;
      const int sl = sk / kn, k = k0 + sk % kn;
      const int t = t0 + (k >> 1) * vstride + (k & 1);
      if (t >= nt) continue;
      const double* gsm = sT + (size_t)sk * G * gs + j;
      double v = 0.0;
      for (int g = 0; g < G; ++g) v += sF[(sl * G + g) * ct + k] * gsm[g * gs];
      p.part[(((int64_t)(r0 / G + sl) * p.Hkv + kvh) * nt + t) * gs + j] = v;
    }
  }
}

// Phase 3 for one routed slot (whole CTA): score_b = sum_t (ascending) sum_kvh
// (ascending) part[kvh][t][b - t step] / (Hq l), then Top-n.  The slot's
// shares are staged tc tiles at a time with cp.async (one round trip each).
__device__ __noinline__ void slot_tail(const RouteParams& p, int slot, uint8_t* smem,
                                       double* scores_out, unsigned long long* tr = nullptr) {
  const int tid = threadIdx.x;
  const int avail = p.slot_avail[slot];
  double* sel = reinterpret_cast<double*>(smem);        // [kMaxAvail]
  int* surv = reinterpret_cast<int*>(sel + kMaxAvail);  // [kMaxAvail]
  double* st = reinterpret_cast<double*>(surv + kMaxAvail);  // [Hkv][tc][gs]
  const int nt = p.ntiles, gs = p.g_stride, hkv = p.Hkv;
  const int step = kRouteTile * p.d / p.l_sel;  // first selection block of tile t = t step
  const int tc = max(1, min(nt, p.tail_stage / (hkv * gs)));
  __syncthreads();  // smem reuse across slots
  for (int b = tid; b < avail; b += blockDim.x) sel[b] = 0.0;
  for (int tb = 0; tb < nt; tb += tc) {
    const int tn = min(tc, nt - tb);
    __syncthreads();
    for (int e = tid; e < hkv * tn * gs; e += blockDim.x) {
      const int kv = e / (tn * gs), rem = e % (tn * gs);
      sm100::cp_async8(st + e, p.part + (((int64_t)slot * hkv + kv) * nt + tb) * gs + rem);
    }
    sm100::cp_async_wait_all();
    __syncthreads();
    const int b_hi = min(avail, (tb + tn - 1) * step + gs);
    for (int b = tb * step + tid; b < b_hi; b += blockDim.x) {
      double v = sel[b];
      for (int t = max(tb, (b - gs + step) / step); t <= min(tb + tn - 1, b / step); ++t)
        for (int kv = 0; kv < hkv; ++kv) v += st[(kv * tn + t - tb) * gs + b - t * step];
      sel[b] = v;
    }
  }
  __syncthreads();
  const double scale = 1.0 / ((double)p.Hq * (double)p.l);
  for (int b = tid; b < avail; b += blockDim.x) {
    sel[b] *= scale;
    if (scores_out != nullptr) scores_out[b] = sel[b];
  }
  __syncthreads();
  tstamp(tr, 8);
  if (scores_out != nullptr) return;
  const int q = p.slot_q[slot];
  topn_write(sel, surv, avail, p.n, p.idx + (int64_t)q * p.n, p.idx_count + q, p.idx_forced + q, tr);
}

__device__ __forceinline__ void arrive(int* w) {
  __syncthreads();
  if (threadIdx.x == 0) sm100::red_add_release_gpu(w, 1);
}
__device__ __forceinline__ void wait_all(int* w, int n) {
  if (threadIdx.x == 0)
    while (sm100::ld_acquire_gpu(w) < n) {
    }
  __syncthreads();
}

template <int MT>
__global__ void __launch_bounds__(kR1Threads, 1)
    route_fused_kernel(const __grid_constant__ RouteParams p, double* scores_out, int scores_slot) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int nctas = gridDim.x * gridDim.y * gridDim.z;
  int* bar = p.counters;  // [0] tiles done, [1] shares done, [2] tail CTAs done; all return to 0
  unsigned long long* tr =
      p.trace != nullptr && threadIdx.x == 0 ? p.trace + kRouteTraceBase + cta * 16 * 4 : nullptr;
  auto stamp = [&](int k) {
    if (tr != nullptr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tr[k] = t;
    }
  };
  stamp(0);
  if (tr != nullptr) tr[14] = clock64();
  if (p.ntiles > 0) {
    tiles_phase<MT>(p, smem, p.trace != nullptr ? p.trace + kRouteTraceBase + cta * 16 * 4 : nullptr);
    stamp(1);
    arrive(bar);
    wait_all(bar, nctas);
    stamp(2);
    shares_phase(p, smem, tr);
    stamp(3);
  }
  const int ntail = scores_out != nullptr ? 1 : p.nr;
  arrive(bar + 1);
  if (cta >= ntail) return;  // no tail work: leave without waiting
  wait_all(bar + 1, nctas);
  stamp(4);
  if (cta == 0 && scores_out == nullptr) {
    for (int u = threadIdx.x; u < p.n_unrouted; u += blockDim.x) {
      const int q = p.unrouted[u];
      p.idx_count[q] = -1;
      p.idx_forced[q] = 0u;
      for (int a = 0; a < p.n; ++a) p.idx[(int64_t)q * p.n + a] = -1;
    }
  }
  for (int slot = cta; slot < ntail; slot += nctas)
    slot_tail(p, scores_out != nullptr ? scores_slot : slot, smem, scores_out,
              threadIdx.x == 0 ? tr : nullptr);
  stamp(5);
  if (tr != nullptr) tr[15] = clock64();
  __syncthreads();
  if (threadIdx.x == 0) {  // the last tail CTA resets the words for the next launch
    const int tail_ctas = min(ntail, nctas);
    if (sm100::atom_add_acq_rel_gpu(bar + 2, 1) == tail_ctas - 1) {
      atomicExch(bar, 0);
      atomicExch(bar + 1, 0);
      atomicExch(bar + 2, 0);
    }
  }
}

__global__ void __launch_bounds__(1024)
    select_only_kernel(const double* scores, int avail, int n, int32_t* idx, int32_t* count,
                       uint32_t* forced) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* sel = reinterpret_cast<double*>(smem);
  int* surv = reinterpret_cast<int*>(sel + kMaxAvail);
  for (int b = threadIdx.x; b < avail; b += blockDim.x) sel[b] = scores[b];
  __syncthreads();
  topn_write(sel, surv, avail, n, idx, count, forced);
}

template <int MT>
cudaError_t launch_fused(const RouteParams& p, double* scores_out, int scores_slot,
                         cudaStream_t s) {
  constexpr int kRows = 8 * MT;
  RouteParams pc = p;
  pc.chunk_rows = (kRows / p.G) * p.G;  // whole slots per row chunk (G <= kRows)
  const int rows_total = p.nr * p.G;
  const int rchunks = (rows_total + pc.chunk_rows - 1) / pc.chunk_rows;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // CTAs per (KV head, row chunk): as many as fit one wave (each CTA takes
  // two tiles per round), trimmed so every CTA runs the same number of rounds
  const int max_ctas = std::max(1, std::min((p.ntiles + 1) / 2, sms / (p.Hkv * rchunks)));
  const int per = std::max(1, (p.ntiles + 2 * max_ctas - 1) / (2 * max_ctas));
  const int ctas = std::max(1, (p.ntiles + 2 * per - 1) / (2 * per));
  if (ctas * p.Hkv * rchunks > sms) return cudaErrorInvalidConfiguration;  // not co-resident
  // shares phase: F [rows][2 per] + M/DEN [rows][2] + staged statistics [rg][2][ntiles]
  const size_t fixed = ((size_t)pc.chunk_rows * (2 * per + 2)) * sizeof(double);
  const size_t budget = 200 * 1024;
  pc.shares_rows = (int)std::max<size_t>(
      1, std::min<size_t>(pc.chunk_rows, (budget - fixed) / (2 * sizeof(double) * std::max(p.ntiles, 1))));
  const size_t shares_smem = fixed + (size_t)pc.shares_rows * 2 * p.ntiles * sizeof(double);
  pc.tail_stage = (int)(96 * 1024 / sizeof(double));  // staged shares per tail round, doubles
  const size_t smem =
      std::max({TileSmem<MT>::bytes, kTopnSmem + (size_t)pc.tail_stage * sizeof(double), shares_smem});
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = route_fused_kernel<MT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&pc, &scores_out, &scores_slot};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(ctas, p.Hkv, rchunks),
                                     dim3(kR1Threads), args, smem, s);
}

cudaError_t launch_chain(const RouteParams& p, double* scores_out, int scores_slot,
                         cudaStream_t s) {
  const int rows = p.nr * p.G;
  return (rows <= 16 && p.G <= 16) ? launch_fused<2>(p, scores_out, scores_slot, s)
         : rows <= 32               ? launch_fused<4>(p, scores_out, scores_slot, s)
         : (rows <= 40 && p.G <= 8) ? launch_fused<5>(p, scores_out, scores_slot, s)
                                    : launch_fused<6>(p, scores_out, scores_slot, s);
}

}  // namespace

cudaError_t launch_route(const RouteParams& p, cudaStream_t s, bool write_idx) {
  (void)write_idx;
  return launch_chain(p, nullptr, -1, s);
}

cudaError_t launch_scores_only(const RouteParams& p, double* scores, int slot, cudaStream_t s) {
  return launch_chain(p, scores, slot, s);
}

cudaError_t launch_select(const double* scores, int avail, int n, int32_t* idx, int32_t* count,
                          uint32_t* forced, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(select_only_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTopnSmem);
  if (e != cudaSuccess) return e;
  select_only_kernel<<<1, 1024, kTopnSmem, s>>>(scores, avail, n, idx, count, forced);
  return cudaGetLastError();
}

}  // namespace specsv_b200
