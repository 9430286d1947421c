// route.cu -- refresh-layer routing on sm_100a: fp64 compressed-block scores
// and Top-n block selection with forced blocks.
//
// Replaces nsa::selection_scores + nsa::select_blocks
// (src/nsa_attention.cpp:38-136) for every query that constructs indices.
//
// One cooperative persistent kernel (one 448-thread CTA per SM, two work
// items in flight), two phases and a single grid-wide arrival barrier:
//  1. tiles (all CTAs).  Work item = (KV head, <= 40 (query, head) rows, 7
//     statistics tiles of 16 compressed blocks).  Warp (item, t) owns all 40
//     rows x tile t and stages its own 16 key rows (cp.async):
//     logit = dot(q_h, ck_i) / sqrt(dh) in fp64 on the FP64 tensor pipe (DMMA
//     m8n8k4; fp32 x fp32 products are exact in fp64).  The key rows are
//     permuted in shared memory so that lane column c of the MMA fragment
//     holds the consecutive blocks 4c .. 4c + 3 of the tile: the whole per-row
//     epilogue stays inside the warp (no cross-warp reductions).  Per row and
//     tile it writes TM = max logit and, through a second small DMMA against
//     the tile-invariant overlap matrix W[block][selection block] (plus a
//     ones column), TD = sum e^(logit - TM) and G[b] = sum_i overlap(i, b)
//     e^(logit_i - TM): the tile's share of selection block b before the
//     softmax normalisation is known, so no per-block probability reaches HBM.
//  2. units (one CTA per (routed query, KV head)): per head M = max_t TM,
//     DEN = sum_t TD e^(TM - M), F_t = e^(TM_t - M) / DEN and the KV head's
//     share of every selection-block score; the query's last unit sums the
//     shares, score_b = sum_kvh sum_t sum_g F G / (Hq l)  (= the reference's
//     sum over blocks and heads of p_hi * overlap / l, nsa_attention.cpp:52-78,
//     regrouped -- contract P3), then Top-n: forced {0, avail-2, avail-1} plus the best remaining by
//     (score desc, id asc), written ascending (nsa_attention.cpp:94-136).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <utility>
#include <cstdint>

#include "attend.h"
#include "sm100.cuh"

namespace specsv_b200 {
namespace {

constexpr int kMT = 5;                    // 8-row m-tiles per row chunk (40 rows)
constexpr int kTB = kRouteTile;           // compressed blocks per statistics tile (16)
constexpr int kTilesPerItem = 7;          // statistics tiles per work item: at 64K, 8 heads x
                                          // 37 items fill 148 SMs twice exactly
constexpr int kSuper = kTB * kTilesPerItem;  // compressed blocks per work item
constexpr int kItemsPerRound = 2;         // items multiplied concurrently by one CTA: a warp's
                                          // DMMA chain is latency-bound, so more warps per SM
constexpr int kRouteThreads = 32 * kTilesPerItem * kItemsPerRound;  // warp = (item, tile)
constexpr int kDhRoute = 128;             // d_head of this build (host-checked)
constexpr int kLd = kDhRoute + 4;         // fp64 q row stride (== 4 mod 16: conflict-free fragments)
constexpr int kCkLd = kDhRoute + 4;       // fp32 key row stride (== 4 mod 32: conflict-free fragments)
constexpr int kWLd = 12;                  // overlap-matrix row stride, doubles (== 4 mod 8)
constexpr int kWCols = 8;                 // overlap matrix columns: g_stride + the ones column <= 8
constexpr size_t kTopnSmem = (size_t)kMaxAvail * 8 + (size_t)kMaxAvail * 4;
constexpr size_t kUnitSmem = 150 * 1024;  // phase-2 staging (see slot_unit)
constexpr size_t kTailSmem = kTopnSmem;
static_assert(kTB == 16, "lane column c of the MMA fragment owns blocks 4c .. 4c + 3");

#ifndef ROUTE_UNROLL
#define ROUTE_UNROLL 2
#endif
constexpr int kRouteUnroll = ROUTE_UNROLL;  // k steps of the logit loop unrolled

struct TileSmem {
  static constexpr size_t q = 0;                                           // [2][40][kLd] f64
  static constexpr size_t ck = q + (size_t)kItemsPerRound * 8 * kMT * kLd * 8;  // [2][kSuper][kCkLd] f32
  static constexpr size_t w = ck + (size_t)kItemsPerRound * kSuper * kCkLd * 4;  // [16][kWLd] f64
  static constexpr size_t bytes = w + (size_t)kTB * kWLd * 8;
  static_assert(bytes <= 227 * 1024, "tile-phase shared memory");
};

// (not volatile: a pure function of its operands, so the compiler may hoist the
// next k step's fragment loads above it)
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void tstamp(unsigned long long* tr, int k) {
  if (tr != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[k] = t;
  }
}

// e^x for x <= 0 (x = logit - tile max), ~2 ulp: x = n ln2 + r, |r| <= ln2/2,
// Taylor to degree 12 (truncation < 2e-16 relative), scaled by 2^n through the
// exponent bits.  x < -708 (including -inf) flushes to 0.
__device__ __forceinline__ double exp_nonpos(double x) {
  if (!(x >= -708.0)) return 0.0;
  const double n = rint(x * 1.4426950408889634);
  double r = fma(n, -6.93147180369123816490e-01, x);
  r = fma(n, -1.90821492927058770002e-10, r);
  double p = 2.08767569878680989792e-09;  // 1/12!
  p = fma(p, r, 2.50521083854417187751e-08);
  p = fma(p, r, 2.75573192239858906526e-07);
  p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05);
  p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03);
  p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02);
  p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return __hiloint2double(__double2hiint(p) + (static_cast<int>(n) << 20), __double2loint(p));
}

// tokens shared by compressed block i ([i d, i d + l)) and selection block b
__device__ __forceinline__ int overlap(int i, int b, int d, int l, int l_sel) {
  const int lo = max(i * d, b * l_sel), hi = min(i * d + l, (b + 1) * l_sel);
  return hi > lo ? hi - lo : 0;
}

// shared-memory key row of tile-local block i (0..15): MMA n-tile nt, column
// n holds block 4 (n / 2) + 2 nt + n % 2, so C-fragment lane column c covers
// the consecutive blocks [4 c, 4 c + 4)
__device__ __forceinline__ int perm_row(int i) {
  return 8 * ((i >> 1) & 1) + 2 * (i >> 2) + (i & 1);
}

// Phase 1.  A work item is rows [r0, r0 + nrows) of KV head kvh x the 112
// compressed blocks of super tile st (7 statistics tiles of 16 blocks); a
// CTA multiplies two items at once, warp (item, w) owning tile w of its item
// for all 40 rows: per k step 5 A + 2 B fragment loads feed 10 DMMAs.  q is
// staged in fp64 (converted once); the keys are staged in fp32 by
// fire-and-forget cp.async and converted per B fragment (2 per 10 DMMAs).
struct Item {
  int kvh, r0, nrows, st;
  bool live;
};

__device__ __forceinline__ Item item_of(const RouteParams& p, int it, int items) {
  const int rows_total = p.nr * p.G;
  const int nst = (p.ntiles + kTilesPerItem - 1) / kTilesPerItem;
  const int rest = it / nst;
  Item I;
  I.live = it < items;
  I.st = it % nst;
  I.kvh = rest % p.Hkv;
  I.r0 = (rest / p.Hkv) * p.chunk_rows;
  I.nrows = I.live ? min(p.chunk_rows, rows_total - I.r0) : 0;
  return I;
}

// Staging of one round, per warp: the warp copies its own tile's 16 key rows
// (permuted, see perm_row) by fire-and-forget cp.async, the item's 7 warps
// convert its q rows to fp64 and meet at the item's named barrier, then each
// warp waits only for its own copies -- a warp starts as soon as its tile
// has landed.
__device__ void stage_tile(const RouteParams& p, uint8_t* smem, const Item& I, int k) {
  constexpr int dh = kDhRoute;
  double* qs = reinterpret_cast<double*>(smem + TileSmem::q) + (size_t)k * 8 * kMT * kLd;
  float* cks = reinterpret_cast<float*>(smem + TileSmem::ck) + (size_t)k * kSuper * kCkLd;
  const int wt = (threadIdx.x >> 5) % kTilesPerItem, lane = threadIdx.x & 31;
  const int it_tid = threadIdx.x % (32 * kTilesPerItem);
#pragma unroll 4
  for (int e = lane; e < kTB * (dh / 4); e += 32) {  // this warp's 16 key rows
    const int b = wt * kTB + e / (dh / 4), x4 = e % (dh / 4);
    const int i = I.st * kSuper + b;
    const bool ok = I.live && i < p.blocks;
    sm100::cp_async16_zfill(cks + (size_t)(wt * kTB + perm_row(b & (kTB - 1))) * kCkLd + x4 * 4,
                            p.ck + ((int64_t)(ok ? i : 0) * p.Hkv + I.kvh) * dh + x4 * 4, ok ? 16u : 0u);
  }
  sm100::cp_async_commit();
  constexpr int kQUnits = 8 * kMT * (dh / 4);
  constexpr int kQPer = (kQUnits + 32 * kTilesPerItem - 1) / (32 * kTilesPerItem);
  float4 v[kQPer];
#pragma unroll
  for (int u = 0; u < kQPer; ++u) {  // the item's q rows: all loads in flight, then fp64 stores
    const int e = it_tid + u * 32 * kTilesPerItem;
    v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e < kQUnits) {
      const int r = e / (dh / 4), x4 = e % (dh / 4);
      if (r < I.nrows) {
        const int rr = I.r0 + r;
        const int h = I.kvh * p.G + (rr & (p.G - 1));
#ifdef ROUTE_DIAG_NO_Q  // timing diagnostics only: no q loads
        v[u] = make_float4(1e-3f * x4, 1.f, 0.5f, -0.25f + h);
#else
        v[u] = __ldg(reinterpret_cast<const float4*>(p.q + ((int64_t)p.slot_q[rr / p.G] * p.Hq + h) * dh) + x4);
#endif
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kQPer; ++u) {
    const int e = it_tid + u * 32 * kTilesPerItem;
    if (e < kQUnits) {
      double* dst = qs + (e / (dh / 4)) * kLd + (e % (dh / 4)) * 4;
      reinterpret_cast<double2*>(dst)[0] = make_double2(v[u].x, v[u].y);
      reinterpret_cast<double2*>(dst)[1] = make_double2(v[u].z, v[u].w);
    }
  }
  sm100::named_bar_sync(1 + k, 32 * kTilesPerItem);  // the item's q rows are in place
  sm100::cp_async_wait<0>();
  __syncwarp();  // this warp's key rows are in place
}

// one warp's statistics tile of a staged item: logits for all rows, TM, TD, G
__device__ void tile_compute(const RouteParams& p, const uint8_t* smem, const Item& I, int k) {
  constexpr int dh = kDhRoute;
  const double* qs = reinterpret_cast<const double*>(smem + TileSmem::q) + (size_t)k * 8 * kMT * kLd;
  const float* cks = reinterpret_cast<const float*>(smem + TileSmem::ck) + (size_t)k * kSuper * kCkLd;
  const double* W = reinterpret_cast<const double*>(smem + TileSmem::w);
  const int wt = (threadIdx.x >> 5) % kTilesPerItem, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const int t = I.st * kTilesPerItem + wt;  // statistics tile
  const int nrows = I.nrows;
  if (!I.live || t >= p.ntiles) return;
  // ---- logits: 40 rows x 16 blocks, fp64 DMMA ----
  double acc[kMT][2][2];
#pragma unroll
  for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  const double* qa = qs + lr * kLd + lc;
  const float* kb = cks + (size_t)(wt * kTB + lr) * kCkLd + lc;
#ifdef ROUTE_DIAG_KSTEPS  // timing diagnostics only: fewer k steps
#define ROUTE_KS ROUTE_DIAG_KSTEPS
#else
#define ROUTE_KS (dh / 4)
#endif
#pragma unroll kRouteUnroll
  for (int s = 0; s < ROUTE_KS; ++s) {
    double a[kMT], b[2];
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt) a[mt] = qa[mt * 8 * kLd + 4 * s];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#ifdef ROUTE_DIAG_B_CONST  // timing diagnostics only (tools/route_variants.sh): no key loads
      b[nt] = 1.0 + 1e-3 * (nt + s);
#else
      b[nt] = kb[nt * 8 * kCkLd + 4 * s];  // fp32 -> fp64, exact
#endif
    }
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) dmma_8x8x4(acc[mt][nt], a[mt], b[nt]);
  }
  // ---- per row: max over the tile (lane column c holds blocks 4 c .. 4 c + 3),
  // e = exp(logit - max), then TD and G through e x W ----
  const int ib = t * kTB + 4 * lc;  // first block of this lane column
  const double* wl = W + lc * kWLd + lr;
  // every m-tile unconditionally (rows past nrows have mvis 0 and are not
  // stored): the 5 rows' exps and G chains are independent, so they interleave
  int mvis[kMT], slot[kMT];
  double mx[kMT];
#pragma unroll
  for (int mt = 0; mt < kMT; ++mt) {
    const int r = 8 * mt + lr;
    slot[mt] = (I.r0 + min(r, nrows - 1)) / p.G;
    mvis[mt] = r < nrows ? p.slot_mvis[slot[mt]] : 0;
    mx[mt] = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        acc[mt][nt][c] = __dmul_rn(acc[mt][nt][c], p.scale);
        if (ib + 2 * nt + c < mvis[mt]) mx[mt] = fmax(mx[mt], acc[mt][nt][c]);
      }
  }
#pragma unroll
  for (int mt = 0; mt < kMT; ++mt) {
    mx[mt] = fmax(mx[mt], __shfl_xor_sync(0xffffffffu, mx[mt], 1));
    mx[mt] = fmax(mx[mt], __shfl_xor_sync(0xffffffffu, mx[mt], 2));
  }
#pragma unroll
  for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#ifdef ROUTE_DIAG_NO_EXP  // timing diagnostics only
        acc[mt][nt][c] = ib + 2 * nt + c < mvis[mt] ? acc[mt][nt][c] - mx[mt] : 0.0;
#else
        acc[mt][nt][c] = ib + 2 * nt + c < mvis[mt] ? exp_nonpos(acc[mt][nt][c] - mx[mt]) : 0.0;
#endif
  // K chunk (nt, c) = blocks {4 k + 2 nt + c : k < 4}: exactly the value lane
  // column k holds, so the A fragment is the exp as it stands; W is stored
  // K-chunk-major (row 4 (2 nt + c) + k) for conflict-free B fragments
  double g[kMT][2];
#pragma unroll
  for (int mt = 0; mt < kMT; ++mt) g[mt][0] = g[mt][1] = 0.0;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double w = wl[4 * (2 * nt + c) * kWLd];
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt) dmma_8x8x4(g[mt], acc[mt][nt][c], w);
    }
#pragma unroll
  for (int mt = 0; mt < kMT; ++mt) {
    const int r = 8 * mt + lr;
    if (r >= nrows) continue;
    const int rr = I.r0 + r;
    const int h = I.kvh * p.G + (rr & (p.G - 1));
    const int64_t srow = ((int64_t)slot[mt] * p.Hq + h) * p.ntiles + t;
    const int64_t grow = ((int64_t)slot[mt] * p.ntiles + t) * p.Hq + h;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int j = 2 * lc + c;
      if (j < p.g_stride) p.gsh[grow * p.g_stride + j] = g[mt][c];
      if (j == p.g_stride) p.TD[srow] = g[mt][c];
    }
    if (lc == 0) p.TM[srow] = mx[mt];
  }
}

// (score desc, id asc): true when (sa, ia) ranks before (sb, ib)
__device__ __forceinline__ bool ranks_before(double sa, int ia, double sb, int ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// Top-n over sel[0, avail) (select_blocks, nsa_attention.cpp:94-136): forced
// blocks first, then the best remaining by (score desc, id asc).
//  1. the best candidate of every 4-lane group -> the K-th best of those is a
//     lower bound of the K-th best overall (K = picks needed <= groups);
//  2. candidates ranking at or before that bound survive (typically ~K);
//  3. exact rank among the survivors.
__device__ void topn_write(const double* sel, int* surv, int avail, int n, int32_t* idx_row,
                           int32_t* count, uint32_t* forced_bits, unsigned long long* tr = nullptr) {
  constexpr int kMaxGroups = 256;  // blockDim.x / 4 <= 256
  __shared__ double gbest_s[kMaxGroups];
  __shared__ int gbest_i[kMaxGroups];
  __shared__ double lb_s;
  __shared__ int lb_i, nsurv;
  __shared__ int picks[64];
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;  // whole CTA
  const int ngroups = nthr >> 2;
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
    lb_s = -INFINITY;  // no bound unless a group maximum holds rank K-1
    lb_i = 0x7fffffff;
  }
  if (want > 0) {
    // 1. per-group best over the group's candidates (b = tid + k nthr)
    double bs = -INFINITY;
    int bi = 0x7fffffff;
    for (int b = tid; b < avail; b += nthr) {
      double sc;
      if (cand(b, sc) && ranks_before(sc, b, bs, bi)) { bs = sc; bi = b; }
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ranks_before(os, oi, bs, bi)) { bs = os; bi = oi; }
    }
    if ((lane & 3) == 0) { gbest_s[tid >> 2] = bs; gbest_i[tid >> 2] = bi; }
    __syncthreads();
    tstamp(tr, 9);
    {  // the group maximum of rank K-1: group tid/4's rank among the groups,
       // counted by its 4 lanes (a quarter of the groups each) and combined
      const int g = tid >> 2, part = tid & 3;
      const double ms = gbest_s[g];
      const int mi = gbest_i[g];
      int rank = 0;
      for (int o = part; o < ngroups; o += 4) rank += ranks_before(gbest_s[o], gbest_i[o], ms, mi) ? 1 : 0;
      rank += __shfl_xor_sync(0xffffffffu, rank, 1);
      rank += __shfl_xor_sync(0xffffffffu, rank, 2);
      if (part == 0 && want <= ngroups && rank == want - 1 && ms != -INFINITY) { lb_s = ms; lb_i = mi; }
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

// Phase 2, one unit = (routed slot, KV head), whole CTA.  Per head g of the
// group (a warp each): M = max_t TM, E_t = e^(TM_t - M), DEN = sum_t TD_t
// E_t, F_t = E_t / DEN.  Then the KV head's share of every selection-block
// score, part[b] = sum_t (ascending) sum_g (ascending) F_gt G_gt[b - t step]
// over the <= 2 tiles touching b.  The last unit of a slot to finish sums the
// Hkv shares in ascending head order -- score_b = sum part / (Hq l), the
// reference's sum over blocks and heads regrouped (contract P3) -- and runs
// the Top-n.
__device__ __noinline__ void slot_unit(const RouteParams& p, int slot, int kvh, uint8_t* smem,
                                       double* scores_out, unsigned long long* tr) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int nthr = blockDim.x;
  const int avail = p.slot_avail[slot];
  const int nt = p.ntiles, gs = p.g_stride, G = p.G;
  const int step = kRouteTile * p.d / p.l_sel;  // first selection block of tile t = t step
  // smem: F [G][nt] | TM, TD staging [G][nt] each | G staging [tiles][G][gs]
  double* sF = reinterpret_cast<double*>(smem);
  double* sTM = sF + G * nt;
  double* sTD = sTM + G * nt;
  double* sG = sTD + G * nt;
  const int gbudget = (int)((150 * 1024) / sizeof(double)) - 3 * G * nt;  // doubles for G tiles
  const int tc = max(2, min(nt + 1, gbudget / (G * gs)));                 // staged tiles per round
  // one fire-and-forget batch (16-byte copies) for TM, TD and the first G round
  // (other CTAs' writes of this launch; this SM never read those lines)
  auto stage_g = [&](int Ts, int T1) {
    const int per = G * gs / 2;  // 16-byte units of one tile's group rows (G gs is even)
    for (int e = tid; e < (T1 - Ts) * per; e += nthr) {
      const int tt = e / per, rem = e % per;
      sm100::cp_async16_zfill(sG + (size_t)tt * G * gs + 2 * rem,
                              p.gsh + (((int64_t)slot * nt + Ts + tt) * p.Hq + kvh * G) * gs + 2 * rem, 16u);
    }
  };
  __syncthreads();  // smem reuse across units
  {
    const double* tm = p.TM + ((int64_t)slot * p.Hq + kvh * G) * nt;  // the group's rows are contiguous
    const double* td = p.TD + ((int64_t)slot * p.Hq + kvh * G) * nt;
    for (int e = tid; e < G * nt / 2; e += nthr) {
      sm100::cp_async16_zfill(sTM + 2 * e, tm + 2 * e, 16u);
      sm100::cp_async16_zfill(sTD + 2 * e, td + 2 * e, 16u);
    }
    sm100::cp_async_commit();  // group 1: TM, TD (the F pass below needs only these)
    stage_g(0, min(nt, tc - 1));
    sm100::cp_async_commit();  // group 2: the first round of G, landing under the F pass
  }
  sm100::cp_async_wait<1>();
  __syncthreads();
  tstamp(tr, 13);
  for (int g = warp; g < G; g += nwarps) {
    double mx = -INFINITY;
    for (int t = lane; t < nt; t += 32) mx = fmax(mx, sTM[g * nt + t]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    double den = 0.0;
    for (int t = lane; t < nt; t += 32) {
      const double tm = sTM[g * nt + t];
      const double e = tm == -INFINITY ? 0.0 : exp_nonpos(tm - mx);
      sF[g * nt + t] = e;
      den += sTD[g * nt + t] * e;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
    const double inv = den > 0.0 ? 1.0 / den : 0.0;
    for (int t = lane; t < nt; t += 32) sF[g * nt + t] *= inv;
  }
  tstamp(tr, 7);
  sm100::cp_async_wait<0>();  // this thread's G copies; the round's barrier publishes them all
  // part[b] over rounds of staged tiles: round [T0, T1) computes the blocks
  // [T0 step, T1 step) (the last round: up to avail), from tiles T0 - 1 .. T1 - 1
  // (tile T0 - 1 overhangs into block T0 step)
  double* part = p.part + ((int64_t)slot * p.Hkv + kvh) * p.sel_pad;
  for (int T0 = 0; T0 < nt; T0 += tc - 1) {
    const int T1 = min(nt, T0 + tc - 1);
    const int Ts = max(0, T0 - 1);
    if (T0 > 0) {  // later rounds (long contexts): stage this round's tiles
      __syncthreads();  // the previous round's readers are done
      stage_g(Ts, T1);
      sm100::cp_async_wait_all();
    }
    __syncthreads();  // F and the staged tiles are visible
    const int b_end = T1 == nt ? avail : min(avail, T1 * step);
    for (int b = T0 * step + tid; b < b_end; b += nthr) {
      const int t_lo = max(0, (b - gs + step) / step), t_hi = min(nt - 1, b / step);
      double v = 0.0;
      for (int t = t_lo; t <= t_hi; ++t) {
        const double* gp = sG + (size_t)(t - Ts) * G * gs + (b - t * step);
        for (int g = 0; g < G; ++g) v += sF[g * nt + t] * gp[g * gs];
      }
      part[b] = v;
    }
  }
  if (nt == 0)
    for (int b = tid; b < avail; b += nthr) part[b] = 0.0;
  // ---- the slot's last unit: scores and Top-n ----
  __shared__ int last;
  tstamp(tr, 14);
  __syncthreads();
  if (tid == 0) {
    // acq_rel: releases this CTA's part writes (ordered before thread 0 by the
    // barrier above, release is cumulative) and, in the last unit, acquires
    // every other unit's
    const int done = sm100::atom_add_acq_rel_gpu(p.slot_done + slot, 1);
    last = done == p.Hkv - 1;
    if (last) p.slot_done[slot] = 0;  // self-resetting; the kernel boundary publishes it
  }
  __syncthreads();
  tstamp(tr, 8);
  if (!last) return;
  double* sel = reinterpret_cast<double*>(smem);        // [kMaxAvail]
  int* surv = reinterpret_cast<int*>(sel + kMaxAvail);  // [kMaxAvail]
  const double scale = 1.0 / ((double)p.Hq * (double)p.l);
  const double* parts = p.part + (int64_t)slot * p.Hkv * p.sel_pad;
  for (int b4 = tid; 4 * b4 < avail; b4 += nthr) {  // 4 blocks per thread; sel_pad % 4 == 0
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    double2 pk[8][2];
#pragma unroll
    for (int kv = 0; kv < 8; ++kv)  // every head's loads in flight (other CTAs' data: L2)
      if (kv < p.Hkv) {
        const double2* src = reinterpret_cast<const double2*>(parts + (int64_t)kv * p.sel_pad) + 2 * b4;
        pk[kv][0] = __ldcg(src);
        pk[kv][1] = __ldcg(src + 1);
      }
#pragma unroll
    for (int kv = 0; kv < 8; ++kv)
      if (kv < p.Hkv) {
        v[0] += pk[kv][0].x;
        v[1] += pk[kv][0].y;
        v[2] += pk[kv][1].x;
        v[3] += pk[kv][1].y;
      }
    for (int kv = 8; kv < p.Hkv; ++kv) {
      const double2* src = reinterpret_cast<const double2*>(parts + (int64_t)kv * p.sel_pad) + 2 * b4;
      const double2 w0 = __ldcg(src), w1 = __ldcg(src + 1);
      v[0] += w0.x;
      v[1] += w0.y;
      v[2] += w1.x;
      v[3] += w1.y;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (4 * b4 + k < avail) {
        sel[4 * b4 + k] = v[k] * scale;
        if (scores_out != nullptr) scores_out[4 * b4 + k] = sel[4 * b4 + k];
      }
  }
  __syncthreads();
  tstamp(tr, 6);
  tstamp(tr, 15);
  if (scores_out != nullptr) return;
  const int q = p.slot_q[slot];
  topn_write(sel, surv, avail, p.n, p.idx + (int64_t)q * p.n, p.idx_count + q, p.idx_forced + q, tr);
}

__device__ __forceinline__ void griddep_wait_r() { sm100::griddep_wait(); }
__device__ __forceinline__ void griddep_launch_r() { sm100::griddep_launch(); }

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

__global__ void __launch_bounds__(kRouteThreads, 1)
    route_fused_kernel(const __grid_constant__ RouteParams p, double* scores_out, int scores_slot) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int cta = blockIdx.x, nctas = gridDim.x;
  int* bar = p.counters;  // [0] tiles done, [2] tail CTAs done; both return to 0
  unsigned long long* tr =
      p.trace != nullptr && threadIdx.x == 0 ? p.trace + kRouteTraceBase + cta * 16 * 4 : nullptr;
  griddep_wait_r();  // the inputs may come from the launch just before (PDL)
  tstamp(tr, 0);
  // ---- phase 1: work items (KV head, row chunk, tile set) over the grid ----
  if (p.ntiles > 0) {
    {  // tile-invariant overlap matrix (+ the ones column for TD), K-chunk-major rows
      double* W = reinterpret_cast<double*>(smem + TileSmem::w);
      for (int e = threadIdx.x; e < kTB * kWCols; e += kRouteThreads) {
        const int i = e / kWCols, j = e % kWCols;  // block i = 4 k + 2 nt + c -> row 4 (2 nt + c) + k
        const int wr = 4 * (i & 3) + (i >> 2);
        W[wr * kWLd + j] = j < p.g_stride ? (double)overlap(i, j, p.d, p.l, p.l_sel)
                                          : (j == p.g_stride ? 1.0 : 0.0);
      }
    }
    const int rows_total = p.nr * p.G;
    const int rchunks = (rows_total + p.chunk_rows - 1) / p.chunk_rows;
    const int items = p.Hkv * rchunks * ((p.ntiles + kTilesPerItem - 1) / kTilesPerItem);
    // item slot k (7 warps) runs items cta + (kItemsPerRound r + k) nctas on its
    // own barrier; with several rounds, slot 1 starts once slot 0's first
    // tiles are staged, so one slot's staging overlaps the other's DMMAs
    const int k = (threadIdx.x >> 5) / kTilesPerItem;
    const bool offset = cta + kItemsPerRound * nctas < items;  // slot 0 has a second round
    __syncthreads();  // the overlap matrix is in place
    if (offset && k == 1) sm100::named_bar_sync(5, kRouteThreads);
    for (int r = 0; cta + (kItemsPerRound * r + k) * nctas < items; ++r) {
      const Item I = item_of(p, cta + (kItemsPerRound * r + k) * nctas, items);
      if (r > 0) sm100::named_bar_sync(3 + k, 32 * kTilesPerItem);  // the slot's previous tiles are done
      if (r < 4) tstamp(tr, 32 + 3 * r);
      stage_tile(p, smem, I, k);
      if (offset && k == 0 && r == 0) sm100::named_bar_arrive(5, kRouteThreads);
      if (r < 4) tstamp(tr, 33 + 3 * r);
      tile_compute(p, smem, I, k);
      if (r < 4) tstamp(tr, 34 + 3 * r);
    }
    tstamp(tr, 1);
  }
  // ---- phase 2: (slot, KV head) units after every tile statistic is out ----
  const int nslots = scores_out != nullptr ? 1 : p.nr;
  const int units = nslots * p.Hkv;
  arrive(bar);
  if (cta >= units) return;  // no unit: leave without waiting
  wait_all(bar, nctas);
  griddep_launch_r();  // no more waiting on other CTAs: the next launch may start placing CTAs
  tstamp(tr, 4);
  if (cta == 0 && scores_out == nullptr) {
    for (int u = threadIdx.x; u < p.n_unrouted; u += blockDim.x) {
      const int q = p.unrouted[u];
      p.idx_count[q] = -1;
      p.idx_forced[q] = 0u;
      for (int a = 0; a < p.n; ++a) p.idx[(int64_t)q * p.n + a] = -1;
    }
  }
#ifdef ROUTE_DIAG_TAIL_TWICE  // timing diagnostics only: the trace then shows a warm second pass
  for (int u = cta; u < units; u += nctas)
    slot_unit(p, scores_out != nullptr ? scores_slot : u / p.Hkv, u % p.Hkv, smem, scores_out, nullptr);
  __syncthreads();
  arrive(bar + 1);
  wait_all(bar + 1, min(units, nctas));
  tstamp(tr, 4);
#endif
  for (int u = cta; u < units; u += nctas)
    slot_unit(p, scores_out != nullptr ? scores_slot : u / p.Hkv, u % p.Hkv, smem, scores_out, tr);
  tstamp(tr, 5);
  __syncthreads();
  if (threadIdx.x == 0) {  // the last unit CTA resets the barrier words for the next launch
    const int unit_ctas = min(units, nctas);
    if (sm100::atom_add_acq_rel_gpu(bar + 2, 1) == unit_ctas - 1) {
      atomicExch(bar, 0);
      atomicExch(bar + 2, 0);
#ifdef ROUTE_DIAG_TAIL_TWICE
      atomicExch(bar + 1, 0);
#endif
    }
  }
}

// Many requests' routing in one cooperative launch (specsv_nsa_verify_batched):
// the tile items of every request share the grid, then ONE grid barrier, then
// every request's (slot, KV head) units -- the per-launch tail and barrier are
// paid once per batch instead of once per request.  Request q uses its own
// workspace regions and counter set (RouteBatch built on the host).
__device__ __forceinline__ int batch_owner(const int32_t* start, int n_req, int i) {
  int q = 0;
  while (q + 1 < n_req && i >= start[q + 1]) ++q;
  return q;
}

__global__ void __launch_bounds__(kRouteThreads, 1)
    route_batch_kernel(const __grid_constant__ RouteBatch b) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int cta = blockIdx.x, nctas = gridDim.x;
  int* bar = b.req[0].counters;  // [0] tiles done, [2] tail CTAs done; both return to 0
  const int items = b.item_start[b.n_req];
  griddep_wait_r();
  if (items > 0) {
    const RouteParams& p0 = b.req[0];  // the overlap matrix is a function of the config only
    double* W = reinterpret_cast<double*>(smem + TileSmem::w);
    for (int e = threadIdx.x; e < kTB * kWCols; e += kRouteThreads) {
      const int i = e / kWCols, j = e % kWCols;
      const int wr = 4 * (i & 3) + (i >> 2);
      W[wr * kWLd + j] = j < p0.g_stride ? (double)overlap(i, j, p0.d, p0.l, p0.l_sel)
                                         : (j == p0.g_stride ? 1.0 : 0.0);
    }
    const int k = (threadIdx.x >> 5) / kTilesPerItem;  // item slot, as in route_fused_kernel
    const bool offset = cta + kItemsPerRound * nctas < items;
    __syncthreads();  // the overlap matrix is in place
    if (offset && k == 1) sm100::named_bar_sync(5, kRouteThreads);
    for (int r = 0; cta + (kItemsPerRound * r + k) * nctas < items; ++r) {
      const int it = cta + (kItemsPerRound * r + k) * nctas;
      const int q = batch_owner(b.item_start, b.n_req, it);
      const Item I = item_of(b.req[q], it - b.item_start[q], b.item_start[q + 1] - b.item_start[q]);
      if (r > 0) sm100::named_bar_sync(3 + k, 32 * kTilesPerItem);
      stage_tile(b.req[q], smem, I, k);
      if (offset && k == 0 && r == 0) sm100::named_bar_arrive(5, kRouteThreads);
      tile_compute(b.req[q], smem, I, k);
    }
  }
  const int units = b.unit_start[b.n_req];
  arrive(bar);
  if (cta >= units) return;  // no unit: leave without waiting
  wait_all(bar, nctas);
  griddep_launch_r();
  if (cta == 0) {
    for (int q = 0; q < b.n_req; ++q) {
      const RouteParams& p = b.req[q];
      for (int u = threadIdx.x; u < p.n_unrouted; u += blockDim.x) {
        const int qq = p.unrouted[u];
        p.idx_count[qq] = -1;
        p.idx_forced[qq] = 0u;
        for (int a = 0; a < p.n; ++a) p.idx[(int64_t)qq * p.n + a] = -1;
      }
    }
  }
  for (int u = cta; u < units; u += nctas) {
    const int q = batch_owner(b.unit_start, b.n_req, u);
    const RouteParams& p = b.req[q];
    const int lu = u - b.unit_start[q];
    slot_unit(p, lu / p.Hkv, lu % p.Hkv, smem, nullptr, nullptr);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // the last unit CTA resets the barrier words for the next launch
    const int unit_ctas = min(units, nctas);
    if (sm100::atom_add_acq_rel_gpu(bar + 2, 1) == unit_ctas - 1) {
      atomicExch(bar, 0);
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

// SM count of the current device, cached per device (a device constant; the
// cache is a per-device atomic, so concurrent callers on different devices or
// threads never see another device's value)
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& slot = cache[dev < 64 ? dev : 63];
  int sms = slot.load(std::memory_order_relaxed);
  if (sms == 0) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev < 64) slot.store(sms, std::memory_order_relaxed);
  }
  return sms;
}

// a cooperative launch (every CTA co-resident: grid barrier) that may also
// start early behind the previous launch (programmatic dependent launch)
template <typename... KArgs, typename... Args>
cudaError_t launch_coop_pdl(void (*kernel)(KArgs...), int ctas, int threads, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeCooperative;
  attr[na++].val.cooperative = 1;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

cudaError_t launch_chain(const RouteParams& p, double* scores_out, int scores_slot, cudaStream_t s) {
  RouteParams pc = p;
  pc.chunk_rows = (8 * kMT / p.G) * p.G;  // whole slots per row chunk (G <= 32 <= 40)
  if (pc.chunk_rows < 1) return cudaErrorInvalidValue;
  const int rows_total = p.nr * p.G;
  const int rchunks = (rows_total + pc.chunk_rows - 1) / pc.chunk_rows;
  const int sms = sm_count();
  const int items = p.Hkv * rchunks * ((p.ntiles + kTilesPerItem - 1) / kTilesPerItem);
  const int units = (scores_out != nullptr ? 1 : p.nr) * p.Hkv;
  const int ctas = std::min(sms, std::max(items, units));  // one CTA per SM: co-resident
  const size_t smem = std::max({TileSmem::bytes, kUnitSmem, kTailSmem});
  cudaError_t e = cudaFuncSetAttribute(route_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_coop_pdl(route_fused_kernel, ctas, kRouteThreads, smem, s, pc, scores_out, scores_slot);
}

}  // namespace

cudaError_t launch_route_batch(RouteBatch& b, cudaStream_t s) {
  const int sms = sm_count();
  b.item_start[0] = 0;
  b.unit_start[0] = 0;
  for (int q = 0; q < b.n_req; ++q) {
    RouteParams& p = b.req[q];
    p.chunk_rows = (8 * kMT / p.G) * p.G;
    if (p.chunk_rows < 1) return cudaErrorInvalidValue;
    const int rchunks = (p.nr * p.G + p.chunk_rows - 1) / p.chunk_rows;
    b.item_start[q + 1] = b.item_start[q] + p.Hkv * rchunks * ((p.ntiles + kTilesPerItem - 1) / kTilesPerItem);
    b.unit_start[q + 1] = b.unit_start[q] + p.nr * p.Hkv;
  }
  const int ctas = std::max(1, std::min(sms, std::max(b.item_start[b.n_req], b.unit_start[b.n_req])));
  const size_t smem = std::max({TileSmem::bytes, kUnitSmem, kTailSmem});
  cudaError_t e = cudaFuncSetAttribute(route_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_coop_pdl(route_batch_kernel, ctas, kRouteThreads, smem, s, b);
}

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
