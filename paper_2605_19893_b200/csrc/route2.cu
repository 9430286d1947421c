// route2.cu -- refresh-layer routing on sm_100a, single-request fast path:
// fp64 compressed-block selection scores and Top-n with forced blocks.
//
// Replaces nsa::selection_scores + nsa::select_blocks
// (src/nsa_attention.cpp:38-136) for the routed queries of one verify call,
// like route_fused_kernel (route.cu), with a different split of the work:
//
//  * one CTA per (KV head, row chunk of <= 40 (query, head) rows, block range).
//    A range is <= 16 statistics tiles of 16 compressed blocks, all staged in
//    shared memory by bulk copies at launch (one mbarrier per tile), one warp
//    per tile: logits by fp64 DMMA (m8n8k4; fp32 x fp32 products are exact in
//    fp64), then per row and tile the max TM, TD = sum e^(logit - TM) and the
//    selection-block shares G (through a DMMA against the overlap matrix), as
//    in route.cu -- but kept in shared memory.
//  * the CTA folds its tiles into ONE (max, denominator) pair per row and its
//    per-row selection-block sums N (on chip), publishes the pair, meets the
//    other ranges of its (KV head, row chunk) at one barrier, and turns N into
//    the KV head's normalised share of each selection block of its range
//    (the softmax over all visible blocks, nsa_attention.cpp:57-63, regrouped).
//  * the last of the CTAs that write a range's shares sums them over the KV
//    heads (score_b = sum over heads and blocks of p * overlap / (Hq l),
//    nsa_attention.cpp:52-78, regrouped -- contract P3, <= 1e-13 relative) and
//    ranks the range's blocks into per-query Top-n candidates; the last range
//    merges the candidates into the final sets (forced {0, avail-2, avail-1}
//    plus the best by (score desc, id asc), ascending, nsa_attention.cpp:94-136).
//
// Every reduction runs in a fixed order, so the scores (and indices) are
// deterministic.  All CTAs are co-resident (cooperative launch, one per SM).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "attend.h"
#include "sm100.cuh"

namespace specsv_b200 {
namespace {

constexpr int kDh = 128;
constexpr int kThreads = 512;          // 16 warps: one per tile, then all for the tail
constexpr int kWarps = kThreads / 32;
static_assert(kWarps == kR2MaxTiles, "one warp per tile");
constexpr int kMT = kR2Rows / 8;       // 8-row m-tiles
constexpr int kLd = kDh + 4;           // fp64 q row stride (== 4 mod 16: conflict-free fragments)
constexpr int kWLd = 12;               // overlap-matrix row stride (doubles)
constexpr int kWCols = 8;              // g_stride + the ones column <= 8
constexpr int kMaxPick = 64;           // n <= 64
constexpr int kTileKeyBytes = 16 * kDh * 4;  // 4 TMA boxes of 32 fp32 x 16 rows, 128B-swizzled
constexpr int kMaxCand = 512;          // candidates the final merge stages per query
constexpr int kMaxRanges = 32;         // ranges (the final merge walks one list per lane)

struct Smem {
  static constexpr size_t KEYS = 0;                                 // [T][4 boxes][16][32] f32 (1024-aligned)
  __host__ __device__ static size_t tm(int T) { return KEYS + (size_t)T * kTileKeyBytes; }  // [40][T]
  __host__ __device__ static size_t td(int T) { return tm(T) + (size_t)kR2Rows * T * 8; }   // [40][T]
  __host__ __device__ static size_t g(int T) { return td(T) + (size_t)kR2Rows * T * 8; }    // [40][T][gs]
  __host__ __device__ static size_t W(int T, int gs) { return g(T) + (size_t)kR2Rows * T * gs * 8; }
  __host__ __device__ static size_t Q(int T, int gs) { return W(T, gs) + 16 * kWLd * 8; }   // [40][kLd] f64
  __host__ __device__ static size_t bars(int T, int gs) { return Q(T, gs) + (size_t)kR2Rows * kLd * 8; }
  __host__ __device__ static size_t misc(int T, int gs) { return bars(T, gs) + 2 * kR2MaxTiles * 8; }
  __host__ __device__ static size_t bytes(int T, int gs) { return misc(T, gs) + 1024 + 1024; }
};

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// e^x for x <= 0, ~2 ulp (the routing kernels' shared exp, route.cu exp_nonpos)
__device__ __forceinline__ double exp_nonpos(double x) {
  if (!(x >= -708.0)) return 0.0;
  const double n = rint(x * 1.4426950408889634);
  double r = fma(n, -6.93147180369123816490e-01, x);
  r = fma(n, -1.90821492927058770002e-10, r);
  double p = 2.08767569878680989792e-09;
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

__device__ __forceinline__ int overlap(int i, int b, int d, int l, int l_sel) {
  const int lo = max(i * d, b * l_sel), hi = min(i * d + l, (b + 1) * l_sel);
  return hi > lo ? hi - lo : 0;
}

__device__ __forceinline__ bool ranks_before(double sa, int ia, double sb, int ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// barrier among the S co-resident CTAs of a group: a counter that returns to 0
// and a generation word that only grows (attend.cu group_barrier)
__device__ void group_barrier(int* cnt, int* gen, int S) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int g = sm100::ld_acquire_gpu(gen);
    if (sm100::atom_add_acq_rel_gpu(cnt, 1) == S - 1) {
      atomicExch(cnt, 0);
      sm100::atom_add_acq_rel_gpu(gen, 1);
    } else {
      while (sm100::ld_acquire_gpu(gen) == g) {
      }
    }
  }
  __syncthreads();
}

// diagnostics: SM cycles since the CTA started (clock64; the globaltimer
// advances in coarse steps on this part and cannot time intra-kernel phases)
__device__ __forceinline__ void stamp(const Route2Params& p, int k, long long c0) {
  if (p.trace != nullptr && threadIdx.x == 0)
    p.trace[kRouteTraceBase + blockIdx.x * 16 + k] = (unsigned long long)(clock64() - c0 + 1);
}

// the best (score desc, id asc) of the live lanes' heads, all lanes
// participate; scores are >= 0, so their bit patterns order like the values.
// Returns the winner's id (ids of live heads are distinct), -1 if none is live.
__device__ __forceinline__ int warp_pop(double score, int id, bool live) {
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(score));
  const unsigned hi = live ? static_cast<unsigned>(bits >> 32) : 0u;
  const unsigned lo = live ? static_cast<unsigned>(bits) : 0u;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, (live && hi == mhi) ? lo : 0u);
  const bool win = live && hi == mhi && lo == mlo;
  const unsigned best = __reduce_min_sync(0xffffffffu, win ? static_cast<unsigned>(id) : 0xffffffffu);
  return best == 0xffffffffu ? -1 : static_cast<int>(best);
}

struct Forced {
  int avail, f1, f2, nforced, target, want;
  __device__ explicit Forced(int a, int n) {
    avail = a;
    f1 = a - 2 > 0 ? a - 2 : -1;
    f2 = a - 1 > 0 ? a - 1 : -1;
    nforced = a > 0 ? 1 + (f1 > 0) + (f2 > 0 && f2 != f1) : 0;
    target = n < a ? n : a;
    want = target - nforced;
  }
  __device__ bool is_forced(int b) const { return b == 0 || b == f1 || b == f2; }
};

__global__ void __launch_bounds__(kThreads, 1) route2_kernel(const __grid_constant__ Route2Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-aligned base inside the shared window (128B-swizzled TMA boxes)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = p.T, gs = p.gs;
  const int item = blockIdx.x;
  const int range = item % p.NR;
  const int grp = item / p.NR;  // (KV head, row chunk)
  const int kvh = grp / p.rc, rchunk = grp % p.rc;
  const int r0 = rchunk * p.chunk_rows;
  const int nrows = min(p.chunk_rows, p.nr * p.G - r0);
  const int t0 = range * T;  // first global tile of the range

  uint8_t* keys = smem + Smem::KEYS;
  double* TM = reinterpret_cast<double*>(smem + Smem::tm(T));
  double* TD = reinterpret_cast<double*>(smem + Smem::td(T));
  double* GS = reinterpret_cast<double*>(smem + Smem::g(T));
  double* W = reinterpret_cast<double*>(smem + Smem::W(T, gs));
  double* qs = reinterpret_cast<double*>(smem + Smem::Q(T, gs));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Smem::bars(T, gs));   // keys landed
  uint64_t* lready = full + kR2MaxTiles;                                       // logits handed over
  uint8_t* misc = smem + Smem::misc(T, gs);
  int* row_mvis = reinterpret_cast<int*>(misc);                 // [40]
  double* own_m = reinterpret_cast<double*>(misc + 160);        // [40]
  double* fnorm = reinterpret_cast<double*>(misc + 160 + 320);  // [40]
  double* gmax = reinterpret_cast<double*>(misc + 160 + 640);   // [40]
  int* flags = reinterpret_cast<int*>(misc + 160 + 960);        // [4]

  // ---- prologue: the tile loads first (one thread, tile order: tile 0 lands
  // first and its warp starts while the rest stream in), then q, W, tables ----
  const long long c_start = clock64();
  stamp(p, 0, c_start);
  if (p.debug_exit == 9) return;
  if (tid == 0) {
    for (int t = 0; t < T; ++t) {
      sm100::mbar_init(&full[t], 1);
      sm100::mbar_init(&lready[t], 1);
    }
    sm100::fence_mbar_init();
    sm100::tma_prefetch(&p.tm_ck);
    for (int t = 0; t < T; ++t) {
      sm100::mbar_expect_tx(&full[t], kTileKeyBytes);
#pragma unroll
      for (int b = 0; b < 4; ++b)  // (32 fp32 of d_head) x 16 blocks; OOB blocks read as 0
        sm100::tma_load_3d(keys + (size_t)t * kTileKeyBytes + b * 2048, &p.tm_ck, 32 * b, kvh,
                           (t0 + t) * 16, &full[t]);
    }
  }
  for (int e = tid; e < kR2Rows * (kDh / 4); e += kThreads) {  // q rows (fp32 -> fp64)
    const int r = e / (kDh / 4), x4 = e % (kDh / 4);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < nrows) {
      const int rr = r0 + r;
      const int h = kvh * p.G + rr % p.G;
      v = __ldg(reinterpret_cast<const float4*>(p.q + ((int64_t)p.slot_q[rr / p.G] * p.Hq + h) * kDh) + x4);
    }
    double* dst = qs + r * kLd + x4 * 4;
    reinterpret_cast<double2*>(dst)[0] = make_double2(v.x, v.y);
    reinterpret_cast<double2*>(dst)[1] = make_double2(v.z, v.w);
  }
  for (int e = tid; e < 16 * kWCols; e += kThreads) {
    // C-fragment lane (lr, lc), n-tile nt, element c holds block i = 8 nt + 2 lc + c;
    // as the W-DMMA's A fragment that is K chunk (nt, c), k = lc: row 4 (2 nt + c) + k
    const int i = e / kWCols, j = e % kWCols;
    const int wr = 4 * (2 * (i >> 3) + (i & 1)) + ((i >> 1) & 3);
    W[wr * kWLd + j] = j < gs ? (double)overlap(i, j, p.d, p.l, p.l_sel) : (j == gs ? 1.0 : 0.0);
  }
  if (tid < kR2Rows) row_mvis[tid] = tid < nrows ? p.slot_mvis[(r0 + tid) / p.G] : 0;
  if (item == 0 && p.scores_out == nullptr) {
    for (int u = tid; u < p.n_unrouted; u += kThreads) {
      const int q = p.unrouted[u];
      p.idx_count[q] = -1;
      p.idx_forced[q] = 0u;
      for (int a = 0; a < p.n; ++a) p.idx[(int64_t)q * p.n + a] = -1;
    }
  }
  __syncthreads();

  // ---- phase 1: 8 DMMA warps (tiles w, w + 8) hand each tile's logits, in
  // their C-fragment layout, to epilogue warp w + 8 through the tile's own
  // (dead) key buffer, so one tile's epilogue overlaps the next tile's DMMAs ----
  const int lr = lane >> 2, lc = lane & 3;
  if (warp < kWarps / 2) {
    for (int t = warp; t < T; t += kWarps / 2) {
      double acc[kMT][2][2];
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
      sm100::mbar_wait(&full[t], 0);
      if (t == 0) stamp(p, 1, c_start);
      const double* qa = qs + lr * kLd + lc;
      // B fragment: key row n = 8 nt + lr of the tile, element k = 4 s + lc, in
      // box s / 8 at 16-byte chunk (s % 8) ^ (n % 8) (128B swizzle; n % 8 = lr)
      const uint8_t* kb = keys + (size_t)t * kTileKeyBytes + lr * 128 + lc * 4;
#pragma unroll 4
      for (int s = 0; s < kDh / 4; ++s) {
        double a[kMT], b[2];
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt) a[mt] = qa[mt * 8 * kLd + 4 * s];
        const uint8_t* kbs = kb + (s >> 3) * 2048 + (((s & 7) ^ lr) << 4);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) b[nt] = *reinterpret_cast<const float*>(kbs + nt * 8 * 128);
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) dmma_8x8x4(acc[mt][nt], a[mt], b[nt]);
      }
      if (p.trace != nullptr && tid == 0 && t == 0)
        p.trace[kRouteTraceBase + blockIdx.x * 16 + 11] = (unsigned long long)(clock64() - c_start);
      __syncwarp();  // every lane's key reads of this tile are done: its buffer takes the logits
      double* lg = reinterpret_cast<double*>(keys + (size_t)t * kTileKeyBytes);
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) lg[((mt * 2 + nt) * 2 + c) * 32 + lane] = acc[mt][nt][c];
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&lready[t]);
    }
    if (p.trace != nullptr && tid == 0)
      p.trace[kRouteTraceBase + blockIdx.x * 16 + 12] = (unsigned long long)(clock64() - c_start);
  } else {
    for (int t = warp - kWarps / 2; t < T; t += kWarps / 2) {
      const int tg = t0 + t;
      sm100::mbar_wait(&lready[t], 0);
      const double* lg = reinterpret_cast<const double*>(keys + (size_t)t * kTileKeyBytes);
      double acc[kMT][2][2];
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) acc[mt][nt][c] = lg[((mt * 2 + nt) * 2 + c) * 32 + lane];
      // per row: tile max, e = exp(logit - max), then TD and G through e x W
      int mv[kMT];
      double mx[kMT];
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt) {
        mv[mt] = row_mvis[8 * mt + lr];
        mx[mt] = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            acc[mt][nt][c] = __dmul_rn(acc[mt][nt][c], p.scale);
            if (tg * 16 + 8 * nt + 2 * lc + c < mv[mt]) mx[mt] = fmax(mx[mt], acc[mt][nt][c]);
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
            acc[mt][nt][c] =
                tg * 16 + 8 * nt + 2 * lc + c < mv[mt] ? exp_nonpos(acc[mt][nt][c] - mx[mt]) : 0.0;
      double g[kMT][2];
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt) g[mt][0] = g[mt][1] = 0.0;
      const double* wl = W + lc * kWLd + lr;
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
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int j = 2 * lc + c;
          if (j < gs) GS[((size_t)r * T + t) * gs + j] = g[mt][c];
          if (j == gs) TD[r * T + t] = g[mt][c];
        }
        if (lc == 0) TM[r * T + t] = mx[mt];
      }
      if (p.trace != nullptr && tid == 256 && t == 0)
        p.trace[kRouteTraceBase + blockIdx.x * 16 + 14] = (unsigned long long)(clock64() - c_start);
    }
  }
  __syncthreads();
  stamp(p, 2, c_start);
  if (p.debug_exit == 1) return;

  // ---- phase 2: fold the range's tiles -> one (max, denominator) per row and
  // the per-row selection-block sums N (relative to that max), on chip ----
  const int spt = p.spt;
  const int nb_tiles = T * spt;          // selection blocks the tiles start
  const int NB = nb_tiles + (gs - spt);  // plus the last tile's overhang
  double* sfac = reinterpret_cast<double*>(smem + Smem::KEYS);  // [40][T] (the keys are dead)
  double* N = sfac + kR2Rows * T;                                // [40][NB]
  {
    // a half-warp per row, lanes over the tiles (T <= 16): max, exp, denominator
    const int half = lane >> 4, hl = lane & 15;
    for (int r = 2 * warp + half; r < kR2Rows; r += 2 * kWarps) {
      const double tm = hl < T ? TM[r * T + hl] : -INFINITY;
      double m = tm;
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
      const double sf = (hl < T && tm != -INFINITY) ? exp_nonpos(tm - m) : 0.0;
      if (hl < T) sfac[r * T + hl] = sf;
      double den = hl < T ? TD[r * T + hl] * sf : 0.0;
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
      if (hl == 0) {
        own_m[r] = m;
        reinterpret_cast<double2*>(p.dm)[(size_t)item * kR2Rows + r] = make_double2(m, den);
      }
    }
  }
  __syncthreads();
  stamp(p, 10, c_start);

  for (int e = tid; e < nrows * NB; e += kThreads) {
    const int r = e / NB, bl = e % NB;
    const int t_lo = max(0, (bl - gs + spt) / spt), t_hi = min(T - 1, bl / spt);
    double v = 0.0;
    for (int t = t_lo; t <= t_hi; ++t) v += sfac[r * T + t] * GS[((size_t)r * T + t) * gs + (bl - t * spt)];
    N[e] = v;
  }
  // ---- the ranges of this (KV head, row chunk) meet: global max / denominator ----
  stamp(p, 3, c_start);
  if (p.debug_exit == 2) return;
  group_barrier(p.bar + 2 * grp, p.bar + 2 * grp + 1, p.NR);
  stamp(p, 4, c_start);
  if (p.debug_exit == 3) return;
  {
    // every range's (max, denominator) of every row in flight at once -> smem
    double2* mds = reinterpret_cast<double2*>(N + kR2Rows * NB);  // [NR][40]
    double* term = reinterpret_cast<double*>(mds + p.NR * kR2Rows);  // [NR][40]
    const double2* src = reinterpret_cast<const double2*>(p.dm) + (size_t)grp * p.NR * kR2Rows;
    for (int e = tid; e < p.NR * kR2Rows; e += kThreads) mds[e] = __ldcg(src + e);
    __syncthreads();
    if (tid < nrows) {
      double m = -INFINITY;
#pragma unroll 8
      for (int c = 0; c < p.NR; ++c) m = fmax(m, mds[c * kR2Rows + tid].x);
      gmax[tid] = m;
    }
    __syncthreads();
    for (int e = tid; e < p.NR * kR2Rows; e += kThreads) {
      const int r = e % kR2Rows;
      const double2 md = mds[e];
      term[e] = (r < nrows && md.y > 0.0) ? md.y * exp_nonpos(md.x - gmax[r]) : 0.0;
    }
    __syncthreads();
    if (tid < nrows) {
      double den = 0.0;
#pragma unroll 8
      for (int c = 0; c < p.NR; ++c) den += term[c * kR2Rows + tid];  // range order
      fnorm[tid] = (den > 0.0 && own_m[tid] != -INFINITY) ? exp_nonpos(own_m[tid] - gmax[tid]) / den : 0.0;
    }
  }
  __syncthreads();
  // this KV head's share of each selection block of the range, per routed slot
  const int B0 = t0 * spt;
  const bool last_range = range == p.NR - 1;
  const int own_end = last_range ? p.s_total : min(p.s_total, B0 + nb_tiles);
  const int n_own = max(0, own_end - B0);
  const int nslots = nrows / p.G;  // whole slots per chunk
  const int s0 = r0 / p.G;
  const int ov = gs - spt;
  const int nwrite = n_own + (last_range ? 0 : ov);
  for (int e = tid; e < nslots * nwrite; e += kThreads) {
    const int sl = e / nwrite, bl = e % nwrite;
    double v = 0.0;
    if (bl < NB)
      for (int g2 = 0; g2 < p.G; ++g2) v += fnorm[sl * p.G + g2] * N[(sl * p.G + g2) * NB + bl];
    const int s = s0 + sl;
    if (bl < n_own)
      p.part[((int64_t)s * p.Hkv + kvh) * p.sel_pad + B0 + bl] = v;
    else
      p.ovh[(((int64_t)s * p.Hkv + kvh) * p.NR + range) * 8 + (bl - n_own)] = v;
  }
  __syncthreads();
  if (tid == 0 || tid == 32) {  // the two range arrivals in flight at once (two warps)
    const int per = p.Hkv * p.rc;
    const int k = tid >> 5;
    int last = 0;
    if (k == 0) {
      if (sm100::atom_add_acq_rel_gpu(p.rcnt + range, 1) == per * (range > 0 ? 2 : 1) - 1) {
        atomicExch(p.rcnt + range, 0);
        last = 1;
      }
    } else if (!last_range && sm100::atom_add_acq_rel_gpu(p.rcnt + range + 1, 1) == 2 * per - 1) {
      atomicExch(p.rcnt + range + 1, 0);
      last = 1;
    }
    flags[k] = last;
  }
  __syncthreads();
  stamp(p, 5, c_start);
  if (p.debug_exit == 4) return;

  // ---- phase 3: the last writer of a range sums its scores over the KV heads
  // and ranks its blocks into per-query Top-n candidates ----
  const double score_scale = 1.0 / ((double)p.Hq * (double)p.l);
  double* sc = reinterpret_cast<double*>(smem + Smem::KEYS);  // [nr][cn] (reuses sfac / N)
  for (int pass = 0; pass < 2; ++pass) {
    if (!flags[pass]) continue;
    const int cc = range + pass;
    const int cB0 = cc * nb_tiles;
    const bool cl = cc == p.NR - 1;
    const int cend = cl ? p.s_total : min(p.s_total, cB0 + nb_tiles);
    const int cn = max(0, cend - cB0);
    __syncthreads();  // the previous pass's readers of sc are done
    for (int e = tid; e < p.nr * cn; e += kThreads) {
      const int s = e / cn, bl = e % cn;
      // every head's load in flight at once (other CTAs' data: L2), summed in head order
      double v = 0.0;
      const double* ps = p.part + (int64_t)s * p.Hkv * p.sel_pad + cB0 + bl;
      const bool has_ov = cc > 0 && bl < ov;
      const double* po = p.ovh + ((int64_t)s * p.Hkv * p.NR + cc - 1) * 8 + bl;
      for (int h0 = 0; h0 < p.Hkv; h0 += 8) {
        double x[8], y[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          x[k] = h0 + k < p.Hkv ? __ldcg(ps + (int64_t)(h0 + k) * p.sel_pad) : 0.0;
          y[k] = has_ov && h0 + k < p.Hkv ? __ldcg(po + (int64_t)(h0 + k) * p.NR * 8) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) v += x[k];
#pragma unroll
        for (int k = 0; k < 8; ++k) v += y[k];
      }
      v *= score_scale;
      sc[e] = v;
      if (p.scores_out != nullptr && s == 0 && cB0 + bl < p.slot_avail[0]) p.scores_out[cB0 + bl] = v;
    }
    __syncthreads();
    stamp(p, 6, c_start);
    if (p.scores_out != nullptr) continue;
    // a thread per (slot, block): the block's rank among the range's
    // non-forced blocks of its slot; ranks < want are the slot's candidates,
    // stored best first
    for (int e = tid; e < p.nr * cn; e += kThreads) {
      const int s = e / cn, bl = e % cn;
      const int b = cB0 + bl;
      const Forced F(p.slot_avail[s], p.n);
      if (b >= F.avail || F.is_forced(b)) continue;
      const double sb = sc[e];
      const double* row = sc + s * cn;
      const int hi = min(cn, F.avail - cB0);
      int rank = 0;
      int o = 0;
      for (; o + 8 <= hi; o += 8) {
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = row[o + k];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          rank += (!F.is_forced(cB0 + o + k) && ranks_before(x[k], cB0 + o + k, sb, b)) ? 1 : 0;
      }
      for (; o < hi; ++o) rank += (!F.is_forced(cB0 + o) && ranks_before(row[o], cB0 + o, sb, b)) ? 1 : 0;
      if (rank < F.want) {
        p.cand_s[((int64_t)s * p.NR + cc) * kMaxPick + rank] = sb;
        p.cand_i[((int64_t)s * p.NR + cc) * kMaxPick + rank] = b;
      }
    }
    if (tid < p.nr) {  // candidates of slot tid in this range
      const Forced F(p.slot_avail[tid], p.n);
      const int hi = min(cend, F.avail);
      int k_own = max(0, hi - cB0);
      if (k_own > 0) {
        k_own -= (cB0 <= 0 && 0 < hi) ? 1 : 0;
        k_own -= (F.f1 > 0 && cB0 <= F.f1 && F.f1 < hi) ? 1 : 0;
        k_own -= (F.f2 > 0 && F.f2 != F.f1 && cB0 <= F.f2 && F.f2 < hi) ? 1 : 0;
      }
      p.cand_n[tid * p.NR + cc] = max(0, min(F.want, k_own));
    }
    __syncthreads();
    stamp(p, 7, c_start);
    if (p.debug_exit == 5) continue;
    if (tid == 0) {
      flags[2] = 0;
      if (sm100::atom_add_acq_rel_gpu(p.fcnt, 1) == p.NR - 1) {
        atomicExch(p.fcnt, 0);
        flags[2] = 1;
      }
    }
    __syncthreads();
    if (!flags[2]) continue;

    // ---- phase 4: the last range merges every range's candidates per query ----
    // staging: the candidates of every slot (flat, slot-major), then per-warp picks
    const int cstride = p.NR * p.n;  // >= a slot's candidates
    double* cs = reinterpret_cast<double*>(smem + Smem::KEYS);                 // [nr][cstride]
    int* ci = reinterpret_cast<int*>(cs + (size_t)p.nr * cstride);             // same
    int* offs = ci + (size_t)p.nr * cstride;                                   // [nr][33]
    int* picks = offs + (size_t)p.nr * 33;                                     // [warps][kMaxPick]
    // every slot's range counts in flight at once, prefix per slot
    for (int s = warp; s < p.nr; s += kWarps) {
      const int kc = lane < p.NR ? __ldcg(p.cand_n + s * p.NR + lane) : 0;
      int incl = kc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      offs[s * 33 + lane] = incl - kc;
      if (lane == 31) offs[s * 33 + 32] = incl;
    }
    __syncthreads();
    // every candidate load of every slot in flight at once: a thread per (slot, range, k)
    const int kq = (p.n + 3) / 4;  // 4 consecutive k per thread
    for (int e = tid; e < p.nr * p.NR * kq; e += kThreads) {
      const int s = e / (p.NR * kq), rem = e % (p.NR * kq);
      const int c = rem / kq, k0 = 4 * (rem % kq);
      const int beg = offs[s * 33 + c], len = offs[s * 33 + c + 1] - beg;
      const int64_t src = ((int64_t)s * p.NR + c) * kMaxPick + k0;
      double v[4];
      int id[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = k0 + k < len ? __ldcg(p.cand_s + src + k) : 0.0;
        id[k] = k0 + k < len ? __ldcg(p.cand_i + src + k) : 0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k0 + k < len) {
          cs[(size_t)s * cstride + beg + k0 + k] = v[k];
          ci[(size_t)s * cstride + beg + k0 + k] = id[k];
        }
    }
    __syncthreads();
    stamp(p, 8, c_start);
    for (int s = warp; s < p.nr; s += kWarps) {
      const Forced F(p.slot_avail[s], p.n);
      const int q = p.slot_q[s];
      int* pk = picks + warp * kMaxPick;
      // k-way merge: lane c walks range c's best-first list
      {
        const int c = lane;
        const int beg = c < p.NR ? offs[s * 33 + c] : 0;
        const int len = c < p.NR ? offs[s * 33 + c + 1] - beg : 0;
        const double* lcs = cs + (size_t)s * cstride;
        const int* lci = ci + (size_t)s * cstride;
        int ptr = 0;
        double hs = 0.0;
        int hid = 0;
        bool live = ptr < len;
        if (live) {
          hs = lcs[beg];
          hid = lci[beg];
        }
        for (int k = 0; k < F.want; ++k) {
          const int best = warp_pop(hs, hid, live);
          if (best < 0) break;
          if (live && hid == best) {
            pk[F.nforced + k] = best;
            ++ptr;
            live = ptr < len;
            if (live) {
              hs = lcs[beg + ptr];
              hid = lci[beg + ptr];
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0 && F.avail > 0) {
        int c = 0;
        pk[c++] = 0;
        if (F.f1 > 0) pk[c++] = F.f1;
        if (F.f2 > 0 && F.f2 != F.f1) pk[c++] = F.f2;
      }
      __syncwarp();
      const int cnt = F.target > 0 ? F.target : 0;
      uint32_t fb = 0u;
      for (int a = lane; a < cnt; a += 32) {  // ascending by a rank-and-scatter (ids are distinct)
        const int v = pk[a];
        int rank = 0;
#pragma unroll 8
        for (int o = 0; o < cnt; ++o) rank += pk[o] < v ? 1 : 0;
        p.idx[(int64_t)q * p.n + rank] = v;
        if (F.is_forced(v) && rank < 32) fb |= 1u << rank;
      }
      for (int a = cnt + lane; a < p.n; a += 32) p.idx[(int64_t)q * p.n + a] = -1;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) fb |= __shfl_xor_sync(0xffffffffu, fb, off);
      if (lane == 0) {
        p.idx_count[q] = cnt;
        p.idx_forced[q] = fb;
      }
      __syncwarp();
    }
    __syncthreads();
    stamp(p, 9, c_start);
  }
}

int sm_count_r2() {
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

}  // namespace

bool route2_plan(int nr, int G, int Hkv, int ntiles, int gs, int spt, int n, Route2Params& p) {
  if (nr < 1 || ntiles < 1 || gs + 1 > kWCols || n > kMaxPick || n < 1) return false;
  const int chunk_rows = (kR2Rows / G) * G;  // whole slots per chunk
  if (chunk_rows < 1) return false;
  const int rc = (nr * G + chunk_rows - 1) / chunk_rows;
  const int groups = Hkv * rc;
  const int sms = std::min(sm_count_r2(), kR2MaxRanges);
  int NR = sms / groups;
  if (NR < 1) return false;
  // the final merge walks one candidate list per lane and stages <= NR x n per query
  NR = std::min({NR, ntiles, kMaxCand / n, kMaxRanges});
  int T = (ntiles + NR - 1) / NR;
  if (T > kR2MaxTiles) return false;
  NR = (ntiles + T - 1) / T;  // no empty ranges
  if (Smem::bytes(T, gs) > 227 * 1024) return false;
  // the tail reuses the tile region (keys + tile statistics): fold arrays and
  // the (max, den) staging, the range scores of every routed slot, the final
  // merge's candidate staging
  const size_t region = Smem::W(T, gs) - Smem::KEYS;
  const size_t nbm = (size_t)T * spt + 8;
  const size_t fold = (size_t)kR2Rows * T * 8 + (size_t)kR2Rows * nbm * 8 + (size_t)NR * kR2Rows * 24;
  const size_t scores = (size_t)nr * nbm * 8;
  const size_t merge = (size_t)nr * NR * n * 12 + (size_t)nr * 33 * 4 + (size_t)kWarps * kMaxPick * 4;
  if (std::max({fold, scores, merge}) > region) return false;
  p.rc = rc;
  p.chunk_rows = chunk_rows;
  p.NR = NR;
  p.T = T;
  p.ntiles = ntiles;
  return true;
}

size_t route2_ws_bytes(int nr, int Hkv, int sel_pad) {
  const size_t items = kR2MaxRanges;
  size_t b = items * kR2Rows * 16;                                // dm
  b += (size_t)nr * Hkv * sel_pad * 8;                            // part
  b += (size_t)nr * Hkv * kR2MaxRanges * 8 * 8;                   // ovh
  b += (size_t)nr * kR2MaxRanges * kMaxPick * (8 + 4);            // cand_s, cand_i
  b += (size_t)nr * kR2MaxRanges * 4;                             // cand_n
  return b + 5 * 256;
}

cudaError_t launch_route2(const Route2Params& p, cudaStream_t s) {
  const size_t smem = Smem::bytes(p.T, p.gs);
  cudaError_t e = cudaFuncSetAttribute(route2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int items = p.Hkv * p.rc * p.NR;
  void* args[] = {const_cast<Route2Params*>(&p)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(route2_kernel), dim3(items), dim3(kThreads),
                                     args, smem, s);
}

}  // namespace specsv_b200
