// attend.cu -- fused NSA verify attention for sm_100a (compressed + selected +
// window branches + learned-gate combine) over all queries of one request.
//
// Replaces verify::group_attend_exact / group_attend_approx / attend_one
// (src/group_attend.cpp:59-139) and the branch kernels they call
// (src/nsa_attention.cpp:138-251), for every layer (refresh layers after the
// routing launch, reuse layers as the single fused launch).
//
// Design ("fused attend"):
//  * S split CTAs per (KV head, query chunk), co-resident (cooperative launch);
//    they split the KEY tiles.  A key tile is 128 keys: 128 compressed blocks
//    (cmp branch), two 64-token selection blocks of the per-request UNION of
//    selected and window blocks (slc and win branches from one QK^T), or the
//    draft-tree rows (win).  Every K/V tile is TMA-staged into shared memory
//    ONCE for all queries and all GQA heads that read it -- the overlap-aware
//    dedup of the paper.
//  * Swap-AB: S^T = K_tile . Q^T on tcgen05 (M = 128 keys, N = query columns),
//    so the key dimension fills the 128-lane MMA; O^T += V^T . P^T (M = d_head).
//    q (pre-scaled by log2(e)/sqrt(dh)) and P are split hi+lo in bf16 (~16
//    mantissa bits).  The hi and lo halves are stacked along N (N = 2 x cols),
//    so each MMA reads its K or V tile from shared memory ONCE: the MMAs are
//    bound by that operand read, not by the tensor pipe.
//  * 12 softmax warps: warp w owns TMEM lane quadrant w%4 (32 keys) and the
//    16-column chunk w/4 (<= 48 columns).  Ownership / routing-bound / window /
//    tree masks are applied in registers per (key, query); masked entries
//    contribute exactly 0.  Row sums stay in registers.
//  * Fast pass: one fixed reference logit per column, no running max (checked
//    at the end of the pass; a robust running-max pass redoes the rare CTA
//    whose logits fall outside the window, see kFastHi).
//  * Split partials are merged behind a per-head global barrier among the S
//    co-resident CTAs, and the gate combine is applied in the same kernel: the
//    branch partial outputs never leave this launch's L2-resident workspace.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "attend.h"
#include "policy.h"
#include "sm100.cuh"

namespace specsv_b200 {
namespace {

using namespace sm100;

constexpr int kDh = 128;
constexpr int kTile = 128;
constexpr int kCols = kAttendCols;  // query columns (queries x heads) per CTA
constexpr int kSoftWarps = 12;      // 4 lane quadrants x 3 column chunks
constexpr int kSoftThreads = kSoftWarps * 32;
static_assert(kSoftThreads == 2 * 3 * 64, "merge: 64 threads per (column, branch), two columns per round");
constexpr int kMaxSplits = 18;
constexpr int kWarpTma = 12;
constexpr int kWarpQk = 13;
constexpr int kWarpPv = 14;
constexpr int kWarpUnion = 15;
static_assert(kWarpPv == kWarpQk + 1 && kWarpUnion == kWarpPv + 1, "warp roles");
constexpr int kThreads = 16 * 32;
constexpr uint32_t kTmemCols = 512;
constexpr int kTmemS = 0;           // two S buffers of [hi | lo] x 48: cols 0, 96
constexpr int kTmemO = 192;         // O_cmp 192, O_slc 288, O_win 384, each [hi | lo] x 48
constexpr int kTmemStride = 2 * kCols;
constexpr float kRescaleThresh = 8.0f;  // log2 units (robust pass)
constexpr int kBarSoft = 1;         // named barriers: softmax warps
constexpr int kBarChunk0 = 3;       // 3..5: the 4 warps of one column chunk
constexpr int kBarPassEnd = 7;
constexpr int kBarRedo = 8;
constexpr int kBarUnion = 9;        // the 12 softmax warps build the union
constexpr int kUnionThreads = kSoftThreads;

// shared memory map (bytes from the 1024-aligned base)
constexpr uint32_t kOffK = 0;        // 2 stages x 32 KB (K tiles: free once their QK is done)
constexpr uint32_t kOffV = 65536;    // 2 stages x 32 KB
constexpr uint32_t kOffQ = 131072;   // Q^T [hi | lo] rows, two 64-element K halves of 96 x 128 B
constexpr uint32_t kQHalf = 2 * kCols * 128;
// P^T of the tile, N = [first active branch hi | lo | second hi | lo] x 48 columns:
// 3 MN atoms x 16 KB, so a tile with both token branches (selected + window,
// whose O accumulators are adjacent in TMEM) is ONE set of N = 192 MMAs
constexpr uint32_t kOffP = kOffQ + 2 * kQHalf;
constexpr uint32_t kOffMisc = kOffP + 49152;
constexpr uint32_t kStageBytes = 32768;

enum Branch { kCmp = 0, kSlc = 1, kWin = 2 };
enum TileKind { kTileCmp = 0, kTileTok = 1, kTileTree = 2 };

struct Misc {
  uint64_t k_full[2], v_full[2], k_empty[2], v_empty[2], s_full[2], s_free[2], pv_done[2];
  // p_full is double-buffered by tile parity like s_full: a softmax warp may
  // finish tile j + 1 before a slower warp arrives for tile j (tile j + 1 only
  // needs PV(j - 1)), and a single barrier would then complete tile j's phase
  // with that warp's P still unwritten (it cannot get two tiles ahead: tile
  // j + 2 needs PV(j), which needs every tile-j arrival)
  uint64_t p_full[2], q_ready, rows_ready, union_ready;
  uint32_t tmem_base;
  int32_t n_union, n_tok_tiles;
  int32_t flag;                   // end-of-pass check failed: redo the tiles in the robust pass
  alignas(16) float mref[kCols];  // fast-pass reference logit per column (log2 units)
  float m2[3][kCols];             // running max (log2 units) per branch and column
  float thr[3][kCols];            // m2 + threshold
  float alpha[kCols];
  float tmax[4][kCols];
  int32_t vote[4][kCols / 16];    // [quadrant][chunk]
  float lred[3][4][kCols];        // row sums per branch, quadrant, column
  uint32_t actw[kSoftWarps][2];   // fast pass: active (branch, column) bits per warp
  int32_t qbound[kMaxChunkQ], qwlo[kMaxChunkQ], qwhi[kMaxChunkQ], qmvis[kMaxChunkQ];
  int32_t qcount[kMaxChunkQ];
  int32_t qsel[kMaxChunkQ * 64];
  uint32_t bitmap[kMaxUnionWords];
  int32_t union_blk[kMaxUnion];
  uint32_t union_own[kMaxUnion];
};
static_assert(sizeof(Misc) + kOffMisc + 1024 <= 232448, "shared memory budget");
static_assert(kTmemO + 3 * kTmemStride <= (int)kTmemCols, "TMEM budget");

[[maybe_unused]] __device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// trace stamps (specsv_debug_attend_trace): compiled only into a diagnostics
// build (SPECSV_TRACE_TILES=1 python -m paper_2605_19893_b200.build --force)
// -- even untaken, the per-tile ones cost ~15% of a softmax warp's
// instructions per tile, and the trace pointer and CTA id they keep live cost
// registers in the tile loop
#ifdef SPECSV_TRACE_TILES
#define TILE_STAMP(cond, slot, val)                            \
  do {                                                         \
    if (cond) p.trace[cta_id * 64 + (slot)] = (val);           \
  } while (0)
#else
#define TILE_STAMP(cond, slot, val) \
  do {                              \
  } while (0)
#endif

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// try_wait already parks the warp briefly in hardware between probes; an
// explicit suspend-time hint delays the wake-up by up to ~1 us (measured), so
// latency-critical waits use the plain form
__device__ __forceinline__ void mbar_sleep_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// a wait that may be long (the union, built by one warp from index rows that
// may still be in flight): back off between probes so the waiting warps leave
// the union warp the issue slots
__device__ __forceinline__ void mbar_backoff_wait(uint64_t* bar, uint32_t parity, bool backoff) {
  while (!mbar_try_wait(bar, parity))
    if (backoff) __nanosleep(256);
}

// transpose-reduce of 16 columns across the warp: returns, in lanes 2c and
// 2c+1, the reduction over all 32 lanes of column c (16 shuffles)
template <bool kMax>
__device__ __forceinline__ float reduce16(float (&v)[16], int lane) {
#pragma unroll
  for (int lvl = 16, half = 8; lvl >= 2; lvl >>= 1, half >>= 1) {
    const bool up = (lane & lvl) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? v[i] : v[i + half];
      const float keep = up ? v[i + half] : v[i];
      const float got = __shfl_xor_sync(0xffffffffu, send, lvl);
      v[i] = kMax ? fmaxf(keep, got) : keep + got;
    }
  }
  const float other = __shfl_xor_sync(0xffffffffu, v[0], 1);
  return kMax ? fmaxf(v[0], other) : v[0] + other;
}

// per-(chunk, head) barrier among the S co-resident split CTAs: a counter
// that returns to 0 plus a generation word that only grows (workspace words
// start at 0 and are owned by this library)
__device__ void group_barrier(int* cnt, int* gen, int S, int tid) {
  __syncthreads();
  if (tid == 0) {
    // the generation cannot advance before this CTA arrives, so reading it
    // first is race-free; acq_rel arrivals publish the CTA's partials (the
    // bar.sync above orders them before thread 0) and acquire the others'
    const int g = sm100::ld_acquire_gpu(gen);
    if (sm100::atom_add_acq_rel_gpu(cnt, 1) == S - 1) {
      // the last arrival: plain stores (no round trip before the others see
      // the new generation); the release orders the reset before it
      *reinterpret_cast<volatile int*>(cnt) = 0;
      sm100::st_release_gpu(gen, g + 1);
    } else {
      while (sm100::ld_acquire_gpu(gen) == g) __nanosleep(32);
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// union of selected + window blocks with per-block query ownership (exact:
// own set; approx: representative's set; both clamped at the query's routing
// bound, layer_roles.cpp:37-50).  Built by the union warp while the
// compressed tiles (which do not need it) are already in flight; the index
// rows are staged with fire-and-forget cp.async (one round trip).
// index rows of the chunk's queries -> smem, fire-and-forget (one round trip).
// Per-query kernel parameters are read once, lane q holding query q's (a
// divergent read of the parameter space serialises per distinct address).
// The union warp's kernel parameters, read into registers before it waits
// for the routing launch: a first read of the parameter bank misses the
// constant cache, and one serialised miss per line after the wait would sit
// on the critical path.
struct UnionArgs {
  const int32_t* idx;
  const int32_t* idx_count;
  int n, l_sel, rows;
  int my_src;  // lane q: query q's index-set row
};

__device__ __forceinline__ UnionArgs union_args(const AttendParams& p, int q0, int nqc, int lane) {
  UnionArgs u;
  u.idx = p.idx;
  u.idx_count = p.idx_count;
  u.n = p.n_sel;
  u.l_sel = p.l_sel;
  u.rows = p.rows;
  u.my_src = lane < nqc ? p.src_row[q0 + lane] : 0;
  // materialise every value now (the loads must not sink below the wait)
  asm volatile("" ::"l"(u.idx), "l"(u.idx_count), "r"(u.n), "r"(u.l_sel), "r"(u.rows), "r"(u.my_src));
  return u;
}

__device__ __forceinline__ void stage_index_rows(const UnionArgs& u, Misc& m, int nqc, int lane) {
  const int n = u.n;
  if (lane < nqc) cp_async4(&m.qcount[lane], u.idx_count + u.my_src);
  for (int i = 0; i < nqc; ++i) {
    const int r = __shfl_sync(0xffffffffu, u.my_src, i);
    for (int k = lane; k < n; k += 32) cp_async4(&m.qsel[i * n + k], u.idx + r * n + k);
  }
}

// position of the j-th (0-based) set bit of v (v has more than j set bits)
__device__ __forceinline__ int nth_set_bit(uint32_t v, int j) {
  int pos = 0;
#pragma unroll
  for (int sh = 16; sh >= 1; sh >>= 1) {
    const int c = __popc(v & ((1u << sh) - 1u));
    if (c <= j) {
      j -= c;
      v >>= sh;
      pos += sh;
    }
  }
  return pos;
}

// The union of selected + window blocks with per-block query ownership, built
// by the 12 softmax warps (kUnionThreads participants, `pt` = this thread's
// index among them) when they reach their first token tile, from the index
// rows the union warp staged (it also zeroed the bitmap and the ownership
// words).  Two steps: (1) set the window (whole-word masks) and selected
// bits; (2) every warp scans the word popcounts in registers (lane L covers
// words [L << lp, (L + 1) << lp)), so any word's union rank is one shuffle
// away; warp k scatters the k-th, (k+12)-th, ... set bit of each word and the
// index-row entries OR their ownership bits.  The build is a short chain of
// dependent instructions per warp: five barrier-separated steps with a
// one-lane-per-word scatter loop took ~4000 SM cycles in the step, this
// ~2500; one warp alone (the union warp, under the compressed tiles) ~9000.
__device__ void coop_union(Misc& m, int pt, int nqc, int n, int l_sel, int rows, int wlo, int whi) {
  const int nsel = (rows + l_sel - 1) / l_sel;
  const int words = (nsel + 31) >> 5;
  const int lane = pt & 31, wid = pt >> 5;
  const int nsl = nqc * n;
  mbar_sleep_wait(&m.rows_ready, 0);
  {  // the window's blocks are contiguous: one OR per bitmap word
    const int b0 = wlo / l_sel, b1 = whi / l_sel;
    const int w = (b0 >> 5) + pt;
    if (b0 <= b1 && w <= (b1 >> 5)) {
      const int lo = max(b0, w << 5) & 31, hi = min(b1, (w << 5) + 31) & 31;
      atomicOr(&m.bitmap[w], (0xFFFFFFFFu >> (31 - hi)) & (0xFFFFFFFFu << lo));
    }
  }
  for (int e = pt; e < nsl; e += kUnionThreads) {
    const int i = e / n, k = e - i * n;
    int b = m.qsel[e];
    if (k >= m.qcount[i] || b < 0 || (int64_t)b * l_sel >= m.qbound[i] || b >= nsel) b = -1;
    m.qsel[e] = b;
    if (b >= 0) atomicOr(&m.bitmap[b >> 5], 1u << (b & 31));
  }
  __syncwarp();
  named_bar_sync(kBarUnion, kUnionThreads);
  const int lp = words <= 32 ? 0 : 32 - __clz(((words + 31) >> 5) - 1);  // 2^lp words per lane
  const int wb = lane << lp, we = min(words, (lane + 1) << lp);
  int local = 0;
  for (int w = wb; w < we; ++w) local += __popc(m.bitmap[w]);
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  const int base = incl - local;  // union rank of word wb's first block
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  {  // scatter: this lane's words, this warp's share of their set bits
    int r = base;
    for (int w = wb; w < we; ++w) {
      const uint32_t bits = m.bitmap[w];
      const int c = __popc(bits);
      for (int j = wid; j < c; j += kSoftWarps)
        if (r + j < kMaxUnion) m.union_blk[r + j] = (w << 5) + nth_set_bit(bits, j);
      r += c;
    }
  }
  // ownership: entry e of the index rows (query e / n) owns its block
  for (int e0 = pt - lane; e0 < nsl; e0 += kUnionThreads) {
    const int e = e0 + lane;
    const int b = e < nsl ? m.qsel[e] : -1;
    const int w = b >= 0 ? (b >> 5) : 0;
    int r = __shfl_sync(0xffffffffu, base, w >> lp);
    for (int w2 = (w >> lp) << lp; w2 < w; ++w2) r += __popc(m.bitmap[w2]);
    r += __popc(m.bitmap[w] & ((1u << (b & 31)) - 1u));
    if (b >= 0 && r < kMaxUnion) atomicOr(&m.union_own[r], 1u << (e / n));
  }
  if (pt == 0) {
    m.n_union = min(total, kMaxUnion);
    m.n_tok_tiles = (min(total, kMaxUnion) + 1) / 2;
  }
  __syncwarp();
  named_bar_sync(kBarUnion, kUnionThreads);
  if (pt < 32) mbar_arrive(&m.union_ready);  // the TMA and MMA warps wait for this
}

// the union's shared state, zeroed by the union warp before it stages the rows
__device__ __forceinline__ void zero_union(Misc& m, int nqc, int n, int l_sel, int rows, int wlo, int whi,
                                           int lane) {
  const int words = ((rows + l_sel - 1) / l_sel + 31) >> 5;
  for (int w = lane; w < words; w += 32) m.bitmap[w] = 0u;
  const int umax = min(kMaxUnion, nqc * n + (whi / l_sel - wlo / l_sel + 1));
  for (int u = lane; u < umax; u += 32) m.union_own[u] = 0u;
}

struct TileInfo {
  int kind;
  int base;    // cmp: first compressed block; tok: union index of the first half
  bool act_a;  // branch A (cmp or slc) has work
  bool act_b;  // branch B (win) has work
};

__device__ __forceinline__ TileInfo tile_info(const Misc& m, int n_cmp, int t, int wlo, int whi,
                                              int l_sel) {
  TileInfo ti;
  if (t < n_cmp) {
    ti.kind = kTileCmp;
    ti.base = t * kTile;
    ti.act_a = true;
    ti.act_b = false;
  } else if (t < n_cmp + m.n_tok_tiles) {
    ti.kind = kTileTok;
    ti.base = 2 * (t - n_cmp);
    const int b0 = m.union_blk[ti.base];
    bool win = (b0 * l_sel <= whi) && (b0 * l_sel + l_sel - 1 >= wlo);
    uint32_t own = m.union_own[ti.base];
    if (ti.base + 1 < m.n_union) {
      const int b1 = m.union_blk[ti.base + 1];
      own |= m.union_own[ti.base + 1];
      win = win || ((b1 * l_sel <= whi) && (b1 * l_sel + l_sel - 1 >= wlo));
    }
    ti.act_a = own != 0u;
    ti.act_b = win;
  } else {
    ti.kind = kTileTree;
    ti.base = 0;
    ti.act_a = false;
    ti.act_b = true;
  }
  return ti;
}

// 16 bf16x2 words (this thread's key row, 16 consecutive N columns from n0)
// into an MN-major SW128 operand of 128 keys whose 64-column atoms are 16 KB apart
__device__ __forceinline__ void store_cols(uint8_t* base, int row, int n0, const uint32_t (&w)[8]) {
  uint8_t* atom = base + (n0 >> 6) * 16384;
  const int u0 = (n0 & 63) >> 3;
  *reinterpret_cast<uint4*>(atom + sw128_off(row, u0)) = make_uint4(w[0], w[1], w[2], w[3]);
  *reinterpret_cast<uint4*>(atom + sw128_off(row, u0 + 1)) = make_uint4(w[4], w[5], w[6], w[7]);
}

// P^T of one branch for this warp's 16 columns x its 32 key rows: masked
// probabilities -> hi at N = nb + c0.., lo at N = nb + 48 + c0.. (bf16), and
// the warp's column sums added to lacc (lanes 2c, 2c+1 hold column c)
__device__ __forceinline__ void write_p(uint8_t* pdst, int row, int c0, int nb, uint32_t cm,
                                        const float (&pe)[16], float& lacc, int lane) {
  float pv[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) pv[e] = ((cm >> e) & 1u) ? pe[e] : 0.f;
  uint32_t hi[8], lo[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float a = pv[2 * e], b = pv[2 * e + 1];
    const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
    const float2 hf = __bfloat1622float2(h2);
    hi[e] = *reinterpret_cast<const uint32_t*>(&h2);
    lo[e] = pack_bf16(a - hf.x, b - hf.y);
  }
  store_cols(pdst, row, nb + c0, hi);
  store_cols(pdst, row, nb + kCols + c0, lo);
  lacc += reduce16<false>(pv, lane);
}

// Softmax reference.  Pass 0 (fast) uses ONE fixed reference logit per column,
// mref = the column's logit against the newest committed key (a key inside
// every query's window), for all tiles and branches: P = 2^(s - mref) needs no
// running max, no cross-warp votes and no O rescales.  fp32/bf16 share the
// same exponent range, so P keeps its relative precision while
// s - mref <= kFastHi; the pass is checked at its end (no active logit above
// mref + kFastHi, every active branch sum >= 2^-kFastHi) and otherwise redone
// in pass 1 (robust) with the classic lazily-raised running max.
constexpr float kFastHi = 48.0f;

// One CTA: split `split` of KV head `kvh` for query chunk `chunk` of the
// request `p` (the single-request and the batched kernels below).
__device__ __forceinline__ void attend_cta(const AttendParams& p, const int split, const int kvh,
                                           const int chunk, const int cta_id) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align inside the shared window without leaving the shared address space
  // (a uintptr_t round trip would turn every Misc access into a generic load)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Misc& m = *reinterpret_cast<Misc*>(smem + kOffMisc);
  const uint32_t sbase = smem_u32(smem);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int S = p.n_splits;
  const int q0 = chunk * p.qc_size;
  const int nqc = min(p.qc_size, p.nq - q0);
  const int ncols = nqc * p.G;
  const int nqk = (ncols + 15) & ~15;  // hi columns; lo columns follow at nqk
  const int nch = nqk >> 4;            // 16-column chunks holding valid columns
  const int gshift = __ffs(p.G) - 1;
#ifdef SPECSV_TRACE_TILES
  const bool trace = p.trace != nullptr;
#endif
  const int n_cmp = p.ch_ncmp[chunk];  // compressed tiles do not depend on the union
  const int cwlo = p.ch_wlo[chunk], cwhi = p.ch_whi[chunk];
  const bool has_tree = (p.gamma > 0) && (q0 + nqc > 1);

  // ---- TMA issue helpers (compressed tiles need no union) ------------------
  auto tile_rows = [&](int t, const CUtensorMap*& tk, const CUtensorMap*& tv, int& r0, int& r1) {
    if (t < n_cmp) {
      tk = &p.tm_ck; tv = &p.tm_cv;
      r0 = t * kTile; r1 = r0 + 64;
    } else if (t < n_cmp + m.n_tok_tiles) {
      tk = &p.tm_k; tv = &p.tm_v;
      const int u0 = 2 * (t - n_cmp);
      r0 = m.union_blk[u0] * p.l_sel;
      r1 = (u0 + 1 < m.n_union ? m.union_blk[u0 + 1] : m.union_blk[u0]) * p.l_sel;
    } else {
      tk = &p.tm_tk; tv = &p.tm_tv;
      r0 = 0; r1 = 64;
    }
  };
  // one K or V stage (v = 0 / 1); a stage is reused for tile J once tile J - 2
  // released it: K after its QK, V after its PV
  auto issue = [&](int t, int J, int v) {
    const int st = J & 1;
    if (J >= 2) mbar_sleep_wait(v ? &m.v_empty[st] : &m.k_empty[st], ((J >> 1) + 1) & 1);
    uint8_t* dst = smem + (v ? kOffV : kOffK) + st * kStageBytes;
    uint64_t* full = v ? &m.v_full[st] : &m.k_full[st];
    TILE_STAMP(trace && J < 8 && !v, 8 + J, globaltimer());
    mbar_expect_tx(full, kStageBytes);
    const CUtensorMap *tk, *tv;
    int r0, r1;
    tile_rows(t, tk, tv, r0, r1);
    const CUtensorMap* tm = v ? tv : tk;
    const uint64_t pol = l2_evict_first_policy();  // each tile is read once per launch
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      tma_load_3d_hint(dst + c * 16384, tm, c * 64, kvh, r0, full, pol);
      tma_load_3d_hint(dst + c * 16384 + 8192, tm, c * 64, kvh, r1, full, pol);
    }
  };
  // stages issued before the CTA-wide barrier (compressed tiles only)
  int pre = 0;
  while (pre < 2 && split + pre * S < n_cmp) ++pre;
  // tile count once the union is known (identical in every role)
  auto tile_count = [&]() {
    const int n_total = n_cmp + m.n_tok_tiles + (has_tree ? 1 : 0);
    return split < n_total ? (n_total - split + S - 1) / S : 0;
  };

  // ---- prologue: everything that needs no other warp goes out first --------
  float4 xa[2], xb[2];  // softmax warps: this thread's q units, in flight over the barrier

  uint4 kr;             //                and its slice of the reference key row
  if (warp == kWarpTma) {
    if (lane == 0) {
      for (int i = 0; i < 2; ++i) {
        mbar_init(&m.k_full[i], 1);
        mbar_init(&m.v_full[i], 1);
        mbar_init(&m.k_empty[i], 1);
        mbar_init(&m.v_empty[i], 1);
        mbar_init(&m.s_full[i], 1);
        mbar_init(&m.s_free[i], 4 * nch);  // the warps of the active column chunks
        mbar_init(&m.pv_done[i], 1);
      }
      mbar_init(&m.p_full[0], 4 * nch);
      mbar_init(&m.p_full[1], 4 * nch);
      mbar_init(&m.q_ready, kSoftWarps);
      mbar_init(&m.rows_ready, 32);
      mbar_init(&m.union_ready, 32);
      m.flag = (p.debug_flags & 1) ? 1 : 0;  // bit 0: force the robust redo (tests)
      fence_mbar_init();
      for (int j = 0; j < pre; ++j) {
        issue(split + j * S, j, 0);
        issue(split + j * S, j, 1);
      }
    }
    __syncwarp();
    tmem_alloc<kTmemCols>(&m.tmem_base);
  } else if (warp < kSoftWarps) {
#ifdef ATTEND_NO_KREF  // timing experiment only: breaks the fast-pass reference
    kr = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
#else
    kr = reinterpret_cast<const uint4*>(p.k_raw + ((int64_t)(p.rows - 1) * p.Hkv + kvh) * kDh)[tid & 15];
#endif
#pragma unroll
    for (int it = 0; it < 2; ++it) {  // 48 columns x 16 units of 8 elements, 2 units per thread
      const int unit = tid + it * kSoftThreads;
      const int c = unit >> 4, u16 = unit & 15;
      if (c < ncols) {
        const int qg = q0 + (c >> gshift);
        const int h = kvh * p.G + (c & (p.G - 1));
        const float4* src = reinterpret_cast<const float4*>(p.q + ((int64_t)qg * p.Hq + h) * kDh + u16 * 8);
        xa[it] = src[0];
        xb[it] = src[1];
      } else {
        xa[it] = make_float4(0.f, 0.f, 0.f, 0.f);
        xb[it] = xa[it];
      }
    }
  } else if (warp == kWarpQk && lane == 0) {
    tma_prefetch(&p.tm_k);
    tma_prefetch(&p.tm_v);
    tma_prefetch(&p.tm_tk);
    tma_prefetch(&p.tm_tv);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = m.tmem_base;
  TILE_STAMP(trace && tid == 0, 0, globaltimer());

  if (warp < kSoftWarps) {
    const int qd = warp & 3, ck = warp >> 2;  // TMEM lane quadrant, column chunk
    const int c0 = 16 * ck;
    const bool active = ck < nch;             // this warp's columns hold queries
    const uint32_t lanebase = tmem + ((uint32_t)(qd * 32) << 16);
    // =================== setup: Q^T (hi rows, then lo rows) and the reference logits ===================
    {
      if (tid < nqc) {
        m.qbound[tid] = p.qbound[q0 + tid];
        m.qwlo[tid] = p.qwlo[q0 + tid];
        m.qwhi[tid] = p.qwhi[q0 + tid];
        m.qmvis[tid] = p.qmvis[q0 + tid];
      }
      const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kr);
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int unit = tid + it * kSoftThreads;
        const int c = unit >> 4, u16 = unit & 15;
        const float sc = p.scale_log2;
        const float x[8] = {xa[it].x * sc, xa[it].y * sc, xa[it].z * sc, xa[it].w * sc,
                            xb[it].x * sc, xb[it].y * sc, xb[it].z * sc, xb[it].w * sc};
        float dot = 0.f;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 kf = __bfloat1622float2(k2[e]);
          dot = fmaf(x[2 * e], kf.x, fmaf(x[2 * e + 1], kf.y, dot));
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
          const float2 hf = __bfloat1622float2(h2);
          hi[e] = *reinterpret_cast<const uint32_t*>(&h2);
          lo[e] = pack_bf16(x[2 * e] - hf.x, x[2 * e + 1] - hf.y);
        }
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
        if (u16 == 0) m.mref[c] = dot;
        uint8_t* half = smem + kOffQ + (u16 >> 3) * kQHalf;
        if (c < nqk) {
          *reinterpret_cast<uint4*>(half + sw128_off(c, u16 & 7)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(half + sw128_off(nqk + c, u16 & 7)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
      TILE_STAMP(trace && tid == 0, 61, globaltimer());
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&m.q_ready);
      TILE_STAMP(trace && tid == 0, 5, globaltimer());
    }

    // =================== passes over this CTA's tiles ===================
    const int row = qd * 32 + lane;  // key row within the tile
    const int gw = p.G < 16 ? p.G : 16;                  // columns per query in this chunk
    const int qa = c0 >> gshift;                         // first chunk query (chunk-local)
    const int nqa = p.G < 16 ? (16 >> gshift) : 1;       // queries in this chunk
    const uint32_t qmask_w = (gw == 32) ? 0xFFFFFFFFu : ((1u << gw) - 1u);
    const uint32_t colvalid = ncols - c0 >= 16 ? 0xFFFFu : (ncols > c0 ? ((1u << (ncols - c0)) - 1u) : 0u);
    const int bar_chunk = kBarChunk0 + ck;               // named barrier of this chunk's 4 warps
    // REUSE: the index rows are staged at once, so the union is built after
    // the first compressed tile (whose K and V stages are then free for the
    // first token tiles) rather than after the last (debug bit 6: after the
    // last, for A/B timing)
    const bool union_early = p.idx_early != 0 && !(p.debug_flags & (8 | 64));
    bool union_seen = false;
    int T = 0x7fffffff;
    int J0 = 0;  // tiles of earlier passes (mbarrier phase base)
    float lacc[3];  // row sums of this warp's quadrant: lanes 2c, 2c+1 hold column c0 + c
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      const bool robust = pass > 0;
      if (robust) {
        named_bar_sync(kBarRedo, kThreads);  // every role has seen the redo decision
        if (tid == 0) m.flag = 0;
      }
      named_bar_sync(kBarSoft, kSoftThreads);  // every column's mref is written
      // running max / threshold: fast = fixed reference, robust = -inf (lazy raise)
      for (int i = tid; i < 3 * kCols; i += kSoftThreads) {
        const float r = m.mref[i % kCols];
        (&m.m2[0][0])[i] = robust ? -INFINITY : r;
        (&m.thr[0][0])[i] = robust ? -INFINITY : r + kFastHi;
      }
      {  // zero the O accumulators (hi and lo columns) of this warp's lanes / columns
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        if (active) {
#pragma unroll
          for (int br = 0; br < 3; ++br) {
            tmem_st16(lanebase + kTmemO + kTmemStride * br + c0, z);
            tmem_st16(lanebase + kTmemO + kTmemStride * br + kCols + c0, z);
          }
        }
        tmem_wait_st();
      }
#pragma unroll
      for (int br = 0; br < 3; ++br) lacc[br] = 0.f;
      named_bar_sync(kBarSoft, kSoftThreads);
      bool ovf = false;       // fast pass: an active logit above mref + kFastHi
      uint32_t act_ab = 0u;   // fast pass: active columns, cmp (bits 0-15) / slc (16-31)
      uint32_t act_w = 0u;    //            and win (bits 0-15), of this lane
#pragma unroll 1
      for (int j = 0; active; ++j) {
        const int t = split + j * S;
        if (!union_seen && (t >= n_cmp || (union_early && j == 1))) {  // the token tiles need the union
          coop_union(m, tid, nqc, p.n_sel, p.l_sel, p.rows, cwlo, cwhi);
          TILE_STAMP(trace && tid == 0, 1, globaltimer());
#ifdef SPECSV_TRACE_TILES
          if ((p.debug_flags & 32) && trace && tid == 0) {  // check: a sequential recount of the union
            int bad = 0, cnt = 0, prev = -1;
            const int nsel = (p.rows + p.l_sel - 1) / p.l_sel;
            for (int b = 0; b < nsel; ++b) {
              bool in = (b * p.l_sel <= cwhi) && (b * p.l_sel + p.l_sel - 1 >= cwlo);
              for (int e = 0; e < nqc * p.n_sel && !in; ++e) in = m.qsel[e] == b;
              if (in) {
                if (cnt < m.n_union && m.union_blk[cnt] != b) bad |= 1;
                ++cnt;
              }
            }
            for (int u = 0; u < m.n_union; ++u) {
              if (m.union_blk[u] <= prev) bad |= 2;
              prev = m.union_blk[u];
            }
            if (cnt != m.n_union) bad |= 4;
            p.trace[cta_id * 64 + 63] = 1000 + bad;
          }
#endif
          union_seen = true;
          T = tile_count();
        }
        if (union_seen && j >= T) break;
#ifdef SPECSV_TRACE_TILES
        const bool cs = trace && tid == 0 && j == 3 && !robust;  // cycle stamps of one tile
        const long long cb = cs ? clock64() : 0;
#endif
        const int J = J0 + j;
        const int sb = J & 1;
        const TileInfo ti = tile_info(m, n_cmp, t, cwlo, cwhi, p.l_sel);
        // per-(row, query) masks for the queries of this chunk -> 16-bit column masks
        uint32_t cm_a = 0u, cm_b = 0u;
        if (ti.kind == kTileCmp) {
          const int i = ti.base + row;
#pragma unroll 4
          for (int k = 0; k < nqa; ++k) {
            const int qi = qa + k;
            if (qi < nqc && i < m.qmvis[qi]) cm_a |= qmask_w << (k * gw);
          }
        } else if (ti.kind == kTileTok) {
          const int u = ti.base + (row >> 6);
          if (u < m.n_union) {
            const int tok = m.union_blk[u] * p.l_sel + (row & 63);
            const uint32_t own = m.union_own[u];
#pragma unroll 4
            for (int k = 0; k < nqa; ++k) {
              const int qi = qa + k;
              if (qi >= nqc) break;
              if (((own >> qi) & 1u) && tok < m.qbound[qi]) cm_a |= qmask_w << (k * gw);
              if (tok >= m.qwlo[qi] && tok <= m.qwhi[qi]) cm_b |= qmask_w << (k * gw);
            }
          }
        } else {
#pragma unroll 4
          for (int k = 0; k < nqa; ++k) {
            const int qg = q0 + qa + k;
            if (qa + k < nqc && qg >= 1 && row < 64 && ((p.tree_mask[qg - 1] >> row) & 1ull))
              cm_b |= qmask_w << (k * gw);
          }
        }
        cm_a &= colvalid;
        cm_b &= colvalid;
        if (!ti.act_a) cm_a = 0u;
        if (!ti.act_b) cm_b = 0u;
        // S^T rows of this quadrant, this warp's 16 columns (log2 units): hi + lo halves
        float s[16];
        TILE_STAMP(cs, 29, clock64() - cb);
        mbar_sleep_wait(&m.s_full[sb], (J >> 1) & 1);
        TILE_STAMP(cs, 30, clock64() - cb);
        TILE_STAMP(trace && tid == 0 && j < 8 && !robust, 24 + j, globaltimer());
        tc_fence_after();
        {
          uint32_t rh[16], rl[16];
          const uint32_t sa = lanebase + kTmemS + kTmemStride * sb + c0;
          tmem_ld16(sa, rh);
          tmem_ld16(sa + nqk, rl);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) s[e] = __uint_as_float(rh[e]) + __uint_as_float(rl[e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&m.s_free[sb]);
        TILE_STAMP(cs, 31, clock64() - cb);

        if (!robust) {
          // ---- fast pass: one exp per element, shared by both branches ----
          float pe[16];
          const uint32_t cm = cm_a | cm_b;
          float mx = -INFINITY;
          const float4* mr4 = reinterpret_cast<const float4*>(&m.mref[c0]);
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const float4 r4 = mr4[e4];
            const float mr[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float d = s[4 * e4 + e] - mr[e];
              mx = fmaxf(mx, ((cm >> (4 * e4 + e)) & 1u) ? d : -INFINITY);
              pe[4 * e4 + e] = fast_exp2(d);
            }
          }
          ovf |= mx > kFastHi;
          if (ti.kind == kTileCmp) act_ab |= cm_a; else act_ab |= cm_a << 16;
          act_w |= cm_b;
          TILE_STAMP(trace && tid == 0 && j < 8, 48 + j, globaltimer());
          // the P region is rewritten only after the previous tile's PV read it
          TILE_STAMP(cs, 37, clock64() - cb);
          if (J > 0 && (ti.act_a || ti.act_b)) mbar_sleep_wait(&m.pv_done[(J - 1) & 1], ((J - 1) >> 1) & 1);
          TILE_STAMP(cs, 38, clock64() - cb);
          if (ti.act_a)
            write_p(smem + kOffP, row, c0, 0, cm_a, pe, lacc[ti.kind == kTileCmp ? kCmp : kSlc], lane);
          if (ti.act_b) write_p(smem + kOffP, row, c0, ti.act_a ? 2 * kCols : 0, cm_b, pe, lacc[kWin], lane);
          TILE_STAMP(cs, 39, clock64() - cb);
        } else {
          // ---- robust pass: lazy running max per active branch; the 4 warps
          // sharing this column chunk vote (columns are independent across chunks)
          bool resc[2] = {false, false};
#pragma unroll 1
          for (int side = 0; side < 2; ++side) {
            if (!(side == 0 ? ti.act_a : ti.act_b)) continue;  // CTA-uniform
            const int br = side == 0 ? (ti.kind == kTileCmp ? kCmp : kSlc) : kWin;
            const uint32_t cm = side == 0 ? cm_a : cm_b;
            bool need = false;
#pragma unroll
            for (int e = 0; e < 16; ++e) need |= ((cm >> e) & 1u) && (s[e] > m.thr[br][c0 + e]);
            const bool any_w = __any_sync(0xffffffffu, need);
            if (lane == 0) m.vote[qd][ck] = any_w ? 1 : 0;
            named_bar_sync(bar_chunk, 128);
            const int any = m.vote[0][ck] | m.vote[1][ck] | m.vote[2][ck] | m.vote[3][ck];
            named_bar_sync(bar_chunk, 128);
            if (!any) continue;
            resc[side] = true;
            float v[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = ((cm >> e) & 1u) ? s[e] : -INFINITY;
            const float mxv = reduce16<true>(v, lane);
            if ((lane & 1) == 0) m.tmax[qd][c0 + (lane >> 1)] = mxv;
            named_bar_sync(bar_chunk, 128);
            if (qd == 0 && lane < 16) {
              const int c = c0 + lane;
              const float old = m.m2[br][c];
              const float tm = fmaxf(fmaxf(m.tmax[0][c], m.tmax[1][c]), fmaxf(m.tmax[2][c], m.tmax[3][c]));
              const float nw = tm > old ? tm : old;
              m.alpha[c] = (nw == old) ? 1.f : (old == -INFINITY ? 0.f : fast_exp2(old - nw));
              m.m2[br][c] = nw;
              m.thr[br][c] = nw + kRescaleThresh;
            }
            named_bar_sync(bar_chunk, 128);
            // O^T (hi and lo columns) and the row sums of this chunk *= alpha,
            // once the previous tile's MMAs into them are complete
            if (j > 0) mbar_sleep_wait(&m.pv_done[(J - 1) & 1], ((J - 1) >> 1) & 1);
            tc_fence_after();
            float al[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) al[e] = m.alpha[c0 + e];
#pragma unroll
            for (int hl = 0; hl < 2; ++hl) {
              const uint32_t ta = lanebase + kTmemO + kTmemStride * br + (hl ? kCols : 0) + c0;
              uint32_t r[16];
              tmem_ld16(ta, r);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * al[e]);
              tmem_st16(ta, r);
            }
            tmem_wait_st();
            lacc[br] *= m.alpha[c0 + (lane >> 1)];
            named_bar_sync(bar_chunk, 128);  // alpha is reused by the other side
          }
          if (J > 0 && (ti.act_a || ti.act_b) && !resc[0] && !resc[1])  // the P region is free
            mbar_sleep_wait(&m.pv_done[(J - 1) & 1], ((J - 1) >> 1) & 1);
#pragma unroll 1
          for (int side = 0; side < 2; ++side) {
            if (!(side == 0 ? ti.act_a : ti.act_b)) continue;
            const int br = side == 0 ? (ti.kind == kTileCmp ? kCmp : kSlc) : kWin;
            float pe[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) pe[e] = fast_exp2(s[e] - m.m2[br][c0 + e]);
            write_p(smem + kOffP, row, c0, (side == 1 && ti.act_a) ? 2 * kCols : 0, side == 0 ? cm_a : cm_b,
                    pe, lacc[br], lane);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&m.p_full[J & 1]);
        TILE_STAMP(cs, 47, clock64() - cb);
        TILE_STAMP(trace && tid == 0 && j < 8 && !robust, 32 + j, globaltimer());
      }
      if (!union_seen) {  // a warp without columns: it still takes part in the union build, once
        coop_union(m, tid, nqc, p.n_sel, p.l_sel, p.rows, cwlo, cwhi);
        union_seen = true;
        T = tile_count();
      }
      TILE_STAMP(trace && tid == 0 && !robust, 2, globaltimer());
      // ---- end of pass: branch row sums, then the fast-pass check ----
      if ((lane & 1) == 0) {
#pragma unroll
        for (int br = 0; br < 3; ++br) m.lred[br][qd][c0 + (lane >> 1)] = lacc[br];
      }
      if (!robust) {
        const uint32_t ab = __reduce_or_sync(0xffffffffu, act_ab);
        const uint32_t wb = __reduce_or_sync(0xffffffffu, act_w);
        if (lane == 0) {
          m.actw[warp][0] = ab;
          m.actw[warp][1] = wb;
        }
        if (__any_sync(0xffffffffu, ovf) && lane == 0) atomicOr(&m.flag, 2);
      }
      named_bar_sync(kBarSoft, kSoftThreads);
      if (!robust && tid < 3 * kCols) {  // one (branch, column) per thread
        const int br = tid / kCols, c = tid % kCols, ckc = c >> 4;
        const int bit = (br == kWin ? 0 : 16 * br) + (c & 15);
        const int wd = br == kWin ? 1 : 0;
        const uint32_t a = m.actw[4 * ckc][wd] | m.actw[4 * ckc + 1][wd] | m.actw[4 * ckc + 2][wd] |
                           m.actw[4 * ckc + 3][wd];
        const float L = m.lred[br][0][c] + m.lred[br][1][c] + m.lred[br][2][c] + m.lred[br][3][c];
        if (((a >> bit) & 1u) && !(L >= 0x1p-48f && L < 0x1p+100f)) atomicOr(&m.flag, 4);
      }
      // the O accumulators are final once the last PV of the pass completed
      if (active && T > 0) mbar_sleep_wait(&m.pv_done[(J0 + T - 1) & 1], ((J0 + T - 1) >> 1) & 1);
      TILE_STAMP(trace && tid == 0 && !robust, 7, globaltimer());
      named_bar_sync(kBarPassEnd, kThreads);  // pass end: the redo decision is visible to every role
      TILE_STAMP(trace && tid == 0, 62 + pass, (unsigned long long)m.flag);
      if (!m.flag) break;
      J0 += T;
    }
    // ---- epilogue: partial (m, l, O = O_hi + O_lo) of this split -> workspace ----
    // The previous launch triggers its dependents after its tile loop, so it
    // may still be merging out of the workspace (and counters) this launch
    // writes from here on: wait for it to complete.  Its completion implies
    // its own predecessor's (it waited here too), so the chain is ordered.
    griddep_wait();
    tc_fence_after();
    const int64_t unit = ((int64_t)chunk * p.Hkv + kvh) * S + split;  // partial slot
    float* ws_ml = p.ws + unit * (3 * kCols * 2);
    float* ws_o = p.ws + p.ws_o_offset + unit * (3 * kCols * kDh);
    for (int i = tid; i < 3 * kCols; i += kSoftThreads) {
      const int br = i / kCols, c = i % kCols;
      ws_ml[2 * i] = m.m2[br][c];
      ws_ml[2 * i + 1] = m.lred[br][0][c] + m.lred[br][1][c] + m.lred[br][2][c] + m.lred[br][3][c];
    }
    if (active) {
#pragma unroll 1
      for (int br = 0; br < 3; ++br) {
        uint32_t rh[16], rl[16];
        const uint32_t ta = lanebase + kTmemO + kTmemStride * br + c0;
        tmem_ld16(ta, rh);
        tmem_ld16(ta + kCols, rl);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (c0 + e < ncols)
            ws_o[((int64_t)br * kCols + c0 + e) * kDh + row] = __uint_as_float(rh[e]) + __uint_as_float(rl[e]);
      }
    }
    TILE_STAMP(trace && tid == 0, 3, globaltimer());
  } else if (warp == kWarpTma) {
    // =================== TMA producer ===================
    // One thread polls: a K stage frees at its tile's QK, well before the V
    // stage of the same tile frees at its PV, so K and V loads go out
    // independently, each as soon as its stage is free (a blocking in-order
    // issue would hold the next K behind the previous V).  The first stages
    // went out in the prologue; token tiles wait for the union.
    int T = 0x7fffffff;
    if (lane == 0) {
      const int jtok = n_cmp > split ? (n_cmp - split + S - 1) / S : 0;  // first token tile
      int nk = pre, nv = pre;
      bool known = false;
      for (;;) {
        if (!known && (nk >= jtok || nv >= jtok) && mbar_test_wait(&m.union_ready, 0)) {
          known = true;
          T = tile_count();
        }
        const int lim = known ? T : jtok;
        if (known && nk >= T && nv >= T) break;
        bool any = false;
        if (nk < lim && (nk < 2 || mbar_test_wait(&m.k_empty[nk & 1], ((nk >> 1) + 1) & 1))) {
          issue(split + nk * S, nk, 0);
          TILE_STAMP(trace && (nk == 2 || nk == 3), nk == 2 ? 56 : 60, globaltimer());
          ++nk;
          any = true;
        }
        if (nv < lim && (nv < 2 || mbar_test_wait(&m.v_empty[nv & 1], ((nv >> 1) + 1) & 1))) {
          TILE_STAMP(trace && nv == 2, 57, globaltimer());
          issue(split + nv * S, nv, 1);
          TILE_STAMP(trace && nv == 2, 58, globaltimer());
          ++nv;
          any = true;
        }
        if (!any && (p.debug_flags & 128)) __nanosleep(20);
      }
    }
    __syncwarp();
    T = __shfl_sync(0xffffffffu, T, 0);
    named_bar_sync(kBarPassEnd, kThreads);
    if (m.flag) {  // robust redo: the same tiles again
      named_bar_sync(kBarRedo, kThreads);
      if (lane == 0)
        for (int j = 0; j < T; ++j) {
          issue(split + j * S, T + j, 0);
          issue(split + j * S, T + j, 1);
        }
      __syncwarp();
      named_bar_sync(kBarPassEnd, kThreads);
    }
  } else if (warp != kWarpUnion) {
    // =================== MMA issuers: QK^T warp and PV warp ===================
    // (two issuing threads so a QK waiting for its K tile never delays the PV
    // of the previous tile; each commit tracks only its own thread's MMAs)
    bool union_seen = false;
    int T = 0x7fffffff;
    auto tiles = [&](int j) {
      if (split + j * S >= n_cmp && !union_seen) {
        mbar_backoff_wait(&m.union_ready, 0, !(p.debug_flags & 8));
        union_seen = true;
        T = tile_count();
      }
      return j < T;
    };
    // one MMA per 16-element K step, hi and lo stacked along N; PV: one or two
    // branches (N = 96 / 192, O_slc and O_win adjacent in TMEM)
    const uint32_t idesc_qk = idesc_bf16(128, 2 * nqk, 0, 0);
    const uint32_t idesc_pv1 = idesc_bf16(128, 2 * kCols, 1, 1);
    const uint32_t idesc_pv2 = idesc_bf16(128, 4 * kCols, 1, 1);
    static_assert(kTmemO + kTmemStride * kSlc + kTmemStride == kTmemO + kTmemStride * kWin, "O_slc | O_win");
    auto qk_pass = [&](int J0) {
      for (int j = 0; tiles(j); ++j) {
        const int J = J0 + j;
        const int sb = J & 1;
        if (J >= 2) mbar_sleep_wait(&m.s_free[sb], ((J >> 1) + 1) & 1);
        mbar_sleep_wait(&m.k_full[sb], (J >> 1) & 1);
        TILE_STAMP(trace && J < 8, 16 + J, globaltimer());
        tc_fence_after();
        const uint32_t kaddr = sbase + kOffK + sb * kStageBytes;
        const uint32_t qaddr = sbase + kOffQ;
        const uint32_t d = tmem + kTmemS + kTmemStride * sb;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint32_t qoff = (kk >> 2) * kQHalf + (kk & 3) * 32;
          umma_f16(d, desc_sw128(kaddr + koff, 16, 1024), desc_sw128(qaddr + qoff, 16, 1024),
                   idesc_qk, kk != 0);
        }
        umma_commit(&m.s_full[sb]);
        umma_commit(&m.k_empty[sb]);  // the K stage is free once its QK is done
      }
    };
    auto pv_pass = [&](int J0) {
      for (int j = 0; tiles(j); ++j) {
        const int J = J0 + j;
        const int st = J & 1;
        mbar_sleep_wait(&m.p_full[J & 1], (J >> 1) & 1);
        const TileInfo ti = tile_info(m, n_cmp, split + j * S, cwlo, cwhi, p.l_sel);
        mbar_sleep_wait(&m.v_full[st], (J >> 1) & 1);
        TILE_STAMP(trace && J < 8, 40 + J, globaltimer());
        tc_fence_after();
        const uint32_t vaddr = sbase + kOffV + st * kStageBytes;
        if (ti.act_a || ti.act_b) {
          const uint32_t pa = sbase + kOffP;
          const int br = ti.act_a ? (ti.kind == kTileCmp ? kCmp : kSlc) : kWin;
          const uint32_t d = tmem + kTmemO + kTmemStride * br;
          const uint32_t idesc = (ti.act_a && ti.act_b) ? idesc_pv2 : idesc_pv1;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_f16(d, desc_sw128(vaddr + kk * 2048, 16384, 1024),
                     desc_sw128(pa + kk * 2048, 16384, 1024), idesc, 1u);
        }
        umma_commit(&m.pv_done[J & 1]);
        umma_commit(&m.v_empty[st]);
      }
    };
    if (lane == 0) {
      mbar_sleep_wait(&m.q_ready, 0);
      tc_fence_after();
      if (warp == kWarpQk) qk_pass(0); else pv_pass(0);
    }
    __syncwarp();
    named_bar_sync(kBarPassEnd, kThreads);
    if (m.flag) {
      named_bar_sync(kBarRedo, kThreads);
      if (lane == 0) {
        tc_fence_after();
        if (warp == kWarpQk) qk_pass(T); else pv_pass(T);
      }
      __syncwarp();
      named_bar_sync(kBarPassEnd, kThreads);
    }
  } else {
    // =================== union warp: the index rows ===================
    // (an L2 prefetch of this CTA's later tiles from here was measured and
    // removed: with the evict-first stage loads it cost ~4% of the step)
    const UnionArgs ua = union_args(p, q0, nqc, lane);
    const bool early = p.idx_early != 0 && !(p.debug_flags & 8);
    zero_union(m, nqc, ua.n, ua.l_sel, ua.rows, cwlo, cwhi, lane);
    if (early) stage_index_rows(ua, m, nqc, lane);
    // REFRESH: the index rows come from the routing launch just before this
    // one (programmatic dependent launch: the rest of this CTA -- q, the
    // compressed tiles -- does not wait for it).  REUSE: they were complete
    // before the previous launch started, and this launch writes nothing the
    // previous one still reads (it triggers after its last workspace read),
    // so they are staged at once, under the compressed tiles.
    if (!early) {
      griddep_wait();
      stage_index_rows(ua, m, nqc, lane);
    }
    cp_async_wait_all();
    __syncwarp();
    TILE_STAMP(trace && lane == 0, 59, globaltimer());
    mbar_arrive(&m.rows_ready);  // the softmax warps build the union from them
    named_bar_sync(kBarPassEnd, kThreads);
    if (m.flag) {
      named_bar_sync(kBarRedo, kThreads);
      named_bar_sync(kBarPassEnd, kThreads);
    }
  }

  // ---- merge of the split partials (per-head barrier) + gated combine ----
  // Every CTA past its tile loop: the next launch may start placing CTAs (its
  // launch latency and prologue run under this merge).  It reads only its
  // inputs before its own epilogue's wait (nsa_verify.h, programmatic
  // dependent launch).  Debug bit 8 (256): trigger after the merge instead.
  const bool late_trigger = (p.debug_flags & 256) != 0;
  if (!late_trigger) griddep_launch();
  tc_fence_before();
  if (S > 1) {
    int* sync = reinterpret_cast<int*>(p.ws + p.ws_sync_offset) + 2 * (chunk * p.Hkv + kvh);
    group_barrier(sync, sync + 1, S, tid);
    TILE_STAMP(trace && tid == 0, 6, globaltimer());
  } else {
    __syncthreads();
  }
  if (warp < kSoftWarps) {
    // 384 threads = 2 columns x 3 branches x 64 threads of 2 d_head lanes each:
    // every load of a column pair is in flight at once (one round trip); the
    // branch contributions meet in shared memory and are summed in branch
    // order (gated_combine, nsa_attention.cpp:239-251)
    const int64_t unit0 = ((int64_t)chunk * p.Hkv + kvh) * S;
    const int task = tid >> 6, l64 = tid & 63;
    const int cpair = task / 3, br = task % 3;
    float2* contrib = reinterpret_cast<float2*>(smem + kOffK);  // [2][3][64]: the K stages are idle now
    for (int c0m = split; c0m < ncols; c0m += 2 * S) {
      const int c = c0m + cpair * S;
      const bool live = c < ncols;
      float2 res = make_float2(0.f, 0.f);
      if (live) {
        const int qg = q0 + (c >> gshift);
        const int h = kvh * p.G + (c & (p.G - 1));
        const float g = p.gates[((int64_t)qg * p.Hq + h) * 3 + br];
        float mv[kMaxSplits], lv[kMaxSplits];
        float2 ov[kMaxSplits];
#pragma unroll
        for (int s2 = 0; s2 < kMaxSplits; ++s2) {  // all loads in flight at once
          if (s2 < S) {
            const float2 ml = *reinterpret_cast<const float2*>(
                p.ws + (unit0 + s2) * (3 * kCols * 2) + 2 * (br * kCols + c));
            mv[s2] = ml.x;
            lv[s2] = ml.y;
            ov[s2] = *reinterpret_cast<const float2*>(
                p.ws + p.ws_o_offset + (unit0 + s2) * (3 * kCols * kDh) + ((int64_t)br * kCols + c) * kDh + 2 * l64);
          } else {
            mv[s2] = -INFINITY;
            lv[s2] = 0.f;
            ov[s2] = make_float2(0.f, 0.f);
          }
        }
        float M = -INFINITY;
#pragma unroll
        for (int s2 = 0; s2 < kMaxSplits; ++s2)
          if (lv[s2] > 0.f) M = fmaxf(M, mv[s2]);
        if (M != -INFINITY) {  // an empty branch contributes 0 (nsa_attention.cpp:244)
          float L = 0.f;
          float2 O = make_float2(0.f, 0.f);
#pragma unroll
          for (int s2 = 0; s2 < kMaxSplits; ++s2) {
            const float f = lv[s2] > 0.f ? fast_exp2(mv[s2] - M) : 0.f;
            L += lv[s2] * f;
            O.x += ov[s2].x * f;
            O.y += ov[s2].y * f;
          }
          if (L > 0.f) res = make_float2(g * (O.x / L), g * (O.y / L));
        }
      }
      named_bar_sync(kBarSoft, kSoftThreads);  // the previous pair's contributions are consumed
      contrib[(cpair * 3 + br) * 64 + l64] = res;
      named_bar_sync(kBarSoft, kSoftThreads);
      if (live && br == 0) {
        const float2 a0 = contrib[(cpair * 3 + 0) * 64 + l64], a1 = contrib[(cpair * 3 + 1) * 64 + l64],
                     a2 = contrib[(cpair * 3 + 2) * 64 + l64];
        const int qg = q0 + (c >> gshift);
        const int h = kvh * p.G + (c & (p.G - 1));
        *reinterpret_cast<float2*>(p.out + ((int64_t)qg * p.Hq + h) * kDh + 2 * l64) =
            make_float2((a0.x + a1.x) + a2.x, (a0.y + a1.y) + a2.y);
      }
    }
    TILE_STAMP(trace && tid == 0, 4, globaltimer());
  }
  tc_fence_before();
  __syncthreads();
  if (late_trigger) griddep_launch();
  if (warp == kWarpTma) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    nsa_attend_kernel(const __grid_constant__ AttendParams p) {
  attend_cta(p, blockIdx.x, p.kvh0 + blockIdx.y, blockIdx.z,
             (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
}

// Many requests of one layer in one launch (specsv_nsa_verify_batched): grid
// (splits, Hkv, requests x chunks).  With fewer splits per head the fixed
// per-launch costs (prologue, split merge) amortise over the requests; at one
// split per head there is no cross-CTA merge and the grid may span waves.
__global__ void __launch_bounds__(kThreads, 1)
    nsa_attend_batch_kernel(const __grid_constant__ AttendBatch b) {
  const int r = blockIdx.z / b.n_chunks, chunk = blockIdx.z % b.n_chunks;
  if (r >= b.n_req) return;
  const AttendParams& p = b.req[r];
  if (chunk * p.qc_size >= p.nq) return;  // this request has fewer query chunks
  if ((int)blockIdx.y >= p.nkvh) return;   // this request attends fewer KV heads
  attend_cta(p, blockIdx.x, p.kvh0 + blockIdx.y, chunk,
             (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
}

}  // namespace

size_t attend_smem_bytes() { return kOffMisc + sizeof(Misc) + 1024; }

bool pdl_enabled() { return !debug_env().no_pdl; }

size_t attend_workspace_floats(int n_chunks, int hkv, int n_splits) {
  const size_t units = (size_t)n_chunks * hkv * n_splits;
  return units * (3 * kCols * 2) + units * (3 * kCols * kDh);  // split partials (m, l), O
}

// the dynamic shared-memory opt-in of a kernel, once per device
template <class K>
cudaError_t smem_opt_in(K* kernel, size_t bytes, std::atomic<int>* done) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& d = done[dev < 64 ? dev : 63];
  if (d.load(std::memory_order_acquire)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) d.store(1, std::memory_order_release);
  return e;
}
std::atomic<int> g_attend_batch_smem[64], g_attend_smem[64];

cudaError_t launch_attend_batch(const AttendBatch& b, int n_splits, int n_heads, bool cooperative,
                                cudaStream_t stream) {
  cudaError_t e = smem_opt_in(nsa_attend_batch_kernel, attend_smem_bytes(), g_attend_batch_smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_splits, n_heads, b.n_req * b.n_chunks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = attend_smem_bytes();
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  // split CTAs of a head meet at a barrier (the host checks the grid fits the
  // device); under programmatic dependent launch the attribute is dropped as
  // in launch_attend below
  if (cooperative && (!pdl_enabled() || debug_env().attend_coop)) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na++].val.cooperative = 1;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, nsa_attend_batch_kernel, b);
}

cudaError_t launch_attend(const AttendParams& p, int n_chunks, cudaStream_t stream) {
  static_assert(kDh == 128, "d_head");
  cudaError_t e = smem_opt_in(nsa_attend_kernel, attend_smem_bytes(), g_attend_smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_splits, p.nkvh, n_chunks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = attend_smem_bytes();
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  // split CTAs of a head meet at a barrier, so the grid must be co-resident
  // (the host checks it fits the device).  Under programmatic dependent launch
  // the attribute is dropped: CTAs are then placed as the previous launch's
  // CTAs retire (a refresh layer's attend streams its compressed tiles under
  // the routing tail), and every CTA still becomes resident because nothing
  // the previous launch waits on depends on this grid.
  const bool coop = p.n_splits > 1 && (!pdl_enabled() || debug_env().attend_coop);
  if (coop) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na++].val.cooperative = 1;
  }
  if (pdl_enabled()) {  // starts while the previous launch's last CTAs finish
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, nsa_attend_kernel, p);
}

int attend_max_coresident() {
  cudaFuncSetAttribute(nsa_attend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)attend_smem_bytes());
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nsa_attend_kernel, kThreads,
                                                attend_smem_bytes());
  cudaGetLastError();
  return sms * per_sm;
}

}  // namespace specsv_b200
