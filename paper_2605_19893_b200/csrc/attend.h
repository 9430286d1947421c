// attend.h -- launch interface of the device kernels (internal to the library).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace specsv_b200 {

constexpr int kAttendCols = 48;     // query columns (queries x GQA heads) per attend CTA
constexpr int kAttendDh = 128;      // d_head of this build (host-checked)
constexpr int kMaxQueries = 65;      // 1 + gamma, gamma <= 64 (one mask word per row)
constexpr int kMaxChunkQ = 32;       // queries per CTA column chunk (64 cols / G, G >= 2)
constexpr int kMaxUnion = 1280;      // union blocks per chunk
constexpr int kMaxUnionWords = 1024; // selection-block bitmap words (32768 blocks)

struct AttendParams {
  CUtensorMap tm_k, tm_v;    // committed K/V bf16, dims (dh, Hkv, rows)
  CUtensorMap tm_ck, tm_cv;  // compressed K (bf16 copy) / V bf16, dims (dh, Hkv, blocks)
  CUtensorMap tm_tk, tm_tv;  // draft rows bf16, dims (dh, Hkv, max(gamma, 1))
  const uint16_t* k_raw;     // committed K bf16 (the fast-pass reference key row; L2 prefetch)
  const uint16_t* v_raw;     // committed V bf16 (L2 prefetch)
  const uint16_t* ck_raw;    // compressed K bf16 copy (L2 prefetch)
  const uint16_t* cv_raw;    // compressed V bf16 (L2 prefetch)
  const float* q;            // [nq][Hq][dh]
  const float* gates;        // [nq][Hq][3]
  float* out;                // [nq][Hq][dh]
  const int32_t* idx;        // [nq][n_sel]
  const int32_t* idx_count;  // [nq]
  float* ws;                 // split partials
  unsigned long long* trace; // optional per-CTA globaltimer stamps [cta][64] (debug)
  int32_t debug_flags;       // tests only (bit 0: force the robust softmax redo pass)
  int64_t ws_o_offset;       // float offset of the O partials inside ws
  int64_t ws_sync_offset;    // float offset of the per-head barrier words (zero-initialised)
  int32_t nq, gamma, Hq, Hkv, G, n_sel;
  int32_t rows, blocks, l, d, l_sel, w, lag;
  int32_t qc_size, n_splits;
  int32_t kvh0, nkvh;            // KV heads [kvh0, kvh0 + nkvh) of this call (head-group shard)
  float scale_log2;
  int32_t pos[kMaxQueries];
  int32_t src_row[kMaxQueries];  // index-set row each query attends with
  uint64_t tree_mask[kMaxQueries];
  // per-query tables (host-computed from pos; config.hpp:55-58, nsa_attention.cpp:161-222)
  int32_t qbound[kMaxQueries];   // min(routing bound, rows): selected tokens < qbound
  int32_t qwlo[kMaxQueries];     // committed window [qwlo, qwhi]
  int32_t qwhi[kMaxQueries];
  int32_t qmvis[kMaxQueries];    // visible compressed blocks
  // per-chunk tables
  int32_t ch_ncmp[kMaxQueries];  // compressed tiles of the chunk (widest visible range)
  int32_t ch_wlo[kMaxQueries];   // union of the chunk's windows
  int32_t ch_whi[kMaxQueries];
};

// Requests per batched attend launch: 8 x sizeof(AttendParams) (~3.8 KB)
// fits the 32 KB kernel-parameter space (tensor maps must stay in param space).
constexpr int kAttendBatch = 8;
// Barrier-word sets in the workspace (request r of a batched launch uses set
// r, a single-request call set 0); the region sits at a fixed workspace offset
// for a given config, so calls with different query counts can share it.
constexpr int kSyncSets = 18;
struct AttendBatch {
  AttendParams req[kAttendBatch];
  int32_t n_req, n_chunks;  // grid z = n_req x n_chunks (the widest request's chunks)
};

// programmatic dependent launch between this library's launches (default on;
// SPECSV_NO_PDL=1 turns it off for A/B timing)
bool pdl_enabled();
size_t attend_smem_bytes();
size_t attend_workspace_floats(int n_chunks, int hkv, int n_splits);  // split partials only
cudaError_t launch_attend(const AttendParams& p, int n_chunks, cudaStream_t stream);
cudaError_t launch_attend_batch(const AttendBatch& b, int n_splits, int n_heads, bool cooperative,
                                cudaStream_t stream);
int attend_max_coresident();

// ---- routing (route.cu) -------------------------------------------------------
constexpr int kRouteTile = 16;      // compressed blocks per routing statistics tile
constexpr int kMaxAvail = 8192;     // selection blocks per query for the Top-n CTA

struct RouteParams {
  const float* q;        // [nq][Hq][dh]
  const float* ck;       // fp32 [blocks][Hkv][dh]
  double* gsh;           // [nr][ntiles][Hq][g_stride] per-tile selection-block shares
  int32_t g_stride;      // selection blocks one 64-block tile touches
  double* TM;            // [nr][Hq][ntiles] tile max
  double* TD;            // [nr][Hq][ntiles] tile denominators
  double* part;          // [nr][Hkv][sel_pad] per-KV-head score shares
  int32_t sel_pad;
  int32_t* counters;     // [3] barrier words; zero-initialised, self-resetting
  int32_t* slot_done;    // [nr] finished units per slot; zero-initialised, self-resetting
  int32_t chunk_rows;    // (slot, head) rows per row chunk, a multiple of G (set at launch)
  int32_t* idx;          // [nq][n]
  int32_t* idx_count;    // [nq]
  uint32_t* idx_forced;  // [nq]
  int32_t nr, nq, Hq, Hkv, G, dh, n;
  int32_t l, d, l_sel;
  int32_t m_pad, ntiles;
  int32_t blocks;        // compressed blocks present in the cache
  double scale;          // 1 / sqrt(dh)
  int32_t slot_q[kMaxQueries];     // routed slot -> query index
  int32_t slot_mvis[kMaxQueries];  // visible compressed blocks
  int32_t slot_avail[kMaxQueries]; // selection blocks available
  int32_t unrouted[kMaxQueries];   // queries that get count = -1
  int32_t n_unrouted;
  unsigned long long* trace;  // diagnostics only: per-CTA phase stamps at kRouteTraceBase
};
constexpr int kRouteTraceBase = 196608;  // route stamps: trace[kRouteTraceBase + cta * 16 + k]

// Requests per batched routing launch (kernel-parameter space); request q
// uses its own workspace regions and counter set q (< kSyncSets).
constexpr int kRouteBatch = 16;
struct RouteBatch {
  RouteParams req[kRouteBatch];
  int32_t n_req;
  int32_t item_start[kRouteBatch + 1];  // tile work items of requests < q (set at launch)
  int32_t unit_start[kRouteBatch + 1];  // (slot, KV head) units of requests < q
};

// ---- routing, single-request fast path (route2.cu) ---------------------------
// One CTA per (KV head, row chunk, block range): the range's 16-block tiles
// stay in shared memory, the softmax statistics are combined per range, and a
// short tail (one barrier among a head's ranges, per-range score sums, per-range
// Top-n candidates, one final merge) replaces the grid-wide unit phase.
constexpr int kR2MaxTiles = 16;   // tiles (16 blocks) per range CTA (one warp each)
constexpr int kR2Rows = 40;       // (slot, head) rows per CTA
constexpr int kR2MaxRanges = 160; // >= SM count
struct Route2Params {
  CUtensorMap tm_ck;       // fp32 compressed K, dims (dh, Hkv, blocks), box 32 x 1 x 16, 128B swizzle
  const float* q;          // [nq][Hq][dh]
  const float* ck;         // fp32 [blocks][Hkv][dh]
  int32_t* idx;            // [nq][n]
  int32_t* idx_count;      // [nq]
  uint32_t* idx_forced;    // [nq]
  double* scores_out;      // diagnostics: dense scores of slot 0, no Top-n (NULL: Top-n)
  double* dm;              // [items][kR2Rows] (range max, range denominator)
  double* part;            // [nr][Hkv][sel_pad] per-KV-head score shares
  double* ovh;             // [nr][Hkv][NR][8] shares a range's last tile overhangs into the next
  double* cand_s;          // [nr][NR][64] Top-n candidates per range (score)
  int32_t* cand_i;         // [nr][NR][64] (block id)
  int32_t* cand_n;         // [nr][NR]
  int32_t* bar;            // [2 * Hkv * rc] range barrier (count, generation) per (KV head, row chunk)
  int32_t* rcnt;           // [NR] arrivals per range
  int32_t* fcnt;           // [1] finished ranges
  int32_t nr, Hq, Hkv, G, n, l, d, l_sel, blocks;
  int32_t rc, chunk_rows, NR, T, ntiles, spt, gs, sel_pad, s_total;
  double scale;            // 1 / sqrt(dh)
  int32_t slot_q[kMaxQueries], slot_mvis[kMaxQueries], slot_avail[kMaxQueries];
  int32_t unrouted[kMaxQueries];
  int32_t n_unrouted;
  unsigned long long* trace;  // diagnostics only: per-CTA phase stamps at kRouteTraceBase
  int32_t debug_exit;         // diagnostics only (timing): 0 = full kernel, k = return after phase k
};
// workspace words of route2's barriers (fixed offset per config; self-resetting)
constexpr int kR2CntInts = 2 * kR2MaxRanges + kR2MaxRanges + 8;
// shape of the range decomposition for one call; false = use route_fused_kernel
bool route2_plan(int nr, int G, int Hkv, int ntiles, int gs, int spt, int n, Route2Params& p);
size_t route2_ws_bytes(int nr, int Hkv, int sel_pad);  // dm/part/ovh/cand regions
cudaError_t launch_route2(const Route2Params& p, cudaStream_t stream);

// ---- routing on the integer tensor pipe (route3.cu, the default) -------------
// Unit = (request, KV head, row chunk of <= 48 (slot, head) rows, 128
// compressed blocks).  Logits come from exact s8 x s8 -> s32 tcgen05 products
// of base-256 digits of fixed-point q and keys; scores carry a certified error
// bound, and a query whose Top-n boundary falls inside it is re-scored in fp64.
constexpr int kR3Rows = 48;     // q rows per unit (MMA N)
constexpr int kR3Tile = 128;    // compressed blocks per unit (MMA M)
constexpr int kR3Batch = 16;    // requests per launch
constexpr int kR3MaxSpan = 64;  // selection blocks one unit touches (host-checked)
struct Route3Req {
  CUtensorMap tm_ck;     // fp32 compressed K, dims (dh, Hkv, blocks), box 128 x 1 x 128, no swizzle
  const float* q;        // [nq][Hq][dh]
  const float* ck;       // fp32 [blocks][Hkv][dh] (the exact re-scoring path)
  int32_t* idx;          // [nq][n]
  int32_t* idx_count;    // [nq]
  uint32_t* idx_forced;  // [nq]
  double* stats;         // [Hkv][nr*G][ntiles][4]: tile max (log2), tile sum, logit error bound, -
  double* gsh;           // [units][kR3Rows][span] per-unit selection-block sums (token weights)
  double* contrib;       // [nr][Hkv][ntiles][span] normalised per-KV-head shares
  double* eps;           // [nr][Hkv] logit error bound (log2 units) over the slot's rows
  int32_t nr, ntiles, nchunks, blocks;
  int32_t slot_q[kMaxQueries];
  int32_t slot_mvis[kMaxQueries];
  int32_t slot_avail[kMaxQueries];
  int32_t unrouted[kMaxQueries];
  int32_t n_unrouted;
};
struct Route3Launch {
  Route3Req req[kR3Batch];
  int32_t n_req;
  int32_t unit_start[kR3Batch + 1];  // units of requests < r (set at launch)
  int32_t task_start[kR3Batch + 1];  // (request, slot) Top-n tasks of requests < r
  int32_t Hq, Hkv, G, n, l, d, l_sel;
  int32_t chunk_rows;  // rows per unit chunk, a multiple of G (<= kR3Rows)
  int32_t spt;         // selection blocks per unit stride (kR3Tile d / l_sel)
  int32_t span;        // selection blocks one unit touches
  double scale;        // 1 / sqrt(dh)
  double c_sl;         // log2(e) / sqrt(dh): logits in log2 units
  int32_t* counters;   // [4] zero-initialised, self-resetting (grid barriers, exits)
  int32_t* fallbacks;  // cumulative count of exact re-scorings (diagnostics; never reset)
  int32_t force_exact; // tests: re-score every query in fp64
  unsigned long long* trace;  // diagnostics: per-CTA stamps at kRouteTraceBase + cta * 16
};
cudaError_t launch_route3(Route3Launch& p, cudaStream_t stream);

cudaError_t launch_route(const RouteParams& p, cudaStream_t stream, bool write_idx);
cudaError_t launch_route_batch(RouteBatch& b, cudaStream_t stream);
cudaError_t launch_scores_only(const RouteParams& p, double* scores, int slot, cudaStream_t stream);
cudaError_t launch_select(const double* scores, int avail, int n, int32_t* idx, int32_t* count,
                          uint32_t* forced, cudaStream_t stream);

// ---- compression (compress.cu) ------------------------------------------------
constexpr int kCompressLayers = 32;  // layers per batched compress launch
struct CompressLayers {
  const void* k[kCompressLayers];
  const void* v[kCompressLayers];
  const float* pe[kCompressLayers];
  float* ck[kCompressLayers];
  void* ck16[kCompressLayers];
  void* cv[kCompressLayers];
  int64_t first[kCompressLayers];
  int64_t count[kCompressLayers];
  int32_t hkv, dh, l, d;
};
cudaError_t launch_compress_layers(const CompressLayers& c, int n_layers, int64_t max_count,
                                   cudaStream_t stream);
cudaError_t launch_compress(const void* k, const void* v, const float* pe, float* ck, void* ck16,
                            void* cv, int64_t first, int64_t last, int hkv, int dh, int l, int d,
                            cudaStream_t stream);

}  // namespace specsv_b200
