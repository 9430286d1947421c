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
constexpr int kMaxUnion = 1024;      // union blocks per chunk
constexpr int kMaxUnionWords = 1024; // selection-block bitmap words (32768 blocks)

struct AttendParams {
  CUtensorMap tm_k, tm_v;    // committed K/V bf16, dims (dh, Hkv, rows)
  CUtensorMap tm_ck, tm_cv;  // compressed K (bf16 copy) / V bf16, dims (dh, Hkv, blocks)
  CUtensorMap tm_tk, tm_tv;  // draft rows bf16, dims (dh, Hkv, max(gamma, 1))
  const uint16_t* k_raw;     // committed K bf16 (the fast-pass reference key row)
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
  int32_t idx_early;             // 1 (REUSE): the index rows predate the previous launch, so the
                                 // union is built without waiting for it; 0 (REFRESH): they come
                                 // from the routing launch just before (programmatic dependent launch)
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

// ---- routing on the integer tensor pipe (route3.cu) --------------------------
// Unit = (request, row chunk of <= kR3Rows (slot, head) rows, KV head, range of
// <= kR3MaxSpr selection blocks); one CTA streams the range's key-digit planes
// (<= 256 compressed blocks) once.  Logits are exact s8 x s8 -> s32 tcgen05
// products of base-256 digits of fixed-point q and keys; every probability
// uses one fixed fp64 reference (no max pass), so per-range partial sums are
// additive.  Scores carry a certified error bound, and a query whose Top-n
// boundary falls inside it is re-scored exactly in fp64.
constexpr int kR3Rows = 48;      // (slot, head) rows per unit (MMA N)
constexpr int kR3Tile = 128;     // compressed blocks per MMA tile (MMA M)
constexpr int kR3MaxBlk = 256;   // compressed blocks per unit (two tiles)
constexpr int kR3MaxSpr = 64;    // selection blocks per unit
constexpr int kR3MaxBps = 16;    // compressed blocks overlapping one selection block (host-checked)
constexpr int kR3Batch = 16;     // requests per launch
constexpr int kR3CntPerReq = 512;  // counter words per request (den arrivals, top arrivals, bounds, lock)
struct Route3Req {
  CUtensorMap tm_ckd;    // int8 digit planes, dims (dh, 4, Hkv, blocks), box 128 x 1 x 1 x 128, SW128
  const int32_t* ckexp;  // [blocks][Hkv] row exponents of the digit planes
  const float* q;        // [nq][Hq][dh]
  const float* ck;       // fp32 [blocks][Hkv][dh] (the exact re-scoring path)
  int32_t* idx;          // [nq][n]
  int32_t* idx_count;    // [nq]
  uint32_t* idx_forced;  // [nq]
  double* den;           // [nchunks][Hkv][nranges][kR3Rows] per-range denominators (token-weighted)
  double* gspill;        // [units][kR3MaxSpr][kR3Rows + 1] selection-block sums of a CTA's earlier units
  double* exact;         // [Hq][blocks] the exact path's logits / e values (scratch, one slot at a time)
  double* contrib;       // [nr][sel_pad] selection scores x Hq (the KV heads' shares, fp64 atomics;
                         // zero between launches)
  int32_t* cnt;          // [kR3CntPerReq] this request's counter set (zero-initialised, self-resetting)
  int32_t nr, nchunks, nranges, spr, blocks, avail_max, sel_pad;
  int32_t slot_q[kMaxQueries];
  int32_t slot_mvis[kMaxQueries];
  int32_t slot_avail[kMaxQueries];
  int32_t unrouted[kMaxQueries];
  int32_t n_unrouted;
};
// the launch-wide fields; the request table follows in Route3LaunchT
struct Route3Common {
  int32_t n_req;
  int32_t Hq, Hkv, G, n, l, d, l_sel;
  int32_t spc;         // slots per row chunk (chunk rows = spc x G <= kR3Rows)
  int32_t bps;         // compressed blocks overlapping one selection block (at most)
  double scale;        // 1 / sqrt(dh)
  double c_sl;         // log2(e) / sqrt(dh): logits in log2 units
  int32_t* exit_cnt;   // [2] CTAs through phase 2, tasks through their wait (the last of each
                       // resets the counters nobody polls any more); self-resetting
  int32_t* fallbacks;  // cumulative count of exact re-scorings (diagnostics; never reset)
  int32_t force_exact; // tests: re-score every query in fp64
  int32_t debug;       // diagnostics (SPECSV_ROUTE3_DEBUG): bit 0 runs the selection twice
  unsigned long long* trace;  // diagnostics: per-CTA stamps at kRouteTraceBase + cta * 16
};
// The kernel parameters of a launch over up to NR requests.  A one-request
// launch passes ~1.9 KB instead of ~33 KB: the command processor copies every
// launch's parameters, and eager per-layer calls issue one per refresh layer.
template <int NR>
struct Route3LaunchT : Route3Common {
  Route3Req req[NR];
  int32_t unit_start[NR + 1];  // units of requests < r (set at launch)
  int32_t task_start[NR + 1];  // (request, slot) Top-n tasks of requests < r
};
using Route3Launch = Route3LaunchT<kR3Batch>;  // the host's staging of any launch
cudaError_t launch_route3(Route3Launch& p, cudaStream_t stream);
int route3_grid();  // CTAs of a route3 launch on this device (one per SM)

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
  void* ckd[kCompressLayers];       // digit planes (NULL: none)
  int32_t* ckexp[kCompressLayers];
  int64_t first[kCompressLayers];
  int64_t count[kCompressLayers];
  int32_t hkv, dh, l, d;
};
cudaError_t launch_compress_layers(const CompressLayers& c, int n_layers, int64_t max_count,
                                   cudaStream_t stream);
cudaError_t launch_compress(const void* k, const void* v, const float* pe, float* ck, void* ck16,
                            void* cv, void* ckd, int32_t* ckexp, int64_t first, int64_t last, int hkv,
                            int dh, int l, int d, cudaStream_t stream);

}  // namespace specsv_b200
