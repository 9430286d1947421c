/*
 * nsa_verify.h -- C-ABI drop-in boundary of the B200-native sparse
 * speculative-verification hot path (NSA over a chain/tree of draft queries).
 *
 * Library: paper_2605_19893_b200/lib/libspecsv_b200.so (sm_100a).
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   specsv_nsa_verify          the per-layer hot section of run_target_pass,
 *                              src/engine.cpp:175-278 (routing | clamp, root
 *                              attend_one, group_attend_exact/approx)
 *   specsv_nsa_route           nsa::selection_scores + nsa::select_blocks,
 *                              include/specsv/nsa/attention.hpp:29-44 (the
 *                              paper's "routing launch")
 *   specsv_nsa_attend_fused    verify::group_attend_exact / group_attend_approx
 *                              / attend_one, include/specsv/verify/group_attend.hpp:50-66
 *                              (compressed + selected + window branches and
 *                              nsa::gated_combine, attention.hpp:46-95)
 *   specsv_compress_append     nsa::extend_compressed_layer,
 *                              include/specsv/nsa/cache.hpp:91-97
 *   specsv_resolve_layer_roles schedule::resolve_layer_roles, layer_roles.hpp:45
 *   specsv_clamp_inherited     schedule::clamp_inherited_indices, layer_roles.hpp:56-57
 *   specsv_load_stats          verify::LoadStats accounting, grouping.hpp:33-52
 *
 * Conventions: plain pointers and sizes only.  "device" pointers are CUDA
 * global memory; "host" pointers are CPU memory.  All entry points are
 * stream-ordered, allocate nothing, keep no global mutable state and are
 * re-entrant across streams and devices.  Errors are returned as
 * specsv_status; specsv_last_error() gives a thread-local message (the
 * reference throws std::invalid_argument for the same conditions,
 * config.hpp:39-50, group_attend.cpp:12,94,126, layer_roles.cpp:20-22).
 *
 * Programmatic dependent launch: the routing and attend kernels are enqueued
 * with programmatic stream serialization, so a call's first kernel may start
 * -- and read its inputs (q, gates, the KV caches, the draft rows, on REUSE
 * the index sets) -- as soon as the kernel enqueued just before it has
 * triggered programmatic completion (griddepcontrol.launch_dependents), not
 * only once it has finished.  This library's own kernels trigger before
 * their last writes and every kernel of it waits (griddepcontrol.wait) for
 * its predecessor's completion before writing anything a predecessor may
 * still touch: routing triggers before its index-set writes, which the
 * attend launch of the same call waits for; attend triggers after its tile
 * loop, before its split merge and its OUTPUT writes.  So a verify call's
 * inputs must not be the output of the verify call enqueued just before it
 * (a kernel or event in between -- e.g. the next layer's projection --
 * orders them as usual).  Kernels that never trigger (ordinary CUDA/PyTorch
 * kernels) complete first, as usual.  A caller whose own producer kernel
 * triggers early, before writing a verify input, must not enqueue it
 * directly before a verify call -- or set SPECSV_NO_PDL=1, which turns the
 * attribute off.
 */
#ifndef SPECSV_B200_NSA_VERIFY_H
#define SPECSV_B200_NSA_VERIFY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPECSV_ABI_VERSION 3  /* 2: specsv_layer_kv.capacity, verify-args KV-head range;
                                 3: specsv_layer_kv.ckd / ckexp (routing digit planes) */

typedef struct CUstream_st* specsv_stream_t; /* == cudaStream_t */

typedef enum specsv_status {
  SPECSV_OK = 0,
  SPECSV_EINVAL = 1,       /* config / argument violates the reference's rules */
  SPECSV_ESTATE = 2,       /* missing index set (reuse source / approx representative) */
  SPECSV_EUNSUPPORTED = 3, /* valid for the reference, not for this sm_100a build */
  SPECSV_ECUDA = 4,        /* CUDA launch / runtime failure */
  SPECSV_ENOSPACE = 5      /* workspace too small */
} specsv_status;

/* NsaConfig, include/specsv/nsa/config.hpp:24-34 (same fields, same meaning) */
typedef struct specsv_nsa_config {
  int64_t l;           /* compression block length */
  int64_t d;           /* compression stride */
  int64_t l_sel;       /* selection block size */
  int64_t n;           /* selected block count (top-n incl. forced) */
  int64_t w;           /* sliding window */
  int64_t n_q_heads;
  int64_t n_kv_heads;
  int64_t d_head;
  int64_t n_layers;
  int64_t routing_lag;
} specsv_nsa_config;

/* CoarseningMode (plan/strategy.hpp:33-34) */
enum { SPECSV_MODE_EXACT = 0, SPECSV_MODE_APPROX = 1 };
/* LayerRole (schedule/layer_roles.hpp:16) */
enum { SPECSV_ROLE_REFRESH = 0, SPECSV_ROLE_REUSE = 1 };

/* One layer's device-resident caches: LayerKv (cache.hpp:15-44, row-major
 * [row][kv_head][d_head], here bf16) plus CompressedLayer (cache.hpp:60-82,
 * [block][kv_head][d_head]).  The pending root's row is part of `rows`
 * (engine.cpp:160-161 appends it before attention). */
typedef struct specsv_layer_kv {
  const void* k;        /* device bf16 [>= rows][Hkv][dh] */
  const void* v;        /* device bf16 [>= rows][Hkv][dh] */
  int64_t rows;         /* committed rows c */
  float* ck;            /* device fp32 [>= blocks][Hkv][dh]  (routing keys, bit-exact pooling) */
  void* ck16;           /* device bf16 [>= blocks][Hkv][dh]  (bf16 copy for the compressed branch) */
  void* cv;             /* device bf16 [>= blocks][Hkv][dh]  (pooled values) */
  int64_t blocks;       /* compressed blocks built over `rows`: (rows - l) / d + 1 */
  int64_t capacity;     /* rows the k / v buffers hold (>= rows); ck / ck16 / cv hold
                           (capacity - l) / d + 1 blocks.  Appends and commits are
                           bounds-checked against it (the reference asserts on the
                           same invariant, cache.hpp:26-30) */
  void* ckd;            /* device int8 [>= blocks][Hkv][4][dh], or NULL: the routing keys as
                           fixed-point digits -- byte s of element x is the base-256 digit
                           of weight 256^s of round(ck[x] * 2^(30 - e)), e = ckexp, digits
                           in [-128, 127].  Written by specsv_compress_append next to ck;
                           the integer tensor-pipe routing kernel streams these planes
                           (NULL selects the fp64 routing kernel over ck) */
  int32_t* ckexp;       /* device [>= blocks][Hkv]: bits 0-15 (signed) e with max_x |ck[x]| <
                           2^e (0 for an all-zero row), bits 16-23 how many of the row's
                           elements the 2^(e-30) grid rounds (the routing error bound);
                           NULL iff ckd is NULL */
} specsv_layer_kv;

/* One verify call: one layer x one request, root + gamma draft queries in
 * flat order (FlatBatch, tree/draft_tree.hpp:41-48). */
typedef struct specsv_verify_args {
  int32_t n_queries;          /* 1 + gamma; query 0 is the pending root */
  int32_t group_size;         /* C (StrategyTuple.group_size) */
  int32_t mode;               /* SPECSV_MODE_* */
  int32_t role;               /* SPECSV_ROLE_* */
  const int64_t* pos;         /* host [nq] absolute positions (c-1, c-1+depth_i) */
  const uint64_t* tree_mask;  /* host [gamma][mask_words]; bit j of row i = mask[i][j]
                                 (ancestor-or-self, draft_tree.cpp:126-141) */
  int32_t mask_words;         /* ceil(gamma / 64) */
  const float* q;             /* device fp32 [nq][Hq][dh] */
  const float* gates;         /* device fp32 [nq][Hq][3] = (g_cmp, g_slc, g_win) */
  const void* tree_k;         /* device bf16 [gamma][Hkv][dh], flat order */
  const void* tree_v;
  int32_t* idx;               /* device [nq][n] ascending, -1 padded.  REFRESH: written.
                                 REUSE: read (the source layer's sets, unclamped) */
  int32_t* idx_count;         /* device [nq]; -1 = no set (approx non-representatives) */
  uint32_t* idx_forced;       /* device [nq]; bit i = idx[q][i] is a forced block (i < 32:
                                 with n > 32 later positions are not flagged; the attend
                                 path does not read the mask) */
  float* out;                 /* device fp32 [nq][Hq][dh] gated-combine output */
  int32_t kv_head_begin;      /* KV-head group sharding: attend only KV heads
                                 [kv_head_begin, kv_head_begin + kv_head_count) and write
                                 only their q heads' rows of `out`; routing (REFRESH) still
                                 scores every head (the reference sums the selection mass
                                 over all Hq heads, nsa_attention.cpp:51-63), so q and gates
                                 stay full-size.  kv_head_count = 0: all heads */
  int32_t kv_head_count;
} specsv_verify_args;

/* LoadStats (grouping.hpp:33-52), group-summed over the draft queries of one
 * layer exactly as Engine::step reports them (engine.hpp:45). */
#define SPECSV_MAX_PAIRS 128
typedef struct specsv_load_stats_t {
  int64_t unique_block_loads;
  int64_t total_requested_loads;
  int64_t dedup_savings;
  int64_t window_token_loads;
  int64_t launches;
  int64_t index_constructions;
  int64_t n_pairs;
  int64_t pairwise_overlap[SPECSV_MAX_PAIRS];
} specsv_load_stats_t;

/* ---- library ----------------------------------------------------------- */
int32_t specsv_abi_version(void);
const char* specsv_last_error(void);
/* NsaConfig::validate (config.hpp:38-51) plus this build's limits. */
specsv_status specsv_validate_config(const specsv_nsa_config* cfg);

/* Bytes of device workspace one verify call needs.  The caller allocates it,
 * zero-fills it ONCE before first use and then reserves it for this library
 * (it holds split partials and per-head barrier words that return to a
 * consistent state after every call).  One workspace per stream. */
size_t specsv_verify_workspace_size(const specsv_nsa_config* cfg, int32_t n_queries,
                                    int64_t max_rows);

/* Workspace for specsv_nsa_verify_batched that routes up to `batch` (<= 16)
 * REFRESH requests in one launch (each needs its own routing regions).  Any
 * workspace of at least specsv_verify_workspace_size works; a larger one lets
 * more requests share a routing launch. */
size_t specsv_verify_workspace_size_batched(const specsv_nsa_config* cfg, int32_t n_queries,
                                            int64_t max_rows, int32_t batch);

/* ---- the hot path ------------------------------------------------------ */
/* Full per-layer verify: REFRESH = routing launch(es) + fused downstream
 * launch; REUSE = one fully fused launch. */
specsv_status specsv_nsa_verify(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                                const specsv_verify_args* args, void* workspace,
                                size_t workspace_bytes, specsv_stream_t stream);

/* The same over `batch` independent requests (one layer each). */
specsv_status specsv_nsa_verify_batched(const specsv_nsa_config* cfg, const specsv_layer_kv* kvs,
                                        const specsv_verify_args* args, int32_t batch,
                                        void* workspace, size_t workspace_bytes,
                                        specsv_stream_t stream);

/* Routing only: fp64 compressed-block scores + Top-n with forced blocks for
 * the queries that construct indices (all in EXACT mode; root + group
 * representatives in APPROX mode).  Writes args->idx / idx_count / idx_forced. */
specsv_status specsv_nsa_route(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                               const specsv_verify_args* args, void* workspace,
                               size_t workspace_bytes, specsv_stream_t stream);

/* Attention only (compressed + selected + window + gate combine) over the
 * index sets in args->idx, clamped per query at its routing bound. */
specsv_status specsv_nsa_attend_fused(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                                      const specsv_verify_args* args, void* workspace,
                                      size_t workspace_bytes, specsv_stream_t stream);

/* Debug/parity: fp64 selection scores (selection_scores, nsa_attention.cpp:38-80)
 * for query `query` of args into device `scores` [ceil(rows / l_sel)]. */
specsv_status specsv_nsa_scores(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                                const specsv_verify_args* args, int32_t query, double* scores,
                                void* workspace, size_t workspace_bytes, specsv_stream_t stream);

/* Top-n over caller-provided fp64 scores (select_blocks, nsa_attention.cpp:94-136):
 * scores device [avail]; writes idx device [n], count device [1], forced device [1]. */
specsv_status specsv_select_blocks(const specsv_nsa_config* cfg, const double* scores,
                                   int64_t visible_len, int32_t* idx, int32_t* count,
                                   uint32_t* forced, specsv_stream_t stream);

/* ---- cache maintenance -------------------------------------------------- */
/* extend_compressed_layer (nsa_cache.cpp:45-66): pools blocks
 * [first_block, last_block) from kv->k / kv->v with fp64 accumulation in the
 * reference's order, writing ck (fp32, bit-exact), ck16 and cv (bf16 RNE).
 * pos_embed: device fp32 [l][dh] or NULL. */
specsv_status specsv_compress_append(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                                     int64_t first_block, int64_t last_block,
                                     const float* pos_embed, specsv_stream_t stream);

/* ---- host policy (C++), same rules as the reference ----------------------- */
/* resolve_layer_roles (layer_roles.cpp:11-35): roles[j] in SPECSV_ROLE_*,
 * source[j] = nearest preceding refresh layer. */
specsv_status specsv_resolve_layer_roles(const int64_t* reuse_set, int64_t n_reuse,
                                         int64_t n_layers, int32_t* roles, int64_t* source);
/* clamp_inherited_indices (layer_roles.cpp:37-50); returns kept count via *out_count */
specsv_status specsv_clamp_inherited(const specsv_nsa_config* cfg, const int32_t* src,
                                     uint32_t src_forced, int32_t count, int64_t causal_bound,
                                     int32_t* out, uint32_t* out_forced, int32_t* out_count);
/* LoadStats of one layer from HOST copies of the index sets (after clamping
 * on reuse layers), the positions and the tree mask; mirrors
 * group_attend_exact/approx (group_attend.cpp:87-139) and engine.cpp:272-275. */
specsv_status specsv_load_stats(const specsv_nsa_config* cfg, int64_t rows, int32_t n_queries,
                                const int64_t* pos, const uint64_t* tree_mask,
                                int32_t mask_words, int32_t group_size, int32_t mode,
                                int32_t role, const int32_t* idx, const int32_t* idx_count,
                                specsv_load_stats_t* out);
/* Algorithmic HBM bytes of one verify call in this build's storage format
 * (DESIGN.md "Algorithmic bytes"): compressed K/V of the widest visible
 * range, the union over all queries of selected and window tokens (bf16
 * K+V, all KV heads), draft rows, q/gates/out; routing adds fp32 ck. */
specsv_status specsv_algorithmic_bytes(const specsv_nsa_config* cfg, int64_t rows,
                                       int32_t n_queries, const int64_t* pos, int32_t role,
                                       const int32_t* idx, const int32_t* idx_count,
                                       int32_t mode, int32_t group_size, int64_t* bytes);

/* ---- diagnostics ------------------------------------------------------- */
/* Per-thread (host thread) debug hook: when `buf` is a device pointer, the
 * next fused-attend launches write per-CTA globaltimer stamps [cta][8]
 * (start, setup done, tile loop done, partials written, merge done); NULL
 * disables.  Not used on the product path. */
specsv_status specsv_debug_attend_trace(unsigned long long* buf);

/* int32 index into a verify workspace of the routing kernel's cumulative count
 * of exact fp64 re-scorings (queries whose certified Top-n boundary fell
 * inside the score error bound); -1 on bad arguments.  Diagnostics only. */
int32_t specsv_debug_route3_counter_offset(const specsv_nsa_config* cfg, int32_t n_queries,
                                           int64_t max_rows);

#ifdef __cplusplus
}
#endif
#endif
