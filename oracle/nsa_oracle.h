/*
 * nsa_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, fp64, -ffp-contract=off) of the reference's
 * sparse-speculative-verification hot path, used as the parity checker for
 * the B200 kernels.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_2605_19893_b200) never links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  The arithmetic order is the reference's, so on
 * identical inputs the results are bit-identical to the compiled reference
 * (pinned by tests/test_oracle_pin.py against oracle/_ref and against the
 * committed golden vectors in tests/golden/).
 *
 * The same C API is exported by oracle/ref_shim.cpp, which implements it by
 * calling the reference's own C++ functions; tests compare the two.
 */
#ifndef SPECSV_NSA_ORACLE_H
#define SPECSV_NSA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* NsaConfig, include/specsv/nsa/config.hpp:24-34 */
typedef struct or_config {
  int64_t l, d, l_sel, n, w, n_q_heads, n_kv_heads, d_head, n_layers, routing_lag;
} or_config;

/* LoadStats, include/specsv/verify/grouping.hpp:33-52 (pairwise list capped) */
#define OR_MAX_PAIRS 128
typedef struct or_stats {
  int64_t unique_block_loads, total_requested_loads, dedup_savings;
  int64_t window_token_loads, launches, index_constructions;
  int64_t n_pairs;
  int64_t pairwise_overlap[OR_MAX_PAIRS];
} or_stats;

enum { OR_MODE_EXACT = 0, OR_MODE_APPROX = 1 };
enum { OR_ROLE_REFRESH = 0, OR_ROLE_REUSE = 1 };
enum { OR_OK = 0, OR_EINVAL = 1, OR_ESTATE = 2 };

/* Identifies the implementation: "oracle-c" or "reference". */
const char* or_impl_name(void);

/* NsaConfig::validate (config.hpp:38-51); 0 when valid. */
int or_validate(const or_config* cfg);

/* splitmix64 stream (include/specsv/rng.hpp:13-44): fills `out` with
 * next_symmetric(a) draws, returns the advanced state. */
uint64_t or_rng_fill_symmetric(uint64_t state, float a, float* out, int64_t count);

/* dot_f32 canonical 4-lane order (kernels.hpp:13-18, kernels_scalar.cpp:12-26) */
double or_dot_f32(const float* a, const float* b, int64_t n);

/* compressed_block_count (cache.hpp:84-86) */
int64_t or_compressed_block_count(int64_t n_rows, const or_config* cfg);

/* build_compressed_layer / pool_block (nsa_cache.cpp:14-45).  k, v are
 * [rows][Hkv][dh]; pe is [l][dh] or NULL.  ck, cv receive
 * [block_count][Hkv][dh]; returns block_count. */
int64_t or_build_compressed(const or_config* cfg, const float* k, const float* v,
                            int64_t committed_len, const float* pe, float* ck, float* cv);

/* selection_scores (nsa_attention.cpp:38-80).  q is [Hq][dh]; ck is
 * [blocks][Hkv][dh].  Writes selection_block_count(visible_len) scores,
 * returns that count. */
int64_t or_selection_scores(const or_config* cfg, const float* q, const float* ck,
                            int64_t blocks, int64_t visible_len, double* scores);

/* select_blocks (nsa_attention.cpp:82-136).  forced == NULL derives the
 * forced set (forced_blocks, :82-92).  Writes ascending indices and forced
 * flags, returns the count. */
int64_t or_select_blocks(const or_config* cfg, const double* scores, int64_t n,
                         int64_t visible_len, const int64_t* forced, int64_t n_forced,
                         int64_t* idx_out, uint8_t* forced_out);

/* One branch for one query: partial = [Hq][dh + 2] doubles, per head
 * (out[dh], run_max, run_den).  nsa_attention.cpp:138-222. */
void or_branch_compressed(const or_config* cfg, const float* q, const float* ck, const float* cv,
                          int64_t blocks, int64_t visible_len, double* partial);
void or_branch_selected(const or_config* cfg, const float* q, const float* k, const float* v,
                        int64_t rows, const int64_t* blocks, int64_t n_blocks,
                        const uint8_t* ownership, int64_t token_bound, double* partial);
void or_branch_window(const or_config* cfg, const float* q, const float* k, const float* v,
                      int64_t rows, int64_t pos, int64_t committed_len, const float* tree_k,
                      const float* tree_v, const int32_t* admitted, int64_t n_admitted,
                      double* partial);

/* merge_partials (nsa_attention.cpp:224-237), one head: a, b, r = [dh + 2] */
void or_merge_partials(int64_t dh, const double* a, const double* b, double* r);

/* gated_combine (nsa_attention.cpp:239-251), one head: gates = {g_cmp, g_slc, g_win} */
void or_gated_combine(int64_t dh, const double* cmp, const double* slc, const double* win,
                      const double* gates, double* out);

/* merged_schedule (group_attend.cpp:20-40): sets are [n_sets][set_stride],
 * counts[n_sets].  Writes unique blocks and ownership [n_sets][n_unique]. */
int64_t or_merged_schedule(const int64_t* sets, const int64_t* counts, int64_t n_sets,
                           int64_t set_stride, int64_t* unique_out, uint8_t* ownership_out);

/* representative_index (group_attend.cpp:112-119) over positions */
int64_t or_representative_index(const int64_t* positions, int64_t n);

/* clamp_inherited_indices (layer_roles.cpp:37-50); returns kept count */
int64_t or_clamp_inherited(const or_config* cfg, const int64_t* src, const uint8_t* src_forced,
                           int64_t count, int64_t causal_bound, int64_t* out,
                           uint8_t* out_forced);

/*
 * One layer of the verify pass over 1 + gamma queries: the per-layer
 * section of run_target_pass (engine.cpp:175-278) without projections.
 *
 *   k, v      committed rows [rows][Hkv][dh] (the pending root's row included)
 *   ck, cv    compressed cache [blocks][Hkv][dh] built over `rows`
 *   tree_k/v  draft rows [gamma][Hkv][dh] in flat order (NULL when gamma == 0)
 *   q         [nq][Hq][dh], nq = 1 + gamma; query 0 is the root
 *   pos       [nq] absolute positions
 *   gates     [nq][Hq][3] (g_cmp, g_slc, g_win)
 *   tree_mask [gamma][mask_words] packed, bit j of row i = mask[i][j]
 *   idx       [nq][n] selected blocks.  REFRESH: output.  REUSE: input holding
 *             the source layer's (unclamped) sets; on return it holds the
 *             clamped sets actually used.  idx_count[q] == -1 marks "no set".
 *   out       [nq][Hq][dh] gated-combine output (fp64)
 *   stats     group-summed LoadStats of the draft queries (engine.hpp:45)
 */
int or_verify_layer(const or_config* cfg, const float* k, const float* v, int64_t rows,
                    const float* ck, const float* cv, int64_t blocks, const float* tree_k,
                    const float* tree_v, int64_t nq, const float* q, const int64_t* pos,
                    const double* gates, const uint64_t* tree_mask, int64_t mask_words,
                    int64_t group_size, int mode, int role, int64_t* idx, int64_t* idx_count,
                    uint8_t* idx_forced, double* out, or_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
