/* draft_tree.h -- the callers on either side of the verify call (SURVEY §8f
 * rows 2-3): draft-tree host utilities that produce the boundary's positions
 * and packed tree mask and consume its outputs (greedy accept), and the
 * commit of accepted draft rows into the committed KV cache.
 *
 * Replaces (reference, C++):
 *   expand_draft_tree   proj/src/draft_tree.cpp:45-82   (tree/draft_tree.hpp:61-67)
 *   flatten_tree        proj/src/draft_tree.cpp:84-124  (tree/draft_tree.hpp:69-72)
 *   build_tree_mask     proj/src/draft_tree.cpp:126-141 (tree/draft_tree.hpp:74-76)
 *   greedy_verify       proj/src/draft_tree.cpp:143-164 (tree/draft_tree.hpp:87-90)
 *   the commit loop     proj/src/engine.cpp:533-547     (LayerKv::append per layer)
 *
 * Trees cross the boundary as flat arrays (DraftTree.nodes,
 * tree/draft_tree.hpp:17-33): node 0 is the root, parent[0] = -1, and the
 * children of a node are the nodes naming it as parent in ascending id
 * (= proposal / materialisation) order.  Malformed trees (parent out of
 * range, depth[i] != depth[parent[i]] + 1, which also rules out cycles) are
 * SPECSV_EINVAL.  Host functions are pure and thread-safe. */
#ifndef SPECSV_B200_DRAFT_TREE_H_
#define SPECSV_B200_DRAFT_TREE_H_

#include <stdint.h>

#include "nsa_verify.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Traversal (tree/draft_tree.hpp:36) */
enum { SPECSV_TRAVERSAL_BFS = 0, SPECSV_TRAVERSAL_DFS = 1 };

typedef struct specsv_draft_tree {
  int64_t n_nodes;       /* root included: gamma = n_nodes - 1 */
  const int64_t* parent; /* [n_nodes]; -1 for the root */
  const int32_t* token;  /* [n_nodes] */
  const int32_t* depth;  /* [n_nodes]; root = 0 */
  const double* score;   /* [n_nodes]; draft log-probability (sibling order key) */
} specsv_draft_tree;

/* ProposeFn (tree/draft_tree.hpp:56-59): the draft model's top-k
 * continuations of node `node_id` -- distinct tokens, descending score.
 * Writes at most k (token, score) pairs and returns how many; a negative
 * return aborts the expansion with SPECSV_EINVAL. */
typedef int64_t (*specsv_propose_fn)(void* ctx, int64_t node_id, int32_t token, int32_t depth,
                                     double cum_score, int64_t k, int32_t* tokens,
                                     double* scores);

/* expand_draft_tree: best-first by cumulative score (ties by proposal
 * order), parents before children, up to depth D and width k; budget < 0 =
 * none (full k-ary expansion).  Writes the nodes into caller arrays of
 * `capacity` entries (SPECSV_ENOSPACE if the tree would not fit) and their
 * count into *n_nodes.  cum_score may be NULL. */
specsv_status specsv_tree_expand(int32_t root_token, specsv_propose_fn propose, void* ctx,
                                 int64_t D, int64_t k, int64_t budget, int64_t capacity,
                                 int64_t* parent, int32_t* token, int32_t* depth, double* score,
                                 double* cum_score, int64_t* n_nodes);

/* flatten_tree: BFS level order or DFS preorder, root excluded, siblings by
 * (score desc, id asc).  order[gamma] (node ids), positions[gamma] =
 * committed_len - 1 + depth, and the boundary's packed ancestor-or-self
 * mask [gamma][mask_words] (bit j of row i = order[j] is an ancestor-or-self
 * of order[i]; mask_words >= ceil(gamma / 64)). */
specsv_status specsv_tree_flatten(const specsv_draft_tree* tree, int32_t traversal,
                                  int64_t committed_len, int64_t* order, int64_t* positions,
                                  uint64_t* mask, int32_t mask_words);

/* build_tree_mask for an explicit ordering of the non-root nodes (every
 * non-root ancestor of a listed node must be listed: SPECSV_EINVAL otherwise). */
specsv_status specsv_tree_mask(const specsv_draft_tree* tree, const int64_t* order,
                               int64_t gamma, uint64_t* mask, int32_t mask_words);

/* greedy_verify at temperature zero: from the root, follow the child whose
 * token equals target_argmax[node] while one exists.  target_argmax covers
 * every node ([n_nodes]).  accepted_nodes / accepted_tokens need n_nodes - 1
 * entries; *n_accepted excludes the bonus token (accepted_count = n + 1). */
specsv_status specsv_tree_greedy_accept(const specsv_draft_tree* tree,
                                        const int32_t* target_argmax, int64_t* accepted_nodes,
                                        int32_t* accepted_tokens, int64_t* n_accepted,
                                        int32_t* bonus_token);

/* Commit (engine.cpp:533-547): for every layer j, copy the draft rows
 * tree_k[j][slots[i]] / tree_v[j][slots[i]] (flat slots, bf16
 * [gamma][Hkv][dh]) to committed rows kvs[j].rows + i of kvs[j].k / .v, in
 * one launch for all layers.  The caller guarantees the caches hold
 * rows + n_accepted rows, then advances kvs[j].rows and extends the
 * compressed blocks (specsv_compress_append).  slots is a HOST array. */
specsv_status specsv_commit_rows(const specsv_nsa_config* cfg, const specsv_layer_kv* kvs,
                                 const void* const* tree_k, const void* const* tree_v,
                                 int32_t n_layers, const int32_t* slots, int32_t n_accepted,
                                 specsv_stream_t stream);

/* The commit plus extend_compressed_layer of the blocks it completes
 * (nsa_cache.cpp:45-66), for every layer in two launches: kvs[j].rows and
 * .blocks are the values BEFORE the commit (the caller advances them after);
 * pos_embed: per-layer device fp32 [l][dh] pointers, or NULL. */
specsv_status specsv_commit_rows_compress(const specsv_nsa_config* cfg, const specsv_layer_kv* kvs,
                                          const void* const* tree_k, const void* const* tree_v,
                                          int32_t n_layers, const int32_t* slots, int32_t n_accepted,
                                          const float* const* pos_embed, specsv_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SPECSV_B200_DRAFT_TREE_H_ */
