// draft_tree.cu -- the callers on either side of the verify call, behind
// include/specsv_b200/draft_tree.h:
//   host (C++): expand_draft_tree / flatten_tree / build_tree_mask /
//               greedy_verify (proj/src/draft_tree.cpp:45-164) over flat node
//               arrays, producing the boundary's positions and packed mask;
//   device:     the commit of accepted draft rows into every layer's
//               committed K/V (proj/src/engine.cpp:533-547) as one launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <deque>
#include <queue>
#include <string>
#include <vector>

#include "attend.h"
#include "policy.h"
#include "sm100.cuh"
#include "specsv_b200/draft_tree.h"

namespace specsv_b200 {
namespace {

// ---- tree shape checks and children lists ----------------------------------
struct Shape {
  std::vector<std::vector<int64_t>> children;  // ascending id = proposal order
};

Shape check_tree(const specsv_draft_tree* t) {
  if (t == nullptr || t->parent == nullptr || t->token == nullptr || t->depth == nullptr ||
      t->score == nullptr)
    throw Error(SPECSV_EINVAL, "null tree array");
  const int64_t n = t->n_nodes;
  if (n < 1) throw Error(SPECSV_EINVAL, "tree needs a root (n_nodes >= 1)");
  if (t->parent[0] != -1 || t->depth[0] != 0)
    throw Error(SPECSV_EINVAL, "node 0 must be the root (parent -1, depth 0)");
  Shape s;
  s.children.resize(n);
  for (int64_t i = 1; i < n; ++i) {
    const int64_t p = t->parent[i];
    if (p < 0 || p >= n || p == i)
      throw Error(SPECSV_EINVAL, "node " + std::to_string(i) + ": parent out of range");
    if (t->depth[i] != t->depth[p] + 1)
      throw Error(SPECSV_EINVAL, "node " + std::to_string(i) + ": depth != parent depth + 1");
    s.children[p].push_back(i);
  }
  return s;
}

// (score desc, id asc): the sibling order of draft_tree.cpp:88-95
std::vector<int64_t> sorted_children(const specsv_draft_tree* t, const Shape& s, int64_t id) {
  std::vector<int64_t> ch = s.children[id];
  std::sort(ch.begin(), ch.end(), [&](int64_t a, int64_t b) {
    if (t->score[a] != t->score[b]) return t->score[a] > t->score[b];
    return a < b;
  });
  return ch;
}

void fill_mask(const specsv_draft_tree* t, const int64_t* order, int64_t gamma, uint64_t* mask,
               int32_t words) {
  if (gamma < 0) throw Error(SPECSV_EINVAL, "negative gamma");
  if (gamma > 0 && (mask == nullptr || order == nullptr)) throw Error(SPECSV_EINVAL, "null output");
  if ((int64_t)words * 64 < gamma) throw Error(SPECSV_EINVAL, "mask_words < ceil(gamma / 64)");
  std::vector<int64_t> slot(t->n_nodes, -1);
  for (int64_t i = 0; i < gamma; ++i) {
    const int64_t id = order[i];
    if (id <= 0 || id >= t->n_nodes) throw Error(SPECSV_EINVAL, "order lists the root or an unknown node");
    if (slot[id] >= 0) throw Error(SPECSV_EINVAL, "order lists a node twice");
    slot[id] = i;
  }
  std::memset(mask, 0, sizeof(uint64_t) * (size_t)gamma * (size_t)words);
  for (int64_t i = 0; i < gamma; ++i)
    for (int64_t cur = order[i]; cur > 0; cur = t->parent[cur]) {  // root is not in the batch
      const int64_t j = slot[cur];
      if (j < 0) throw Error(SPECSV_EINVAL, "an ancestor of a listed node is not listed");
      mask[i * words + j / 64] |= 1ull << (j % 64);
    }
}

// ---- commit kernel -----------------------------------------------------------
constexpr int kCommitLayers = 32;  // layers per launch (param space); more = more launches
constexpr int kCommitRows = 64;    // accepted rows per call (<= depth <= routing lag in practice)

struct CommitParams {
  int n_layers, n_rows, units;  // units = 16-byte pieces of one [Hkv][dh] bf16 row
  int32_t slots[kCommitRows];
  int64_t rows[kCommitLayers];
  uint4* k[kCommitLayers];
  uint4* v[kCommitLayers];
  const uint4* tk[kCommitLayers];
  const uint4* tv[kCommitLayers];
};

// grid (accepted row, layer): one CTA copies one K row and one V row; 16-byte
// coalesced loads and stores, one pass over 2 x Hkv x dh x 2 bytes
__global__ void __launch_bounds__(128) commit_rows_kernel(const __grid_constant__ CommitParams p) {
  // (launched with programmatic dependent launch: resident under the previous
  // launch's tail, then in stream order for its inputs and the rows it writes)
  sm100::griddep_wait();
  const int i = blockIdx.x, j = blockIdx.y;
  const int64_t src = (int64_t)p.slots[i] * p.units, dst = (p.rows[j] + i) * p.units;
  for (int u = threadIdx.x; u < p.units; u += blockDim.x) {
    p.k[j][dst + u] = __ldg(p.tk[j] + src + u);
    p.v[j][dst + u] = __ldg(p.tv[j] + src + u);
  }
}

}  // namespace
}  // namespace specsv_b200

using namespace specsv_b200;

extern "C" {

specsv_status specsv_tree_expand(int32_t root_token, specsv_propose_fn propose, void* ctx,
                                 int64_t D, int64_t k, int64_t budget, int64_t capacity,
                                 int64_t* parent, int32_t* token, int32_t* depth, double* score,
                                 double* cum_score, int64_t* n_nodes) {
  return guarded([&] {
    if (propose == nullptr || parent == nullptr || token == nullptr || depth == nullptr ||
        score == nullptr || n_nodes == nullptr)
      throw Error(SPECSV_EINVAL, "null argument");
    if (D < 1 || k < 1) throw Error(SPECSV_EINVAL, "expand_draft_tree: D and k must be >= 1");
    if (capacity < 1) throw Error(SPECSV_ENOSPACE, "capacity < 1");
    struct Cand {
      int64_t parent;
      int32_t token, depth;
      double score, cum;
      int64_t seq;  // creation order: the deterministic tie-break
    };
    // best = highest cumulative score, then earliest proposal (draft_tree.cpp:39-42)
    auto worse = [](const Cand& a, const Cand& b) {
      if (a.cum != b.cum) return a.cum < b.cum;
      return a.seq > b.seq;
    };
    std::priority_queue<Cand, std::vector<Cand>, decltype(worse)> frontier(worse);
    std::vector<double> cum(1, 0.0);
    int64_t n = 1, seq = 0;
    parent[0] = -1;
    token[0] = root_token;
    depth[0] = 0;
    score[0] = 0.0;
    std::vector<int32_t> tk((size_t)k);
    std::vector<double> sc((size_t)k);
    auto propose_children = [&](int64_t id) {
      if (depth[id] >= D) return;
      const int64_t got = propose(ctx, id, token[id], depth[id], cum[id], k, tk.data(), sc.data());
      if (got < 0 || got > k) throw Error(SPECSV_EINVAL, "propose returned an invalid count");
      for (int64_t i = 0; i < got; ++i)
        frontier.push(Cand{id, tk[i], depth[id] + 1, sc[i], cum[id] + sc[i], seq++});
    };
    propose_children(0);
    const int64_t cap = budget < 0 ? INT64_MAX : budget;  // budget counts non-root nodes
    while (!frontier.empty() && n - 1 < cap) {
      const Cand c = frontier.top();
      frontier.pop();
      if (n >= capacity) throw Error(SPECSV_ENOSPACE, "tree exceeds the output capacity");
      parent[n] = c.parent;
      token[n] = c.token;
      depth[n] = c.depth;
      score[n] = c.score;
      cum.push_back(c.cum);
      ++n;
      propose_children(n - 1);
    }
    if (cum_score != nullptr) std::copy(cum.begin(), cum.end(), cum_score);
    *n_nodes = n;
  });
}

specsv_status specsv_tree_flatten(const specsv_draft_tree* tree, int32_t traversal,
                                  int64_t committed_len, int64_t* order, int64_t* positions,
                                  uint64_t* mask, int32_t mask_words) {
  return guarded([&] {
    const Shape s = check_tree(tree);
    if (traversal != SPECSV_TRAVERSAL_BFS && traversal != SPECSV_TRAVERSAL_DFS)
      throw Error(SPECSV_EINVAL, "unknown traversal");
    const int64_t gamma = tree->n_nodes - 1;
    if (gamma > 0 && (order == nullptr || positions == nullptr)) throw Error(SPECSV_EINVAL, "null output");
    int64_t g = 0;
    if (traversal == SPECSV_TRAVERSAL_BFS) {  // level order, siblings adjacent
      std::deque<int64_t> queue{0};
      while (!queue.empty()) {
        const int64_t id = queue.front();
        queue.pop_front();
        if (id != 0) order[g++] = id;
        for (int64_t c : sorted_children(tree, s, id)) queue.push_back(c);
      }
    } else {  // preorder, parent and first child adjacent
      std::vector<int64_t> stack{0};
      while (!stack.empty()) {
        const int64_t id = stack.back();
        stack.pop_back();
        if (id != 0) order[g++] = id;
        const auto ch = sorted_children(tree, s, id);
        for (auto it = ch.rbegin(); it != ch.rend(); ++it) stack.push_back(*it);
      }
    }
    for (int64_t i = 0; i < gamma; ++i) positions[i] = committed_len - 1 + tree->depth[order[i]];
    fill_mask(tree, order, gamma, mask, mask_words);
  });
}

specsv_status specsv_tree_mask(const specsv_draft_tree* tree, const int64_t* order, int64_t gamma,
                               uint64_t* mask, int32_t mask_words) {
  return guarded([&] {
    check_tree(tree);
    fill_mask(tree, order, gamma, mask, mask_words);
  });
}

specsv_status specsv_tree_greedy_accept(const specsv_draft_tree* tree,
                                        const int32_t* target_argmax, int64_t* accepted_nodes,
                                        int32_t* accepted_tokens, int64_t* n_accepted,
                                        int32_t* bonus_token) {
  return guarded([&] {
    const Shape s = check_tree(tree);
    if (target_argmax == nullptr || n_accepted == nullptr || bonus_token == nullptr)
      throw Error(SPECSV_EINVAL, "null argument");
    if (tree->n_nodes > 1 && (accepted_nodes == nullptr || accepted_tokens == nullptr))
      throw Error(SPECSV_EINVAL, "null output");
    int64_t cur = 0, na = 0;
    for (;;) {
      const int32_t want = target_argmax[cur];
      int64_t next = -1;
      for (int64_t c : s.children[cur])
        if (tree->token[c] == want) {
          next = c;  // sibling tokens are distinct: at most one matches
          break;
        }
      if (next < 0) break;
      accepted_nodes[na] = next;
      accepted_tokens[na] = tree->token[next];
      ++na;
      cur = next;
    }
    *n_accepted = na;
    *bonus_token = target_argmax[cur];
  });
}

specsv_status specsv_commit_rows(const specsv_nsa_config* cfg, const specsv_layer_kv* kvs,
                                 const void* const* tree_k, const void* const* tree_v,
                                 int32_t n_layers, const int32_t* slots, int32_t n_accepted,
                                 specsv_stream_t stream) {
  return guarded([&] {
    if (cfg == nullptr || (n_layers > 0 && (kvs == nullptr || tree_k == nullptr || tree_v == nullptr)))
      throw Error(SPECSV_EINVAL, "null argument");
    validate_config(*cfg);
    if (n_layers < 0 || n_accepted < 0) throw Error(SPECSV_EINVAL, "negative count");
    if (n_accepted > kCommitRows)
      throw Error(SPECSV_EUNSUPPORTED, "more than 64 accepted rows in one commit");
    if (n_accepted == 0 || n_layers == 0) return;
    if (slots == nullptr) throw Error(SPECSV_EINVAL, "null slots");
    const int64_t row_bytes = cfg->n_kv_heads * cfg->d_head * 2;
    if (row_bytes % 16 != 0) throw Error(SPECSV_EUNSUPPORTED, "Hkv * dh * 2 must be a multiple of 16");
    CommitParams p{};
    p.n_rows = n_accepted;
    p.units = (int)(row_bytes / 16);
    for (int32_t i = 0; i < n_accepted; ++i) {
      if (slots[i] < 0) throw Error(SPECSV_EINVAL, "negative draft slot");
      p.slots[i] = slots[i];
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    for (int32_t j0 = 0; j0 < n_layers; j0 += kCommitLayers) {
      p.n_layers = std::min(kCommitLayers, n_layers - j0);
      for (int jj = 0; jj < p.n_layers; ++jj) {
        const specsv_layer_kv& kv = kvs[j0 + jj];
        if (kv.k == nullptr || kv.v == nullptr || tree_k[j0 + jj] == nullptr || tree_v[j0 + jj] == nullptr)
          throw Error(SPECSV_EINVAL, "null cache or draft-row pointer");
        if (kv.rows < 0) throw Error(SPECSV_EINVAL, "negative rows");
        if (kv.rows + n_accepted > kv.capacity)  // LayerKv::append's assert (cache.hpp:26-30)
          throw Error(SPECSV_EINVAL, "commit exceeds the cache capacity");
        p.rows[jj] = kv.rows;
        p.k[jj] = reinterpret_cast<uint4*>(const_cast<void*>(kv.k));
        p.v[jj] = reinterpret_cast<uint4*>(const_cast<void*>(kv.v));
        p.tk[jj] = reinterpret_cast<const uint4*>(tree_k[j0 + jj]);
        p.tv[jj] = reinterpret_cast<const uint4*>(tree_v[j0 + jj]);
      }
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(n_accepted, p.n_layers);
      lc.blockDim = dim3(128);
      lc.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = pdl_enabled() ? 1 : 0;
      cudaLaunchKernelEx(&lc, commit_rows_kernel, p);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) throw Error(SPECSV_ECUDA, std::string("commit launch: ") + cudaGetErrorString(e));
    }
  });
}

specsv_status specsv_commit_rows_compress(const specsv_nsa_config* cfg, const specsv_layer_kv* kvs,
                                          const void* const* tree_k, const void* const* tree_v,
                                          int32_t n_layers, const int32_t* slots, int32_t n_accepted,
                                          const float* const* pos_embed, specsv_stream_t stream) {
  return guarded([&] {
    const specsv_status st = specsv_commit_rows(cfg, kvs, tree_k, tree_v, n_layers, slots, n_accepted, stream);
    if (st != SPECSV_OK) throw Error(st, last_error());
    if (n_accepted == 0 || n_layers == 0) return;
    if (cfg->d_head > 1024) throw Error(SPECSV_EUNSUPPORTED, "d_head too large");
    cudaStream_t sm = reinterpret_cast<cudaStream_t>(stream);
    CompressLayers c{};
    c.hkv = (int32_t)cfg->n_kv_heads;
    c.dh = (int32_t)cfg->d_head;
    c.l = (int32_t)cfg->l;
    c.d = (int32_t)cfg->d;
    for (int32_t j0 = 0; j0 < n_layers; j0 += kCompressLayers) {
      const int nl = std::min(kCompressLayers, n_layers - j0);
      int64_t max_count = 0;
      for (int jj = 0; jj < nl; ++jj) {
        const specsv_layer_kv& kv = kvs[j0 + jj];
        if (!kv.ck || !kv.ck16 || !kv.cv) throw Error(SPECSV_EINVAL, "null cache pointer");
        const int64_t rows = kv.rows + n_accepted;
        const int64_t want = rows >= cfg->l ? (rows - cfg->l) / cfg->d + 1 : 0;
        if (kv.blocks < 0 || kv.blocks > want) throw Error(SPECSV_EINVAL, "compressed block count exceeds the rows");
        c.k[jj] = kv.k;
        c.v[jj] = kv.v;
        c.pe[jj] = pos_embed != nullptr ? pos_embed[j0 + jj] : nullptr;
        c.ck[jj] = kv.ck;
        c.ck16[jj] = kv.ck16;
        c.cv[jj] = kv.cv;
        c.ckd[jj] = kv.ckd;
        c.ckexp[jj] = kv.ckexp;
        c.first[jj] = kv.blocks;
        c.count[jj] = want - kv.blocks;
        max_count = std::max(max_count, want - kv.blocks);
      }
      const cudaError_t e = launch_compress_layers(c, nl, max_count, sm);
      if (e != cudaSuccess) throw Error(SPECSV_ECUDA, std::string("compress launch: ") + cudaGetErrorString(e));
    }
  });
}

}  // extern "C"
