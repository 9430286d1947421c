// ref_tree_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Flat-array C entry points over the reference's own draft-tree utilities
// (proj/src/draft_tree.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libspecsv_ref.so): expand_draft_tree, flatten_tree and
// greedy_verify.  Used by tests/test_draft_tree.py to pin
// include/specsv_b200/draft_tree.h against the reference, and by
// tests/golden/make_tree_golden.py to write the fixtures the CPU tests keep
// when /root/reference is absent.  No reference source is copied here.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "specsv/tree/draft_tree.hpp"

using namespace specsv;

namespace {

tree::DraftTree from_arrays(int64_t n, const int64_t* parent, const int32_t* token,
                            const int32_t* depth, const double* score) {
  tree::DraftTree t;
  for (int64_t i = 0; i < n; ++i) {
    tree::DraftNode d;
    d.id = i;
    d.parent = parent[i];
    d.token = token[i];
    d.depth = depth[i];
    d.score = score[i];
    d.cum_score = parent[i] < 0 ? 0.0 : t.nodes[parent[i]].cum_score + score[i];
    t.nodes.push_back(d);
    t.children.emplace_back();
    if (parent[i] >= 0) t.children[parent[i]].push_back(i);
  }
  return t;
}

}  // namespace

extern "C" {

typedef int64_t (*or_propose_fn)(void* ctx, int64_t node_id, int32_t token, int32_t depth,
                                 double cum_score, int64_t k, int32_t* tokens, double* scores);

// 0 ok, 1 invalid argument, 5 capacity
int or_ref_tree_expand(int32_t root_token, or_propose_fn propose, void* ctx, int64_t D, int64_t k,
                       int64_t budget, int64_t capacity, int64_t* parent, int32_t* token,
                       int32_t* depth, double* score, double* cum_score, int64_t* n_nodes) {
  try {
    auto fn = [&](const tree::DraftNode& node, int64_t kk) {
      std::vector<int32_t> tk(kk);
      std::vector<double> sc(kk);
      const int64_t got = propose(ctx, node.id, node.token, node.depth, node.cum_score, kk,
                                  tk.data(), sc.data());
      std::vector<tree::TokenScore> out;
      for (int64_t i = 0; i < got; ++i) out.push_back(tree::TokenScore{tk[i], sc[i]});
      return out;
    };
    const auto t = tree::expand_draft_tree(
        root_token, fn, D, k, budget < 0 ? std::nullopt : std::optional<int64_t>(budget));
    if ((int64_t)t.nodes.size() > capacity) return 5;
    for (size_t i = 0; i < t.nodes.size(); ++i) {
      parent[i] = t.nodes[i].parent;
      token[i] = t.nodes[i].token;
      depth[i] = t.nodes[i].depth;
      score[i] = t.nodes[i].score;
      cum_score[i] = t.nodes[i].cum_score;
    }
    *n_nodes = (int64_t)t.nodes.size();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

// mask: unpacked bool bytes [gamma][gamma]
int or_ref_tree_flatten(int64_t n, const int64_t* parent, const int32_t* token, const int32_t* depth,
                        const double* score, int32_t traversal, int64_t committed_len,
                        int64_t* order, int64_t* positions, uint8_t* mask) {
  const auto t = from_arrays(n, parent, token, depth, score);
  const auto fb = tree::flatten_tree(t, traversal == 0 ? tree::Traversal::BFS : tree::Traversal::DFS,
                                     committed_len);
  for (int64_t i = 0; i < fb.gamma; ++i) {
    order[i] = fb.order[i];
    positions[i] = fb.positions[i];
    for (int64_t j = 0; j < fb.gamma; ++j) mask[i * fb.gamma + j] = fb.mask[i][j] ? 1 : 0;
  }
  return 0;
}

int or_ref_tree_greedy(int64_t n, const int64_t* parent, const int32_t* token, const int32_t* depth,
                       const double* score, const int32_t* argmax, int64_t* nodes, int32_t* tokens,
                       int64_t* n_accepted, int32_t* bonus) {
  try {
    const auto t = from_arrays(n, parent, token, depth, score);
    const auto vr = tree::greedy_verify(t, std::span<const int32_t>(argmax, (size_t)n));
    for (size_t i = 0; i < vr.accepted_nodes.size(); ++i) {
      nodes[i] = vr.accepted_nodes[i];
      tokens[i] = vr.accepted_tokens[i];
    }
    *n_accepted = (int64_t)vr.accepted_nodes.size();
    *bonus = vr.bonus_token;
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

}  // extern "C"
