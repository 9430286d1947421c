// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exports the oracle C API (nsa_oracle.h) implemented by calling the
// reference's own C++ functions, compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/.  No
// reference source is copied here; this file only adapts flat arrays to the
// reference's types and replays the per-layer section of run_target_pass
// (engine.cpp:175-278) with the same calls in the same order.
#include <cmath>
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <vector>

#include "nsa_oracle.h"
#include "specsv/kernels.hpp"
#include "specsv/nsa/attention.hpp"
#include "specsv/nsa/cache.hpp"
#include "specsv/nsa/config.hpp"
#include "specsv/rng.hpp"
#include "specsv/schedule/layer_roles.hpp"
#include "specsv/verify/group_attend.hpp"

using namespace specsv;

namespace {

nsa::NsaConfig to_cfg(const or_config* c) {
  nsa::NsaConfig cfg;
  cfg.l = c->l;
  cfg.d = c->d;
  cfg.l_sel = c->l_sel;
  cfg.n = c->n;
  cfg.w = c->w;
  cfg.n_q_heads = c->n_q_heads;
  cfg.n_kv_heads = c->n_kv_heads;
  cfg.d_head = c->d_head;
  cfg.n_layers = c->n_layers;
  cfg.routing_lag = c->routing_lag;
  return cfg;
}

nsa::LayerKv make_kv(const nsa::NsaConfig& cfg, const float* k, const float* v, int64_t rows) {
  nsa::LayerKv kv(cfg.n_kv_heads, cfg.d_head);
  const size_t n = static_cast<size_t>(rows * cfg.n_kv_heads * cfg.d_head);
  kv.k.assign(k, k + n);
  kv.v.assign(v, v + n);
  kv.rows = rows;
  return kv;
}

nsa::CompressedLayer make_cc(const nsa::NsaConfig& cfg, const float* ck, const float* cv,
                             int64_t blocks, int64_t source_rows) {
  nsa::CompressedLayer cc;
  cc.n_kv_heads = cfg.n_kv_heads;
  cc.d_head = cfg.d_head;
  cc.block_count = blocks;
  cc.source_rows = source_rows;
  const size_t n = static_cast<size_t>(blocks * cfg.n_kv_heads * cfg.d_head);
  cc.k.assign(ck, ck + n);
  cc.v.assign(cv, cv + n);
  return cc;
}

void store_partials(const std::vector<nsa::BranchPartial>& parts, int64_t dh, double* out) {
  for (size_t h = 0; h < parts.size(); ++h) {
    double* p = out + h * (dh + 2);
    std::memcpy(p, parts[h].out.data(), sizeof(double) * dh);
    p[dh] = parts[h].run_max;
    p[dh + 1] = parts[h].run_den;
  }
}

nsa::BranchPartial load_partial(int64_t dh, const double* p) {
  nsa::BranchPartial b(dh);
  std::memcpy(b.out.data(), p, sizeof(double) * dh);
  b.run_max = p[dh];
  b.run_den = p[dh + 1];
  return b;
}

}  // namespace

extern "C" {

const char* or_impl_name(void) { return "reference"; }

int or_validate(const or_config* c) {
  try {
    to_cfg(c).validate();
  } catch (const std::invalid_argument&) {
    return OR_EINVAL;
  }
  return OR_OK;
}

uint64_t or_rng_fill_symmetric(uint64_t state, float a, float* out, int64_t count) {
  // Rng keeps its state private; replay through a fresh stream per call and
  // report the advanced state the same way the generator does.
  Rng rng(state);
  for (int64_t i = 0; i < count; ++i) out[i] = rng.next_symmetric(a);
  return state + static_cast<uint64_t>(count) * 0x9e3779b97f4a7c15ull;
}

double or_dot_f32(const float* a, const float* b, int64_t n) {
  return kernels::active().dot_f32(a, b, static_cast<size_t>(n));
}

int64_t or_compressed_block_count(int64_t n_rows, const or_config* c) {
  return nsa::compressed_block_count(n_rows, to_cfg(c));
}

int64_t or_build_compressed(const or_config* c, const float* k, const float* v,
                            int64_t committed_len, const float* pe, float* ck, float* cv) {
  const auto cfg = to_cfg(c);
  auto kv = make_kv(cfg, k, v, committed_len);
  auto cc = nsa::build_compressed_layer(kv, committed_len, cfg, pe);
  std::memcpy(ck, cc.k.data(), sizeof(float) * cc.k.size());
  std::memcpy(cv, cc.v.data(), sizeof(float) * cc.v.size());
  return cc.block_count;
}

int64_t or_selection_scores(const or_config* c, const float* q, const float* ck, int64_t blocks,
                            int64_t visible_len, double* scores) {
  const auto cfg = to_cfg(c);
  auto cc = make_cc(cfg, ck, ck, blocks, 0);
  auto s = nsa::selection_scores(q, cc, visible_len, cfg);
  std::memcpy(scores, s.data(), sizeof(double) * s.size());
  return static_cast<int64_t>(s.size());
}

int64_t or_select_blocks(const or_config* c, const double* scores, int64_t n,
                         int64_t visible_len, const int64_t* forced, int64_t n_forced,
                         int64_t* idx_out, uint8_t* forced_out) {
  const auto cfg = to_cfg(c);
  const int64_t avail = nsa::selection_block_count(visible_len, cfg);
  std::vector<double> s(scores, scores + (avail > 0 ? avail : 0));
  nsa::SelectedIndexSet r =
      forced == nullptr
          ? nsa::select_blocks(s, n, visible_len, cfg)
          : nsa::select_blocks(s, n, visible_len, cfg, std::span<const int64_t>(forced, n_forced));
  for (size_t i = 0; i < r.indices.size(); ++i) {
    idx_out[i] = r.indices[i];
    if (forced_out) forced_out[i] = r.forced[i] ? 1 : 0;
  }
  return static_cast<int64_t>(r.indices.size());
}

void or_branch_compressed(const or_config* c, const float* q, const float* ck, const float* cv,
                          int64_t blocks, int64_t visible_len, double* partial) {
  const auto cfg = to_cfg(c);
  auto cc = make_cc(cfg, ck, cv, blocks, 0);
  store_partials(nsa::branch_attend_compressed(q, cc, visible_len, cfg), cfg.d_head, partial);
}

void or_branch_selected(const or_config* c, const float* q, const float* k, const float* v,
                        int64_t rows, const int64_t* blocks, int64_t n_blocks,
                        const uint8_t* ownership, int64_t token_bound, double* partial) {
  const auto cfg = to_cfg(c);
  auto kv = make_kv(cfg, k, v, rows);
  std::vector<bool> own;
  if (ownership) own.assign(ownership, ownership + n_blocks);
  store_partials(nsa::branch_attend_selected(q, kv, std::span<const int64_t>(blocks, n_blocks),
                                             ownership ? &own : nullptr, token_bound, cfg),
                 cfg.d_head, partial);
}

void or_branch_window(const or_config* c, const float* q, const float* k, const float* v,
                      int64_t rows, int64_t pos, int64_t committed_len, const float* tree_k,
                      const float* tree_v, const int32_t* admitted, int64_t n_admitted,
                      double* partial) {
  const auto cfg = to_cfg(c);
  auto kv = make_kv(cfg, k, v, rows);
  nsa::LayerKv scratch(cfg.n_kv_heads, cfg.d_head);
  nsa::TreeRowsView view;
  int64_t max_row = -1;
  for (int64_t i = 0; i < n_admitted; ++i) max_row = std::max<int64_t>(max_row, admitted[i]);
  if (tree_k != nullptr) {
    scratch = make_kv(cfg, tree_k, tree_v, max_row + 1);
    view.scratch = &scratch;
    view.admitted = std::span<const int32_t>(admitted, n_admitted);
  }
  store_partials(nsa::branch_attend_window(q, kv, pos, cfg.w, committed_len,
                                           tree_k ? &view : nullptr, cfg),
                 cfg.d_head, partial);
}

void or_merge_partials(int64_t dh, const double* a, const double* b, double* r) {
  auto m = nsa::merge_partials(load_partial(dh, a), load_partial(dh, b));
  std::memcpy(r, m.out.data(), sizeof(double) * dh);
  r[dh] = m.run_max;
  r[dh + 1] = m.run_den;
}

void or_gated_combine(int64_t dh, const double* cmp, const double* slc, const double* win,
                      const double* g, double* out) {
  nsa::GateVector gv{g[0], g[1], g[2]};
  auto o = nsa::gated_combine(load_partial(dh, cmp), load_partial(dh, slc), load_partial(dh, win),
                              gv);
  std::memcpy(out, o.data(), sizeof(double) * dh);
}

int64_t or_merged_schedule(const int64_t* sets, const int64_t* counts, int64_t n_sets,
                           int64_t stride, int64_t* uniq, uint8_t* own) {
  std::vector<nsa::SelectedIndexSet> v(n_sets);
  for (int64_t s = 0; s < n_sets; ++s) v[s].indices.assign(sets + s * stride, sets + s * stride + counts[s]);
  auto sched = verify::merged_schedule(v);
  const int64_t nu = static_cast<int64_t>(sched.unique_blocks.size());
  for (int64_t i = 0; i < nu; ++i) uniq[i] = sched.unique_blocks[i];
  if (own)
    for (int64_t s = 0; s < n_sets; ++s)
      for (int64_t i = 0; i < nu; ++i) own[s * nu + i] = sched.ownership[s][i] ? 1 : 0;
  return nu;
}

int64_t or_representative_index(const int64_t* positions, int64_t n) {
  std::vector<verify::MemberQuery> ms(n);
  for (int64_t i = 0; i < n; ++i) ms[i].pos = positions[i];
  try {
    return verify::representative_index(ms);
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

int64_t or_clamp_inherited(const or_config* c, const int64_t* src, const uint8_t* src_forced,
                           int64_t count, int64_t causal_bound, int64_t* out,
                           uint8_t* out_forced) {
  nsa::SelectedIndexSet s;
  s.indices.assign(src, src + count);
  if (src_forced)
    for (int64_t i = 0; i < count; ++i) s.forced.push_back(src_forced[i] != 0);
  auto r = schedule::clamp_inherited_indices(s, causal_bound, to_cfg(c));
  for (size_t i = 0; i < r.indices.indices.size(); ++i) {
    out[i] = r.indices.indices[i];
    if (out_forced) out_forced[i] = r.indices.forced[i] ? 1 : 0;
  }
  return static_cast<int64_t>(r.indices.indices.size());
}

int or_verify_layer(const or_config* c, const float* k, const float* v, int64_t rows,
                    const float* ck, const float* cv, int64_t blocks, const float* tree_k,
                    const float* tree_v, int64_t nq, const float* q, const int64_t* pos,
                    const double* gates, const uint64_t* tree_mask, int64_t mask_words,
                    int64_t C, int mode, int role, int64_t* idx, int64_t* idx_count,
                    uint8_t* idx_forced, double* out, or_stats* st) {
  try {
    const auto cfg = to_cfg(c);
    cfg.validate();
    const int64_t gamma = nq - 1, h = cfg.n_q_heads * cfg.d_head, n = cfg.n;
    const bool approx = mode == OR_MODE_APPROX;
    auto kv = make_kv(cfg, k, v, rows);
    auto cc = make_cc(cfg, ck, cv, blocks, rows);
    nsa::LayerKv scratch(cfg.n_kv_heads, cfg.d_head);
    if (gamma > 0) scratch = make_kv(cfg, tree_k, tree_v, gamma);

    std::vector<std::vector<nsa::GateVector>> gv(nq, std::vector<nsa::GateVector>(cfg.n_q_heads));
    for (int64_t qi = 0; qi < nq; ++qi)
      for (int64_t hh = 0; hh < cfg.n_q_heads; ++hh) {
        const double* g = gates + (qi * cfg.n_q_heads + hh) * 3;
        gv[qi][hh] = nsa::GateVector{g[0], g[1], g[2]};
      }
    std::vector<std::vector<int32_t>> admitted(nq);
    for (int64_t i = 0; i < gamma; ++i)
      for (int64_t j = 0; j < gamma; ++j)
        if ((tree_mask[i * mask_words + j / 64] >> (j % 64)) & 1ull)
          admitted[1 + i].push_back(static_cast<int32_t>(j));

    const auto groups = verify::partition_groups(gamma, C);
    std::vector<std::optional<nsa::SelectedIndexSet>> pass(nq);

    // routing, engine.cpp:176-197
    auto route = [&](int64_t qi) {
      const int64_t vis = cfg.routing_visible_len(pos[qi]);
      auto scores = nsa::selection_scores(q + qi * h, cc, vis, cfg);
      return nsa::select_blocks(scores, cfg.n, vis, cfg);
    };
    const bool reuse = role == OR_ROLE_REUSE;
    if (!reuse) {
      pass[0] = route(0);
      if (!approx) {
        for (int64_t qi = 1; qi < nq; ++qi) pass[qi] = route(qi);
      } else {
        for (const auto& g : groups) {
          std::vector<verify::MemberQuery> probe(g.size());
          for (int64_t i = 0; i < g.size(); ++i) probe[i].pos = pos[1 + g.begin + i];
          const int64_t rep = verify::representative_index(probe);
          pass[1 + g.begin + rep] = route(1 + g.begin + rep);
        }
      }
    } else {
      // engine.cpp:198-208
      for (int64_t qi = 0; qi < nq; ++qi) {
        if (idx_count[qi] < 0) continue;
        nsa::SelectedIndexSet src;
        src.indices.assign(idx + qi * n, idx + qi * n + idx_count[qi]);
        for (int64_t i = 0; i < idx_count[qi]; ++i) src.forced.push_back(idx_forced[qi * n + i] != 0);
        auto clamped =
            schedule::clamp_inherited_indices(src, cfg.routing_visible_len(pos[qi]), cfg);
        pass[qi] = std::move(clamped.indices);
      }
    }
    for (int64_t qi = 0; qi < nq; ++qi) {
      for (int64_t i = 0; i < n; ++i) idx[qi * n + i] = -1;
      if (!pass[qi].has_value()) {
        idx_count[qi] = -1;
        continue;
      }
      idx_count[qi] = static_cast<int64_t>(pass[qi]->indices.size());
      for (int64_t i = 0; i < idx_count[qi]; ++i) {
        idx[qi * n + i] = pass[qi]->indices[i];
        idx_forced[qi * n + i] = pass[qi]->forced[i] ? 1 : 0;
      }
    }
    if (!pass[0].has_value()) return OR_ESTATE;

    verify::GroupAttendContext ctx{&kv, &cc, &cfg};
    {
      verify::MemberQuery rm;
      rm.q = q;
      rm.pos = pos[0];
      rm.routing_bound = cfg.routing_visible_len(pos[0]);
      rm.indices = &*pass[0];
      rm.gates = gv[0];
      auto rr = verify::attend_one(ctx, rm, rm.indices->indices, nullptr);
      std::memcpy(out, rr.out.data(), sizeof(double) * h);
    }
    verify::LoadStats total;
    for (const auto& g : groups) {
      if (!approx) {
        for (int64_t i = 0; i < g.size(); ++i)
          if (!pass[1 + g.begin + i].has_value()) return OR_ESTATE;
      } else {
        std::vector<verify::MemberQuery> probe(g.size());
        for (int64_t i = 0; i < g.size(); ++i) probe[i].pos = pos[1 + g.begin + i];
        if (!pass[1 + g.begin + verify::representative_index(probe)].has_value()) return OR_ESTATE;
      }
    }
    for (const auto& g : groups) {
      std::vector<verify::MemberQuery> members(g.size());
      for (int64_t i = 0; i < g.size(); ++i) {
        const int64_t qi = 1 + g.begin + i;
        auto& mm = members[i];
        mm.q = q + qi * h;
        mm.pos = pos[qi];
        mm.routing_bound = cfg.routing_visible_len(pos[qi]);
        mm.indices = pass[qi].has_value() ? &*pass[qi] : nullptr;
        mm.gates = gv[qi];
        mm.intra.scratch = &scratch;
        mm.intra.admitted = admitted[qi];
      }
      auto gres = approx ? verify::group_attend_approx(ctx, members)
                         : verify::group_attend_exact(ctx, members);
      if (reuse) gres.stats.index_constructions = 0;
      total.add(gres.stats);
      for (int64_t i = 0; i < g.size(); ++i)
        std::memcpy(out + (1 + g.begin + i) * h, gres.members[i].out.data(), sizeof(double) * h);
    }
    std::memset(st, 0, sizeof(*st));
    st->unique_block_loads = total.unique_block_loads;
    st->total_requested_loads = total.total_requested_loads;
    st->dedup_savings = total.dedup_savings;
    st->window_token_loads = total.window_token_loads;
    st->launches = total.launches;
    st->index_constructions = total.index_constructions;
    st->n_pairs = std::min<int64_t>(OR_MAX_PAIRS, total.pairwise_overlap.size());
    for (int64_t i = 0; i < st->n_pairs; ++i) st->pairwise_overlap[i] = total.pairwise_overlap[i];
    return OR_OK;
  } catch (const std::invalid_argument&) {
    return OR_EINVAL;
  }
}

}  // extern "C"
