// policy.cpp -- host-side C++ policy of the verify path (no device code).
//
// Same rules as the reference (paths relative to /root/reference/proj):
//   validate_config      NsaConfig::validate, include/specsv/nsa/config.hpp:38-51
//   resolve_layer_roles  src/layer_roles.cpp:11-35
//   clamp_inherited      src/layer_roles.cpp:37-50
//   representative       src/group_attend.cpp:112-119
//   load_stats           src/group_attend.cpp:87-139 + engine.cpp:272-275
#include "policy.h"
#include "attend.h"

#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace specsv_b200 {

namespace {
thread_local DebugEnv g_env;
}  // namespace

const DebugEnv& debug_env() { return g_env; }

void refresh_debug_env() {
  DebugEnv e;
  for (char** p = environ; p != nullptr && *p != nullptr; ++p) {
    const char* v = *p;
    if (std::strncmp(v, "SPECSV_", 7) != 0) continue;
    v += 7;
    const char* eq = std::strchr(v, '=');
    if (eq == nullptr) continue;
    const std::string name(v, eq - v);
    const char* val = eq + 1;
    const bool one = val[0] == '1';
    if (name == "ROUTE_LEGACY") e.route_legacy = one;
    else if (name == "ROUTE3_FORCE_EXACT") e.force_exact = one;
    else if (name == "ATTEND_FORCE_ROBUST") e.force_robust = true;
    else if (name == "NO_PDL") e.no_pdl = one;
    else if (name == "ATTEND_COOP") e.attend_coop = one;
    else if (name == "ROUTE3_DEBUG") e.route3_debug = std::atoi(val);
    else if (name == "ATTEND_DEBUG") e.attend_debug = std::atoi(val);
    else if (name == "ATTEND_SPLITS") e.attend_splits = std::atoi(val);
    else if (name == "ATTEND_SPLITS_REFRESH") e.attend_splits_refresh = std::atoi(val);
  }
  g_env = e;
}

std::string& last_error() {
  thread_local std::string msg;
  return msg;
}

void validate_config(const specsv_nsa_config& c) {
  auto fail = [](const std::string& m) { throw Error(SPECSV_EINVAL, "NsaConfig: " + m); };
  if (c.l <= 0) fail("l must be positive");
  if (c.d <= 0 || c.d > c.l) fail("d must satisfy 0 < d <= l");
  if (c.l_sel <= 0 || c.l_sel % c.d != 0) fail("l_sel must be a positive multiple of d");
  if (c.n < 3) fail("n must be at least 3 (initial + local blocks)");
  if (c.w <= 0) fail("w must be positive");
  if (c.n_q_heads <= 0 || c.n_kv_heads <= 0 || c.n_q_heads % c.n_kv_heads != 0)
    fail("n_q_heads must be a positive multiple of n_kv_heads");
  if (c.d_head <= 0) fail("d_head must be positive");
  if (c.n_layers <= 0) fail("n_layers must be positive");
  if (c.routing_lag < 0) fail("routing_lag must be nonnegative");
  if (c.w < c.routing_lag) fail("w must cover the routing lag");
}

void check_build_limits(const specsv_nsa_config& c) {
  auto unsup = [](const std::string& m) { throw Error(SPECSV_EUNSUPPORTED, m); };
  if (c.d_head != 128) unsup("this sm_100a build supports d_head == 128");
  if (c.l_sel != 64) unsup("this sm_100a build supports l_sel == 64 (two blocks per 128-key tile)");
  const int64_t g = c.n_q_heads / c.n_kv_heads;
  if (g > 32 || (g & (g - 1)) != 0) unsup("GQA group size must be a power of two <= 32");
  if (c.n > 64) unsup("n must be <= 64");
  if (c.n_q_heads > 128) unsup("n_q_heads must be <= 128");
  if (c.w / c.l_sel + 2 + c.n > 1280) unsup("w / l_sel + n must be <= 1278 (per-chunk block union)");
  if ((c.l - 1) / c.d > 7) unsup("l must be <= 8 * d (routing halo)");
  if ((kRouteTile * c.d) % c.l_sel != 0)
    unsup("d must be a multiple of 4 (16-block routing tiles start on selection-block boundaries)");
  if (((kRouteTile - 1) * c.d + c.l - 1) / c.l_sel + 2 > 8)
    unsup("15 d + l must be <= 448 (selection blocks one 16-block routing tile touches)");
}

int64_t routing_visible_len(const specsv_nsa_config& c, int64_t pos) {
  const int64_t v = pos + 1 - c.routing_lag;
  return v > 0 ? v : 0;
}

int64_t visible_blocks(const specsv_nsa_config& c, int64_t blocks, int64_t visible_len) {
  if (visible_len < c.l) return 0;
  const int64_t by_len = (visible_len - c.l) / c.d + 1;
  return std::min(by_len, blocks);
}

int64_t selection_block_count(const specsv_nsa_config& c, int64_t visible_len) {
  return visible_len > 0 ? (visible_len + c.l_sel - 1) / c.l_sel : 0;
}

int64_t representative(const int64_t* pos, int64_t n) {
  if (n <= 0) throw Error(SPECSV_EINVAL, "representative_index: empty group");
  int64_t rep = 0;
  for (int64_t i = 1; i < n; ++i)
    if (pos[i] >= pos[rep]) rep = i;
  return rep;
}

std::vector<int32_t> source_rows(const specsv_nsa_config& c, int32_t nq, const int64_t* pos,
                                 int32_t group_size, int32_t mode) {
  (void)c;
  std::vector<int32_t> src(nq);
  for (int32_t q = 0; q < nq; ++q) src[q] = q;
  if (mode == SPECSV_MODE_APPROX) {
    const int32_t gamma = nq - 1;
    for (int32_t b = 0; b < gamma; b += group_size) {
      const int32_t e = std::min(b + group_size, gamma);
      const int32_t rep = 1 + b + static_cast<int32_t>(representative(pos + 1 + b, e - b));
      for (int32_t q = 1 + b; q < 1 + e; ++q) src[q] = rep;
    }
  }
  return src;
}

std::vector<int32_t> routed_queries(int32_t nq, const int64_t* pos, int32_t group_size,
                                    int32_t mode) {
  std::vector<int32_t> r{0};
  if (mode == SPECSV_MODE_EXACT) {
    for (int32_t q = 1; q < nq; ++q) r.push_back(q);
  } else {
    const int32_t gamma = nq - 1;
    for (int32_t b = 0; b < gamma; b += group_size) {
      const int32_t e = std::min(b + group_size, gamma);
      r.push_back(1 + b + static_cast<int32_t>(representative(pos + 1 + b, e - b)));
    }
  }
  return r;
}

void resolve_layer_roles(const int64_t* reuse, int64_t n_reuse, int64_t n_layers, int32_t* roles,
                         int64_t* source) {
  if (n_layers < 1) throw Error(SPECSV_EINVAL, "resolve_layer_roles: need at least one layer");
  std::vector<int64_t> s(reuse, reuse + n_reuse);
  std::sort(s.begin(), s.end());
  s.erase(std::unique(s.begin(), s.end()), s.end());
  for (int64_t id : s) {
    if (id == 0) throw Error(SPECSV_EINVAL, "resolve_layer_roles: layer 0 must refresh");
    if (id < 0 || id >= n_layers) throw Error(SPECSV_EINVAL, "resolve_layer_roles: layer id out of range");
  }
  for (int64_t j = 0; j < n_layers; ++j) roles[j] = SPECSV_ROLE_REFRESH;
  for (int64_t id : s) roles[id] = SPECSV_ROLE_REUSE;
  int64_t last = 0;
  for (int64_t j = 0; j < n_layers; ++j) {
    if (roles[j] == SPECSV_ROLE_REFRESH) last = j;
    source[j] = roles[j] == SPECSV_ROLE_REFRESH ? j : last;
  }
}

int32_t clamp_inherited(const specsv_nsa_config& c, const int32_t* src, uint32_t src_forced,
                        int32_t count, int64_t bound, int32_t* out, uint32_t* out_forced) {
  int32_t n = 0;
  uint32_t f = 0;
  for (int32_t i = 0; i < count; ++i) {
    if (static_cast<int64_t>(src[i]) * c.l_sel >= bound) continue;
    if ((src_forced >> i) & 1u) f |= 1u << n;
    out[n++] = src[i];
  }
  if (out_forced) *out_forced = f;
  return n;
}

static int64_t overlap(const int32_t* a, int32_t na, const int32_t* b, int32_t nb) {
  int64_t s = 0;
  int32_t i = 0, j = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (a[i] > b[j]) ++j;
    else { ++s; ++i; ++j; }
  }
  return s;
}

void load_stats(const specsv_nsa_config& c, int64_t rows, int32_t nq, const int64_t* pos,
                const uint64_t* tree_mask, int32_t mask_words, int32_t C, int32_t mode,
                int32_t role, const int32_t* idx, const int32_t* cnt, specsv_load_stats_t* st) {
  std::memset(st, 0, sizeof(*st));
  if (C < 1) throw Error(SPECSV_EINVAL, "partition_groups: C must be >= 1");
  const int32_t gamma = nq - 1, n = static_cast<int32_t>(c.n);
  auto win_rows = [&](int32_t q) {
    const int64_t lo = std::max<int64_t>(0, pos[q] - c.w + 1);
    const int64_t hi = std::min<int64_t>(pos[q], rows - 1);
    int64_t r = hi >= lo ? hi - lo + 1 : 0;
    for (int32_t j = 0; j < gamma; ++j)
      if ((tree_mask[static_cast<int64_t>(q - 1) * mask_words + j / 64] >> (j % 64)) & 1ull) ++r;
    return r;
  };
  for (int32_t b = 0; b < gamma; b += C) {
    const int32_t e = std::min(b + C, gamma), size = e - b, q0 = 1 + b;
    if (mode == SPECSV_MODE_EXACT) {
      std::vector<int32_t> all;
      for (int32_t i = 0; i < size; ++i) {
        const int32_t q = q0 + i;
        if (cnt[q] < 0) throw Error(SPECSV_ESTATE, "group_attend_exact: member without index set");
        all.insert(all.end(), idx + static_cast<int64_t>(q) * n, idx + static_cast<int64_t>(q) * n + cnt[q]);
        st->total_requested_loads += cnt[q];
        st->window_token_loads += win_rows(q);
        if (i > 0 && st->n_pairs < SPECSV_MAX_PAIRS)
          st->pairwise_overlap[st->n_pairs++] =
              overlap(idx + static_cast<int64_t>(q - 1) * n, cnt[q - 1], idx + static_cast<int64_t>(q) * n, cnt[q]);
      }
      std::sort(all.begin(), all.end());
      all.erase(std::unique(all.begin(), all.end()), all.end());
      st->unique_block_loads += static_cast<int64_t>(all.size());
      st->index_constructions += role == SPECSV_ROLE_REUSE ? 0 : size;
    } else {
      const int32_t rep = q0 + static_cast<int32_t>(representative(pos + q0, size));
      if (cnt[rep] < 0) throw Error(SPECSV_ESTATE, "group_attend_approx: representative without index set");
      for (int32_t i = 0; i < size; ++i) st->window_token_loads += win_rows(q0 + i);
      st->unique_block_loads += cnt[rep];
      st->total_requested_loads += static_cast<int64_t>(cnt[rep]) * size;
      st->index_constructions += role == SPECSV_ROLE_REUSE ? 0 : 1;
    }
  }
  st->dedup_savings = st->total_requested_loads - st->unique_block_loads;
}

int64_t algorithmic_bytes(const specsv_nsa_config& c, int64_t rows, int32_t nq, const int64_t* pos,
                          int32_t role, const int32_t* idx, const int32_t* cnt, int32_t mode,
                          int32_t C) {
  const int64_t H = c.n_kv_heads, dh = c.d_head, Hq = c.n_q_heads;
  const int64_t blocks = rows >= c.l ? (rows - c.l) / c.d + 1 : 0;
  const std::vector<int32_t> src = source_rows(c, nq, pos, C, mode);
  int64_t mmax = 0;
  for (int32_t q = 0; q < nq; ++q)
    mmax = std::max(mmax, visible_blocks(c, blocks, routing_visible_len(c, pos[q])));
  // compressed branch: bf16 K copy + bf16 V of the widest visible range
  int64_t bytes = mmax * H * dh * (2 + 2);
  // routing reads the fp32 keys of the routed queries' visible range
  if (role == SPECSV_ROLE_REFRESH) bytes += mmax * H * dh * 4;
  // union over all queries of selected tokens and window tokens, bf16 K+V, all heads
  std::vector<std::pair<int64_t, int64_t>> iv;
  for (int32_t q = 0; q < nq; ++q) {
    const int64_t bound = std::min(routing_visible_len(c, pos[q]), rows);
    const int32_t s = src[q];
    for (int32_t k = 0; k < (cnt[s] > 0 ? cnt[s] : 0); ++k) {
      const int64_t lo = static_cast<int64_t>(idx[static_cast<int64_t>(s) * c.n + k]) * c.l_sel;
      const int64_t hi = std::min(lo + c.l_sel, bound);
      if (hi > lo) iv.emplace_back(lo, hi);
    }
    const int64_t wlo = std::max<int64_t>(0, pos[q] - c.w + 1), whi = std::min<int64_t>(pos[q], rows - 1);
    if (whi >= wlo) iv.emplace_back(wlo, whi + 1);
  }
  std::sort(iv.begin(), iv.end());
  int64_t tokens = 0, cur_lo = -1, cur_hi = -1;
  for (auto& [lo, hi] : iv) {
    if (lo > cur_hi) {
      tokens += cur_hi - cur_lo;
      cur_lo = lo;
      cur_hi = hi;
    } else {
      cur_hi = std::max(cur_hi, hi);
    }
  }
  tokens += cur_hi - cur_lo;
  bytes += tokens * H * dh * 2 * 2;
  bytes += static_cast<int64_t>(nq - 1) * H * dh * 2 * 2;      // draft rows
  bytes += static_cast<int64_t>(nq) * Hq * dh * 4 * 2;         // q in, out
  bytes += static_cast<int64_t>(nq) * Hq * 3 * 4;              // gates
  return bytes;
}

}  // namespace specsv_b200
