// planner.cpp -- host-side planner policy behind include/specsv_b200/planner.h:
// strategy tuples and precision classes, the offline profile table with O(1)
// preselection, the online EMA guard and the linear step-latency cost model.
//
// Same rules as the reference (paths relative to /root/reference/proj):
//   strategy   src/strategy.cpp:9-92, include/specsv/plan/strategy.hpp:14-45
//   profile    src/profile.cpp:12-99 (bucket_of, ProfileTable::at/put,
//              summarize, profile_offline, preselect)
//   refiner    src/refiner.cpp:9-90
//   cost model src/cost_model.cpp:9-131
// The reference's JSON profile I/O (profile.cpp:101-187) is host file
// plumbing outside the verify path and is not part of this build.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "policy.h"
#include "specsv_b200/planner.h"

struct specsv_profile_table {
  // grid[bucket][class]: ranked candidates (empty optional = no entry)
  std::array<std::array<std::optional<std::vector<specsv_profiled_candidate>>, SPECSV_PLAN_CLASSES>,
             SPECSV_PLAN_BUCKETS>
      grid;
  mutable int64_t entry_accesses = 0;
};

namespace specsv_b200 {
namespace {

const char* mode_str(int32_t m) { return m == SPECSV_MODE_EXACT ? "exact" : "approx"; }
const char* class_str(int32_t c) {
  switch (c) {
    case SPECSV_CLASS_STRICT: return "strict";
    case SPECSV_CLASS_REUSE_ONLY: return "reuse-only";
    case SPECSV_CLASS_APPROX_ONLY: return "approx-only";
    case SPECSV_CLASS_APPROX_REUSE: return "approx-reuse";
  }
  return "?";
}

void check_class(int32_t cls) {
  if (cls < 0 || cls >= SPECSV_PLAN_CLASSES) throw Error(SPECSV_EINVAL, "precision class out of range");
}
void check_bucket(int32_t b) {
  if (b < 0 || b >= SPECSV_PLAN_BUCKETS) throw Error(SPECSV_EINVAL, "ProfileTable: bucket out of range");
}

// StrategyTuple::to_string (strategy.cpp:37-50): "D,k,T,C,M" (+ "/S=a+b")
std::string to_string(const specsv_strategy& s) {
  std::ostringstream os;
  os << s.depth << ',' << s.width << ',' << (s.traversal == SPECSV_TRAVERSAL_BFS ? "BFS" : "DFS")
     << ',' << s.group_size << ',' << mode_str(s.mode);
  if (s.n_reuse > 0) {
    os << "/S=";
    for (int32_t i = 0; i < s.n_reuse; ++i) os << (i ? "+" : "") << s.reuse_set[i];
  }
  return os.str();
}

// satisfies (strategy.cpp:52-63)
bool satisfies(const specsv_strategy& s, int32_t cls) {
  if (s.depth < 1 || s.width < 1 || s.group_size < 1) return false;
  const bool exact = s.mode == SPECSV_MODE_EXACT;
  const bool no_reuse = s.n_reuse == 0;
  switch (cls) {
    case SPECSV_CLASS_STRICT: return exact && no_reuse;
    case SPECSV_CLASS_REUSE_ONLY: return exact && !no_reuse;
    case SPECSV_CLASS_APPROX_ONLY: return !exact && no_reuse;
    case SPECSV_CLASS_APPROX_REUSE: return !exact && !no_reuse;
  }
  return false;
}

// the table entry of (bucket, class); counts one access (ProfileTable::at, profile.cpp:18-27)
const std::vector<specsv_profiled_candidate>& entry_at(const specsv_profile_table& t, int32_t b,
                                                       int32_t cls) {
  check_bucket(b);
  check_class(cls);
  const auto& slot = t.grid[b][cls];
  if (!slot.has_value())
    throw Error(SPECSV_EINVAL, "ProfileTable: no entry for bucket " + std::to_string(b) +
                                   ", class " + class_str(cls));
  ++t.entry_accesses;
  return *slot;
}

// summarize (profile.cpp:43-56): E[A], E[T] over the trace's steps, E[A]/E[T]
specsv_profiled_candidate summarize(const specsv_strategy& s, const double* acc, const double* lat,
                                    int32_t steps) {
  if (steps <= 0) throw Error(SPECSV_EINVAL, "profile_offline: empty or ragged evaluation trace");
  double sa = 0.0, st = 0.0;
  for (int32_t i = 0; i < steps; ++i) sa += acc[i];
  for (int32_t i = 0; i < steps; ++i) st += lat[i];
  specsv_profiled_candidate c;
  c.strategy = s;
  c.exp_accepted = sa / static_cast<double>(steps);
  c.exp_latency = st / static_cast<double>(steps);
  if (c.exp_latency <= 0.0) throw Error(SPECSV_EINVAL, "profile_offline: nonpositive latency");
  c.throughput = c.exp_accepted / c.exp_latency;
  return c;
}

constexpr int kDim = 5;  // base, launch, block, index, window (cost_model.cpp:39)

std::array<double, kDim> regressors(const specsv_step_accounting& a) {
  return {1.0, static_cast<double>(a.launches), static_cast<double>(a.unique_loads),
          static_cast<double>(a.constructions), static_cast<double>(a.window_tokens)};
}

// Gauss-Jordan with partial pivoting over the free coordinates
// (cost_model.cpp:46-74); false when singular
bool solve(const std::array<std::array<double, kDim>, kDim>& a, const std::array<double, kDim>& b,
           const std::array<bool, kDim>& free_coord, std::array<double, kDim>& x) {
  std::vector<int> idx;
  for (int i = 0; i < kDim; ++i)
    if (free_coord[i]) idx.push_back(i);
  const int n = static_cast<int>(idx.size());
  std::vector<std::vector<double>> m(n, std::vector<double>(n + 1, 0.0));
  for (int r = 0; r < n; ++r) {
    for (int c = 0; c < n; ++c) m[r][c] = a[idx[r]][idx[c]];
    m[r][n] = b[idx[r]];
  }
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::fabs(m[r][col]) > std::fabs(m[piv][col])) piv = r;
    if (std::fabs(m[piv][col]) < 1e-12) return false;
    std::swap(m[piv], m[col]);
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = m[r][col] / m[col][col];
      for (int c = col; c <= n; ++c) m[r][c] -= f * m[col][c];
    }
  }
  x.fill(0.0);
  for (int r = 0; r < n; ++r) x[idx[r]] = m[r][n] / m[r][r];
  return true;
}

}  // namespace
}  // namespace specsv_b200

using namespace specsv_b200;

extern "C" {

int32_t specsv_plan_bucket_of(int64_t context_len) {
  if (context_len < 0) {
    last_error() = "bucket_of: negative context length";
    return -1;
  }
  const int64_t b = context_len / SPECSV_PLAN_BUCKET_WIDTH;
  return b >= SPECSV_PLAN_BUCKETS ? SPECSV_PLAN_BUCKETS - 1 : static_cast<int32_t>(b);
}

int32_t specsv_plan_satisfies(const specsv_strategy* s, int32_t cls) {
  return s != nullptr && cls >= 0 && cls < SPECSV_PLAN_CLASSES && satisfies(*s, cls) ? 1 : 0;
}

specsv_status specsv_plan_validate_strategy(const specsv_strategy* s, int32_t cls) {
  return guarded([&] {
    if (s == nullptr) throw Error(SPECSV_EINVAL, "null strategy");
    check_class(cls);
    if (!satisfies(*s, cls))
      throw Error(SPECSV_EINVAL,
                  "strategy " + to_string(*s) + " violates precision class " + class_str(cls));
  });
}

specsv_status specsv_plan_parse_strategy(const char* text, specsv_strategy* out) {
  return guarded([&] {  // parse_strategy (strategy.cpp:72-92)
    if (text == nullptr || out == nullptr) throw Error(SPECSV_EINVAL, "null argument");
    std::vector<std::string> parts;
    std::stringstream ss(text);
    std::string item;
    while (std::getline(ss, item, ',')) parts.push_back(item);
    if (parts.size() != 5)
      throw Error(SPECSV_EINVAL, std::string("strategy must be D,k,T,C,M (got '") + text + "')");
    specsv_strategy s;
    std::memset(&s, 0, sizeof(s));
    s.budget = -1;
    s.depth = std::stoll(parts[0]);
    s.width = std::stoll(parts[1]);
    if (parts[2] == "BFS" || parts[2] == "bfs") s.traversal = SPECSV_TRAVERSAL_BFS;
    else if (parts[2] == "DFS" || parts[2] == "dfs") s.traversal = SPECSV_TRAVERSAL_DFS;
    else throw Error(SPECSV_EINVAL, "bad traversal '" + parts[2] + "'");
    s.group_size = std::stoll(parts[3]);
    if (parts[4] == "exact") s.mode = SPECSV_MODE_EXACT;
    else if (parts[4] == "approx" || parts[4] == "approximate") s.mode = SPECSV_MODE_APPROX;
    else throw Error(SPECSV_EINVAL, "bad coarsening mode '" + parts[4] + "'");
    if (s.depth < 1 || s.width < 1 || s.group_size < 1)
      throw Error(SPECSV_EINVAL, "strategy fields must be >= 1");
    *out = s;
  });
}

specsv_status specsv_plan_strategy_to_string(const specsv_strategy* s, char* buf, size_t cap) {
  return guarded([&] {
    if (s == nullptr || buf == nullptr || cap == 0) throw Error(SPECSV_EINVAL, "null argument");
    const std::string t = to_string(*s);
    const size_t n = std::min(cap - 1, t.size());
    std::memcpy(buf, t.data(), n);
    buf[n] = '\0';
  });
}

specsv_profile_table* specsv_plan_profile_create(void) { return new specsv_profile_table(); }
void specsv_plan_profile_destroy(specsv_profile_table* t) { delete t; }

specsv_status specsv_plan_profile_offline(specsv_eval_fn eval, void* user,
                                          const specsv_strategy* candidates, int32_t n,
                                          int32_t max_steps, specsv_profile_table* out) {
  return guarded([&] {  // profile_offline (profile.cpp:60-96)
    if (eval == nullptr || out == nullptr || (n > 0 && candidates == nullptr) || max_steps < 1)
      throw Error(SPECSV_EINVAL, "null argument");
    specsv_profile_table table;
    std::vector<double> acc(max_steps), lat(max_steps);
    for (int32_t b = 0; b < SPECSV_PLAN_BUCKETS; ++b) {
      for (int32_t c = 0; c < SPECSV_PLAN_CLASSES; ++c) {
        std::vector<specsv_profiled_candidate> entry;
        for (int32_t i = 0; i < n; ++i) {
          if (!satisfies(candidates[i], c)) continue;
          const int32_t steps = eval(&candidates[i], b, c, acc.data(), lat.data(), max_steps, user);
          if (steps > max_steps) throw Error(SPECSV_EINVAL, "profile_offline: trace overflow");
          entry.push_back(summarize(candidates[i], acc.data(), lat.data(), steps));
        }
        if (entry.empty())
          throw Error(SPECSV_EINVAL,
                      std::string("profile_offline: no valid candidate for class ") + class_str(c));
        std::stable_sort(entry.begin(), entry.end(),
                         [](const specsv_profiled_candidate& x, const specsv_profiled_candidate& y) {
                           return x.throughput > y.throughput;
                         });
        if (entry.size() > SPECSV_PLAN_PER_ENTRY) entry.resize(SPECSV_PLAN_PER_ENTRY);
        table.grid[b][c] = std::move(entry);
      }
    }
    out->grid = std::move(table.grid);
    out->entry_accesses = 0;
  });
}

specsv_status specsv_plan_profile_put(specsv_profile_table* t, int32_t bucket, int32_t cls,
                                      const specsv_profiled_candidate* c, int32_t count) {
  return guarded([&] {
    if (t == nullptr || (count > 0 && c == nullptr) || count < 0) throw Error(SPECSV_EINVAL, "null argument");
    check_bucket(bucket);
    check_class(cls);
    t->grid[bucket][cls] = std::vector<specsv_profiled_candidate>(c, c + count);
  });
}

specsv_status specsv_plan_profile_entry(const specsv_profile_table* t, int32_t bucket,
                                        int32_t cls, specsv_profiled_candidate* out,
                                        int32_t capacity, int32_t* count) {
  return guarded([&] {
    if (t == nullptr || count == nullptr) throw Error(SPECSV_EINVAL, "null argument");
    const auto& e = entry_at(*t, bucket, cls);
    const int32_t k = std::min<int32_t>(capacity, static_cast<int32_t>(e.size()));
    for (int32_t i = 0; i < k; ++i) out[i] = e[i];
    *count = static_cast<int32_t>(e.size());
  });
}

int64_t specsv_plan_profile_stored(const specsv_profile_table* t) {
  if (t == nullptr) return 0;
  int64_t n = 0;
  for (const auto& row : t->grid)
    for (const auto& slot : row)
      if (slot) n += static_cast<int64_t>(slot->size());
  return n;
}

int64_t specsv_plan_profile_accesses(specsv_profile_table* t, int64_t assign) {
  if (t == nullptr) return 0;
  const int64_t n = t->entry_accesses;
  if (assign >= 0) t->entry_accesses = assign;
  return n;
}

specsv_status specsv_plan_preselect(const specsv_profile_table* t, int32_t bucket, int32_t cls,
                                    specsv_profiled_candidate* out) {
  return guarded([&] {  // preselect (profile.cpp:98-101)
    if (t == nullptr || out == nullptr) throw Error(SPECSV_EINVAL, "null argument");
    const auto& e = entry_at(*t, bucket, cls);
    *out = e.front();
  });
}

void specsv_plan_refiner_init(specsv_refiner_state* st) {
  if (st == nullptr) return;
  std::memset(st, 0, sizeof(*st));
  st->consts.alpha = 0.40;
  st->consts.rho = 0.85;
  st->consts.warmup = 8;
  st->consts.hysteresis = 5;
}

double specsv_plan_observed_throughput(const specsv_refiner_state* st, int64_t rank) {
  if (st == nullptr) return 0.0;
  for (int32_t i = 0; i < st->n_explored; ++i)
    if (st->explored_rank[i] == rank && st->explored_steps[i] > 0 && st->explored_sum_latency[i] > 0.0)
      return st->explored_sum_accepted[i] / st->explored_sum_latency[i];
  return 0.0;
}

specsv_status specsv_plan_refine_step(specsv_refiner_state* st, double accepted, double latency,
                                      const double* exp_accepted, int32_t n_candidates,
                                      specsv_refine_decision* out) {
  return guarded([&] {  // refine_step (refiner.cpp:26-90)
    if (st == nullptr || out == nullptr) throw Error(SPECSV_EINVAL, "null argument");
    if (n_candidates <= 0 || exp_accepted == nullptr)
      throw Error(SPECSV_EINVAL, "refine_step: empty profile entry");
    out->switched = 0;
    out->settled_now = 0;
    out->active_rank = st->active_rank;
    st->steps_seen += 1;
    int32_t slot = -1;  // explored slot of the active rank
    for (int32_t i = 0; i < st->n_explored; ++i)
      if (st->explored_rank[i] == st->active_rank) slot = i;
    if (slot < 0) {
      if (st->n_explored >= SPECSV_PLAN_MAX_RANKS)
        throw Error(SPECSV_EUNSUPPORTED, "refine_step: explored-rank capacity exceeded");
      slot = st->n_explored++;
      st->explored_rank[slot] = st->active_rank;
      st->explored_sum_accepted[slot] = 0.0;
      st->explored_sum_latency[slot] = 0.0;
      st->explored_steps[slot] = 0;
    }
    st->explored_sum_accepted[slot] += accepted;
    st->explored_sum_latency[slot] += latency;
    st->explored_steps[slot] += 1;
    if (st->settled) return;
    if (!st->ema_primed) {
      st->ema = accepted;
      st->ema_primed = 1;
    } else {
      st->ema = st->consts.alpha * accepted + (1.0 - st->consts.alpha) * st->ema;
    }
    if (st->steps_seen <= st->consts.warmup) return;
    if (st->active_rank >= n_candidates) throw Error(SPECSV_EINVAL, "refine_step: rank outside the entry");
    const double expected = exp_accepted[st->active_rank];
    if (st->ema < st->consts.rho * expected) st->below_count += 1;
    else st->below_count = 0;
    if (st->below_count < st->consts.hysteresis) return;
    // sustained mismatch: the next rank while transitions remain
    const int64_t next_rank = st->active_rank + 1;
    if (st->transitions < SPECSV_PLAN_MAX_TRANSITIONS && next_rank < n_candidates) {
      st->active_rank = next_rank;
      st->transitions += 1;
      st->ema_primed = 0;
      st->below_count = 0;
      out->switched = 1;
      out->active_rank = st->active_rank;
      return;
    }
    // out of transitions (or candidates): settle on the best explored
    int64_t best_rank = st->active_rank;
    double best_thr = -1.0;
    for (int32_t i = 0; i < st->n_explored; ++i) {
      if (st->explored_steps[i] == 0 || st->explored_sum_latency[i] <= 0.0) continue;
      const double thr = st->explored_sum_accepted[i] / st->explored_sum_latency[i];
      if (thr > best_thr || (thr == best_thr && st->explored_rank[i] < best_rank)) {
        best_thr = thr;
        best_rank = st->explored_rank[i];
      }
    }
    st->settled = 1;
    st->below_count = 0;
    out->settled_now = 1;
    out->switched = best_rank != st->active_rank;
    st->active_rank = best_rank;
    out->active_rank = best_rank;
  });
}

void specsv_cost_default_coeffs(specsv_cost_coeffs* c) {
  if (c == nullptr) return;
  c->c_block = 1.0;
  c->c_index = 4.0;
  c->c_launch = 0.5;
  c->c_window = 0.02;
  c->c_base = 10.0;
}

specsv_status specsv_cost_validate(const specsv_cost_coeffs* c) {
  return guarded([&] {
    if (c == nullptr) throw Error(SPECSV_EINVAL, "null argument");
    if (c->c_block < 0 || c->c_index < 0 || c->c_launch < 0 || c->c_window < 0 || c->c_base < 0)
      throw Error(SPECSV_EINVAL, "CostCoeffs: coefficients must be nonnegative");
  });
}

specsv_status specsv_cost_account_step(const specsv_load_stats_t* per_layer, int64_t n_layers,
                                       const int64_t* reuse_set, int64_t n_reuse,
                                       specsv_step_accounting* out) {
  return guarded([&] {  // account_step (cost_model.cpp:9-24)
    if (out == nullptr || (n_layers > 0 && per_layer == nullptr)) throw Error(SPECSV_EINVAL, "null argument");
    if (n_layers <= 0) throw Error(SPECSV_EINVAL, "account_step: stats must cover every layer");
    std::vector<int32_t> roles(n_layers);
    std::vector<int64_t> source(n_layers);
    resolve_layer_roles(reuse_set, n_reuse, n_layers, roles.data(), source.data());
    specsv_step_accounting a{};
    a.layers = n_layers;
    for (int64_t j = 0; j < n_layers; ++j) {
      const bool reuse = roles[j] == SPECSV_ROLE_REUSE;
      a.unique_loads += per_layer[j].unique_block_loads;
      // a reuse layer constructs no indices (engine.cpp:274; the reference's
      // tests/test_cost_model.cpp:26-35 checks this on raw per-layer stats)
      a.constructions += reuse ? 0 : per_layer[j].index_constructions;
      a.launches += reuse ? 1 : 2;  // kReuseLaunches / kRefreshLaunches (layer_roles.hpp:23-24)
      a.window_tokens += per_layer[j].window_token_loads;
    }
    *out = a;
  });
}

double specsv_cost_estimate_latency(const specsv_step_accounting* a, const specsv_cost_coeffs* c) {
  if (a == nullptr || c == nullptr) return 0.0;  // estimate_latency (cost_model.cpp:26-31)
  return c->c_base + c->c_launch * static_cast<double>(a->launches) +
         c->c_block * static_cast<double>(a->unique_loads) +
         c->c_index * static_cast<double>(a->constructions) +
         c->c_window * static_cast<double>(a->window_tokens);
}

double specsv_cost_index_share(const specsv_step_accounting* a, const specsv_cost_coeffs* c) {
  const double total = specsv_cost_estimate_latency(a, c);  // index_share (cost_model.cpp:33-37)
  if (total <= 0.0) return 0.0;
  return c->c_index * static_cast<double>(a->constructions) / total;
}

specsv_status specsv_cost_fit(const specsv_fit_sample* samples, int64_t n, specsv_cost_coeffs* out) {
  return guarded([&] {  // fit_cost_coeffs (cost_model.cpp:78-131)
    if (out == nullptr) throw Error(SPECSV_EINVAL, "null argument");
    if (n <= 0 || samples == nullptr) throw Error(SPECSV_EINVAL, "fit_cost_coeffs: no samples");
    std::array<std::array<double, kDim>, kDim> ata{};
    std::array<double, kDim> atb{};
    for (int64_t k = 0; k < n; ++k) {
      const auto r = regressors(samples[k].acc);
      for (int i = 0; i < kDim; ++i) {
        atb[i] += r[i] * samples[k].measured;
        for (int j = 0; j < kDim; ++j) ata[i][j] += r[i] * r[j];
      }
    }
    // active set: clamp the most negative coordinate to zero and refit
    std::array<bool, kDim> free_coord;
    free_coord.fill(true);
    std::array<double, kDim> x{};
    for (int pass = 0; pass < kDim + 1; ++pass) {
      if (!solve(ata, atb, free_coord, x)) break;  // degenerate design
      int worst = -1;
      double worst_val = 0.0;
      for (int i = 0; i < kDim; ++i)
        if (free_coord[i] && x[i] < worst_val) {
          worst = i;
          worst_val = x[i];
        }
      if (worst == -1) {
        out->c_base = x[0];
        out->c_launch = x[1];
        out->c_block = x[2];
        out->c_index = x[3];
        out->c_window = x[4];
        return;
      }
      free_coord[worst] = false;
      x[worst] = 0.0;
    }
    // nothing fit cleanly: the mean latency as a flat model
    double mean = 0.0;
    for (int64_t k = 0; k < n; ++k) mean += samples[k].measured;
    out->c_base = mean / static_cast<double>(n);
    out->c_launch = out->c_block = out->c_index = out->c_window = 0.0;
  });
}

}  // extern "C"
