/*
 * planner.h -- C-ABI of the host-side planner policy: the strategy tuple and
 * precision classes, the offline profile table with O(1) preselection, the
 * online EMA guard ("refiner") and the linear step-latency cost model fitted
 * to measured step times.  Pure host C++ (no device code), in the same
 * library as nsa_verify.h.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   specsv_plan_bucket_of / _satisfies / _validate_strategy / _parse_strategy
 *       plan::bucket_of, satisfies, validate_strategy, parse_strategy
 *       (include/specsv/plan/strategy.hpp:20-48, plan/profile.hpp:20-24)
 *   specsv_plan_profile_offline / _preselect
 *       plan::profile_offline, preselect (plan/profile.hpp:58-76,
 *       src/profile.cpp:58-99); the evaluator is a C callback
 *   specsv_plan_refine_step
 *       plan::refine_step (plan/refiner.hpp:16-62, src/refiner.cpp:26-90)
 *   specsv_cost_account_step / _estimate_latency / _index_share / _fit
 *       cost::account_step, estimate_latency, index_share, fit_cost_coeffs
 *       (include/specsv/cost/cost_model.hpp:14-57, src/cost_model.cpp)
 *
 * Errors follow nsa_verify.h: specsv_status plus specsv_last_error().
 */
#ifndef SPECSV_B200_PLANNER_H
#define SPECSV_B200_PLANNER_H

#include "specsv_b200/nsa_verify.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SPECSV_PLAN_BUCKETS 4          /* kNumBuckets (profile.hpp:15) */
#define SPECSV_PLAN_BUCKET_WIDTH 4096  /* kBucketWidth (profile.hpp:16) */
#define SPECSV_PLAN_CLASSES 4          /* kNumClasses (strategy.hpp:20) */
#define SPECSV_PLAN_PER_ENTRY 12       /* kCandidatesPerEntry (profile.hpp:17) */
#define SPECSV_PLAN_MAX_REUSE 64       /* reuse-set layers carried by a tuple */
#define SPECSV_PLAN_MAX_RANKS 64       /* ranks the refiner can explore */

/* PrecisionClass (strategy.hpp:17) */
enum { SPECSV_CLASS_STRICT = 0, SPECSV_CLASS_REUSE_ONLY = 1, SPECSV_CLASS_APPROX_ONLY = 2,
       SPECSV_CLASS_APPROX_REUSE = 3 };
/* tree::Traversal (draft_tree.hpp:35) */
enum { SPECSV_TRAVERSAL_BFS = 0, SPECSV_TRAVERSAL_DFS = 1 };

/* StrategyTuple (strategy.hpp:26-38): theta_d = (D, k, T), theta_s = (C, M, S) */
typedef struct specsv_strategy {
  int64_t depth;
  int64_t width;
  int32_t traversal;   /* SPECSV_TRAVERSAL_* */
  int32_t mode;        /* SPECSV_MODE_* */
  int64_t group_size;
  int64_t budget;      /* node budget; < 0 = none (std::optional) */
  int32_t n_reuse;
  int32_t reserved;
  int64_t reuse_set[SPECSV_PLAN_MAX_REUSE];
} specsv_strategy;

/* ProfiledCandidate (profile.hpp:26-31) */
typedef struct specsv_profiled_candidate {
  specsv_strategy strategy;
  double exp_accepted; /* E[A] */
  double exp_latency;  /* E[T] */
  double throughput;   /* E[A] / E[T] */
} specsv_profiled_candidate;

/* context bucket [0,4K) [4K,8K) [8K,12K) [12K,inf); -1 for a negative length */
int32_t specsv_plan_bucket_of(int64_t context_len);
int32_t specsv_plan_satisfies(const specsv_strategy* s, int32_t cls);
specsv_status specsv_plan_validate_strategy(const specsv_strategy* s, int32_t cls);
/* "D,k,T,C,M" (e.g. "4,2,BFS,2,exact"); reuse set empty, no budget */
specsv_status specsv_plan_parse_strategy(const char* text, specsv_strategy* out);
/* StrategyTuple::to_string into buf (NUL-terminated, truncated to cap) */
specsv_status specsv_plan_strategy_to_string(const specsv_strategy* s, char* buf, size_t cap);

/* ---- offline profile (opaque table) ------------------------------------- */
typedef struct specsv_profile_table specsv_profile_table;
/* Evaluator (EvaluateFn, profile.hpp:47-50): run the strategy on the bucket's
 * calibration prompts and write per-step accepted counts / latencies; return
 * the number of steps written (<= capacity), or < 0 on failure. */
typedef int32_t (*specsv_eval_fn)(const specsv_strategy* s, int32_t bucket, int32_t cls,
                                  double* step_accepted, double* step_latency, int32_t capacity,
                                  void* user);
specsv_profile_table* specsv_plan_profile_create(void);
void specsv_plan_profile_destroy(specsv_profile_table* t);
/* profile_offline: every class-valid candidate on every bucket, the best
 * SPECSV_PLAN_PER_ENTRY by throughput kept per (bucket, class) (stable order);
 * EINVAL when some class has no valid candidate or a trace is empty/ragged */
specsv_status specsv_plan_profile_offline(specsv_eval_fn eval, void* user,
                                          const specsv_strategy* candidates, int32_t n,
                                          int32_t max_steps, specsv_profile_table* out);
specsv_status specsv_plan_profile_put(specsv_profile_table* t, int32_t bucket, int32_t cls,
                                      const specsv_profiled_candidate* c, int32_t count);
/* one entry access (ProfileTable::at): copies up to capacity candidates */
specsv_status specsv_plan_profile_entry(const specsv_profile_table* t, int32_t bucket,
                                        int32_t cls, specsv_profiled_candidate* out,
                                        int32_t capacity, int32_t* count);
int64_t specsv_plan_profile_stored(const specsv_profile_table* t);
/* entry accesses so far (ProfileTable::entry_accesses); assign >= 0 then
 * stores assign as the new count (the reference's tests zero it directly) */
int64_t specsv_plan_profile_accesses(specsv_profile_table* t, int64_t assign);
/* preselect: rank-1 candidate of (bucket, class), exactly one entry access */
specsv_status specsv_plan_preselect(const specsv_profile_table* t, int32_t bucket, int32_t cls,
                                    specsv_profiled_candidate* out);

/* ---- online guard (refiner.hpp) ------------------------------------------ */
typedef struct specsv_guard_constants {
  double alpha;        /* EMA coefficient, 0.40 */
  double rho;          /* acceptance-drop ratio, 0.85 */
  int64_t warmup;      /* minimum observation count m, 8 */
  int64_t hysteresis;  /* consecutive sub-threshold steps h, 5 */
} specsv_guard_constants;

typedef struct specsv_refiner_state {
  specsv_guard_constants consts;
  double ema;
  int32_t ema_primed;
  int32_t settled;
  int64_t steps_seen;
  int64_t below_count;
  int64_t transitions;
  int64_t active_rank;
  int32_t n_explored;
  int32_t reserved;
  int64_t explored_rank[SPECSV_PLAN_MAX_RANKS];
  double explored_sum_accepted[SPECSV_PLAN_MAX_RANKS];
  double explored_sum_latency[SPECSV_PLAN_MAX_RANKS];
  int64_t explored_steps[SPECSV_PLAN_MAX_RANKS];
} specsv_refiner_state;

typedef struct specsv_refine_decision {
  int32_t switched;
  int32_t settled_now;
  int64_t active_rank;
} specsv_refine_decision;

#define SPECSV_PLAN_MAX_TRANSITIONS 2  /* kMaxTransitions (refiner.hpp:60) */
#define SPECSV_PLAN_EARLY_WINDOW 32    /* kDefaultEarlyWindow (refiner.hpp:61) */

/* fresh per-request state with the default constants */
void specsv_plan_refiner_init(specsv_refiner_state* st);
/* one guard update against the entry the active strategy came from
 * (exp_accepted[rank] = E[A] of the entry's candidates) */
specsv_status specsv_plan_refine_step(specsv_refiner_state* st, double accepted, double latency,
                                      const double* exp_accepted, int32_t n_candidates,
                                      specsv_refine_decision* out);
/* RefinerState::observed_throughput (0 when the rank was never run) */
double specsv_plan_observed_throughput(const specsv_refiner_state* st, int64_t rank);

/* ---- cost model (cost_model.hpp) ------------------------------------------ */
typedef struct specsv_cost_coeffs {
  double c_block;   /* per unique selected-block load, 1.0 */
  double c_index;   /* per index construction, 4.0 */
  double c_launch;  /* per modeled launch, 0.5 */
  double c_window;  /* per window token, 0.02 */
  double c_base;    /* fixed per step, 10.0 */
} specsv_cost_coeffs;

typedef struct specsv_step_accounting {
  int64_t unique_loads;
  int64_t constructions;
  int64_t launches;
  int64_t window_tokens;
  int64_t layers;
} specsv_step_accounting;

typedef struct specsv_fit_sample {
  specsv_step_accounting acc;
  double measured;
} specsv_fit_sample;

void specsv_cost_default_coeffs(specsv_cost_coeffs* c);
specsv_status specsv_cost_validate(const specsv_cost_coeffs* c);
/* per-layer (group-summed) LoadStats under the layer-role plan of reuse_set;
 * reuse layers contribute no index constructions and one launch, refresh
 * layers two (layer_roles.hpp:23-24) */
specsv_status specsv_cost_account_step(const specsv_load_stats_t* per_layer, int64_t n_layers,
                                       const int64_t* reuse_set, int64_t n_reuse,
                                       specsv_step_accounting* out);
double specsv_cost_estimate_latency(const specsv_step_accounting* a, const specsv_cost_coeffs* c);
double specsv_cost_index_share(const specsv_step_accounting* a, const specsv_cost_coeffs* c);
/* nonnegative least squares (active-set clamping) of measured step times */
specsv_status specsv_cost_fit(const specsv_fit_sample* samples, int64_t n, specsv_cost_coeffs* out);

#ifdef __cplusplus
}
#endif
#endif
