// policy.h -- host-side C++ rules shared by the C-ABI and the launchers.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "specsv_b200/nsa_verify.h"

namespace specsv_b200 {

struct Error : std::runtime_error {
  specsv_status code;
  Error(specsv_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// thread-local message behind specsv_last_error()
std::string& last_error();

// Diagnostic / test switches (SPECSV_* environment variables), read in one
// pass over the environment at the start of every C-ABI call (getenv per use
// cost ~1 us each on the per-call host path).  Thread-local.
struct DebugEnv {
  bool route_legacy = false;    // SPECSV_ROUTE_LEGACY=1: fp64-DMMA routing kernel
  bool force_exact = false;     // SPECSV_ROUTE3_FORCE_EXACT=1: every query through the exact path
  bool force_robust = false;    // SPECSV_ATTEND_FORCE_ROBUST: the attend robust redo pass
  bool no_pdl = false;          // SPECSV_NO_PDL=1: no programmatic dependent launch
  bool attend_coop = false;     // SPECSV_ATTEND_COOP=1: cooperative attend launches under PDL
  int route3_debug = 0;         // SPECSV_ROUTE3_DEBUG
  int attend_debug = 0;         // SPECSV_ATTEND_DEBUG
  int attend_splits = 0;        // SPECSV_ATTEND_SPLITS=k: at most k split CTAs per head (timing)
  int attend_splits_refresh = 0;  // SPECSV_ATTEND_SPLITS_REFRESH=k: the same, refresh layers only
};
const DebugEnv& debug_env();
void refresh_debug_env();

// runs a C-ABI body: exceptions become a status code plus the thread-local message
template <class F>
specsv_status guarded(F&& f) {
  try {
    refresh_debug_env();
    f();
    last_error().clear();
    return SPECSV_OK;
  } catch (const Error& e) {
    last_error() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return SPECSV_EINVAL;
  }
}

void validate_config(const specsv_nsa_config& c);
void check_build_limits(const specsv_nsa_config& c);
int64_t routing_visible_len(const specsv_nsa_config& c, int64_t pos);
int64_t visible_blocks(const specsv_nsa_config& c, int64_t blocks, int64_t visible_len);
int64_t selection_block_count(const specsv_nsa_config& c, int64_t visible_len);
int64_t representative(const int64_t* pos, int64_t n);
std::vector<int32_t> source_rows(const specsv_nsa_config& c, int32_t nq, const int64_t* pos,
                                 int32_t group_size, int32_t mode);
std::vector<int32_t> routed_queries(int32_t nq, const int64_t* pos, int32_t group_size,
                                    int32_t mode);
void resolve_layer_roles(const int64_t* reuse, int64_t n_reuse, int64_t n_layers, int32_t* roles,
                         int64_t* source);
int32_t clamp_inherited(const specsv_nsa_config& c, const int32_t* src, uint32_t src_forced,
                        int32_t count, int64_t bound, int32_t* out, uint32_t* out_forced);
void load_stats(const specsv_nsa_config& c, int64_t rows, int32_t nq, const int64_t* pos,
                const uint64_t* tree_mask, int32_t mask_words, int32_t C, int32_t mode,
                int32_t role, const int32_t* idx, const int32_t* cnt, specsv_load_stats_t* st);
int64_t algorithmic_bytes(const specsv_nsa_config& c, int64_t rows, int32_t nq, const int64_t* pos,
                          int32_t role, const int32_t* idx, const int32_t* cnt, int32_t mode,
                          int32_t C);

}  // namespace specsv_b200
