// abi.cpp -- the C-ABI boundary (include/specsv_b200/nsa_verify.h): argument
// validation with the reference's rules, workspace layout, TMA descriptor
// encoding and the launch sequence of one verify call.
//
// One verify call == the per-layer hot section of run_target_pass
// (src/engine.cpp:175-278):  REFRESH -> routing launches (route.cu) + fused
// attend launch (attend.cu);  REUSE -> fused attend launch only, reading the
// source layer's index sets and clamping them per query in-kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <climits>

#include "attend.h"
#include "policy.h"
#include "specsv_b200/nsa_verify.h"

namespace specsv_b200 {
namespace {

thread_local unsigned long long* g_trace = nullptr;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(SPECSV_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static const EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// bf16 [rows][hkv][dh] as a 3-D map (dh, hkv, rows) with 64x1x64 SWIZZLE_128B boxes
void encode_rows_map(CUtensorMap* m, const void* base, int64_t rows, int64_t hkv, int64_t dh) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) throw Error(SPECSV_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)dh, (cuuint64_t)hkv, (cuuint64_t)std::max<int64_t>(rows, 1)};
  const cuuint64_t strides[2] = {(cuuint64_t)(dh * 2), (cuuint64_t)(hkv * dh * 2)};
  const cuuint32_t box[3] = {64, 1, 64};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(SPECSV_ECUDA, "cuTensorMapEncodeTiled failed");
}

// int8 digit planes [blocks][hkv][4][dh] as a 4-D map (dh, plane, hkv, blocks)
// with 128 x 1 x 1 x 128 SWIZZLE_128B boxes: one box is one digit plane of a
// 128-block routing tile, already in the K-major SW128 layout of the MMA's A
// operand (rows past `blocks` read as zeros)
void encode_ckd_map(CUtensorMap* m, const void* base, int64_t blocks, int64_t hkv, int64_t dh) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) throw Error(SPECSV_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[4] = {(cuuint64_t)dh, 4, (cuuint64_t)hkv, (cuuint64_t)std::max<int64_t>(blocks, 1)};
  const cuuint64_t strides[3] = {(cuuint64_t)dh, (cuuint64_t)(4 * dh), (cuuint64_t)(hkv * 4 * dh)};
  const cuuint32_t box[4] = {(cuuint32_t)dh, 1, 1, (cuuint32_t)kR3Tile};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(SPECSV_ECUDA, "cuTensorMapEncodeTiled (digit planes) failed");
}

// co-resident CTAs of the attend kernel on this device (a device constant,
// computed once per device)
int coresident_for_device() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  dev = std::min(dev, 63);
  int s = cache[dev].load();
  if (s == 0) {
    s = std::max(1, attend_max_coresident());
    cache[dev].store(s);
  }
  return s;
}

int qc_size_for(const specsv_nsa_config& c);

// split CTAs per (KV head, query chunk): all of them must be co-resident
int splits_for(const specsv_nsa_config& c, int32_t nq, int n_heads, int cap_override = 0) {
  const int nchunks = (nq + qc_size_for(c) - 1) / qc_size_for(c);
  const int groups = n_heads * nchunks;
  int cap = debug_env().attend_splits > 0 ? std::min(18, debug_env().attend_splits) : 18;
  if (cap_override > 0) cap = std::min(cap, cap_override);
  return std::max(1, std::min(cap, coresident_for_device() / groups));
}

// KV heads of a call: [begin, begin + count), count 0 = all
int head_count(const specsv_nsa_config& c, const specsv_verify_args& a) {
  return a.kv_head_count > 0 ? a.kv_head_count : (int)c.n_kv_heads;
}

// a cooperative grid larger than the device's co-resident CTAs would be
// rejected by the driver (or, without the attribute, deadlock at the split
// barrier): refuse it with a message before launching
void check_coresident(int ctas, const char* what) {
  const int cap = coresident_for_device();
  if (ctas > cap)
    throw Error(SPECSV_ECUDA, std::string(what) + ": cooperative grid of " + std::to_string(ctas) +
                                  " CTAs exceeds the " + std::to_string(cap) + " co-resident CTAs");
}

// routing counter set: [0] tiles done, [2] tail CTAs done, [4..] per-slot units
constexpr int kCntSetInts = 4 + kMaxQueries;

struct Layout {
  size_t sync_off = 0, sync_bytes = 0;  // attend barrier words: fixed position per config
  int max_chunks = 1;                   // query chunks of the widest call (kMaxQueries)
  size_t r3cnt_off = 0;                 // route3 words: [0] exit count, [4] fallbacks, then one
                                        // counter set per request of a launch (fixed position)
  size_t r3_den_off = 0, r3_spill_off = 0, r3_contrib_off = 0, r3_exact_off = 0;  // route3 regions (per request)
  size_t attend_off = 0, attend_bytes = 0;
  size_t E_off = 0, TM_off = 0, TD_off = 0, F_off = 0, sel_off = 0, cnt_off = 0;
  int64_t sel_pad = 0;
  size_t total = 0;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// route3 unit shape: slots per row chunk (whole slots, <= kR3Rows rows), the
// widest selection-block range whose compressed blocks fit one unit
// (kR3MaxBlk), and a bound on the ranges per (chunk, KV head)
int64_t route3_spc(const specsv_nsa_config& c) {
  return std::max<int64_t>(1, kR3Rows / (c.n_q_heads / c.n_kv_heads));
}
int64_t route3_spr_max(const specsv_nsa_config& c) {
  for (int64_t spr = kR3MaxSpr; spr > 1; --spr) {
    bool ok = true;
    for (int64_t b0 = 0; b0 < 64 && ok; ++b0) {  // the pattern repeats with period d / gcd
      const int64_t num = b0 * c.l_sel - c.l;
      const int64_t lo = num >= 0 ? num / c.d + 1 : 0;
      const int64_t hi = ((b0 + spr) * c.l_sel - 1) / c.d;
      ok = hi - lo + 1 <= kR3MaxBlk;
    }
    if (ok) return spr;
  }
  return 1;
}
int64_t route3_nchunks(const specsv_nsa_config& c, int32_t nr) {
  const int64_t spc = route3_spc(c);
  return (nr + spc - 1) / spc;
}
constexpr int64_t kR3SmBound = 160;  // >= SM count: the ranges a single request spreads over
int64_t route3_nranges_bound(const specsv_nsa_config& c, int64_t sel_pad) {
  const int64_t per = std::max<int64_t>(1, c.n_kv_heads);  // one row chunk (the fewest units)
  return std::max<int64_t>((sel_pad + route3_spr_max(c) - 1) / route3_spr_max(c), (kR3SmBound + per - 1) / per);
}

// queries per column chunk: 64 columns / G, and few enough that the chunk's
// union (n selected blocks per query + the window blocks) fits kMaxUnion
int qc_size_for(const specsv_nsa_config& c) {
  const int G = static_cast<int>(c.n_q_heads / c.n_kv_heads);
  const int64_t win_blocks = c.w / c.l_sel + 2;
  const int64_t by_union = (kMaxUnion - win_blocks) / std::max<int64_t>(c.n, 1);
  return (int)std::max<int64_t>(1, std::min<int64_t>(std::min(kAttendCols / G, kMaxChunkQ), by_union));
}

Layout layout_for(const specsv_nsa_config& c, int32_t nq, int64_t max_rows) {
  const int splits = 18;  // upper bound of splits_for(); a batched launch keeps R x S <= 18
  Layout L;
  const int nchunks = (nq + qc_size_for(c) - 1) / qc_size_for(c);
  L.max_chunks = (kMaxQueries + qc_size_for(c) - 1) / qc_size_for(c);
  // every self-resetting word (attend barrier sets, routing grid barrier and
  // per-slot counters) first, at offsets that depend on the config only: a
  // workspace shared by calls of different query counts or context lengths
  // must never read one call's data as another call's counter
  L.sync_off = 0;
  L.sync_bytes = (size_t)kSyncSets * L.max_chunks * c.n_kv_heads * 2 * sizeof(int32_t);
  L.cnt_off = align_up(L.sync_off + L.sync_bytes, 256);
  L.r3cnt_off = align_up(L.cnt_off + (size_t)kSyncSets * kCntSetInts * sizeof(int32_t), 256);
  L.attend_off = align_up(L.r3cnt_off + (8 + (size_t)kR3Batch * kR3CntPerReq) * sizeof(int32_t), 256);
  L.attend_bytes = attend_workspace_floats(nchunks, (int)c.n_kv_heads, splits) * sizeof(float);
  const int64_t maxblk = max_rows >= c.l ? (max_rows - c.l) / c.d + 1 : 0;
  const int64_t m_pad = align_up(std::max<int64_t>(maxblk, 1), kRouteTile);
  const int64_t ntiles = m_pad / kRouteTile;
  L.sel_pad = (int64_t)align_up((size_t)((max_rows + c.l_sel - 1) / c.l_sel + 1), 32);
  size_t off = align_up(L.attend_off + L.attend_bytes, 256);
  const int64_t gs = ((kRouteTile - 1) * c.d + c.l - 1) / c.l_sel + 1;  // = g_stride
  L.E_off = off;  // per-tile selection-block shares [nq][ntiles][Hq][gs]
  off = align_up(off + (size_t)nq * ntiles * c.n_q_heads * gs * 8, 256);
  L.TM_off = off;
  off = align_up(off + (size_t)nq * c.n_q_heads * ntiles * 8, 256);
  L.TD_off = off;
  off = align_up(off + (size_t)nq * c.n_q_heads * ntiles * 8, 256);
  L.F_off = off;  // per-KV-head score shares [nq][Hkv][sel_pad]
  off = align_up(off + (size_t)nq * c.n_kv_heads * L.sel_pad * 8, 256);
  {  // route3: per-range den rows, spilled selection-block sums, per-KV-head shares
    const int64_t chunks = route3_nchunks(c, nq);
    const int64_t nranges = route3_nranges_bound(c, L.sel_pad);
    L.r3_den_off = off;
    off = align_up(off + (size_t)(chunks * c.n_kv_heads * nranges * kR3Rows * 8), 256);
    L.r3_spill_off = off;
    off = align_up(off + (size_t)(chunks * c.n_kv_heads * nranges * (kR3Rows + 1) * kR3MaxSpr * 8), 256);
    L.r3_contrib_off = off;
    off = align_up(off + (size_t)(nq * L.sel_pad * 8), 256);
    L.r3_exact_off = off;  // the exact path's scratch, one slot at a time
    off = align_up(off + (size_t)c.n_q_heads * std::max<int64_t>(maxblk, 1) * 8, 256);
  }
  L.total = off;
  return L;
}

void validate_args(const specsv_nsa_config& c, const specsv_layer_kv& kv,
                   const specsv_verify_args& a) {
  if (a.n_queries < 1 || a.n_queries > kMaxQueries)
    throw Error(SPECSV_EUNSUPPORTED, "n_queries must be in [1, 65] (gamma <= 64)");
  if (a.group_size < 1) throw Error(SPECSV_EINVAL, "partition_groups: C must be >= 1");
  if (a.mode != SPECSV_MODE_EXACT && a.mode != SPECSV_MODE_APPROX)
    throw Error(SPECSV_EINVAL, "mode must be EXACT or APPROX");
  if (a.role != SPECSV_ROLE_REFRESH && a.role != SPECSV_ROLE_REUSE)
    throw Error(SPECSV_EINVAL, "role must be REFRESH or REUSE");
  if (a.pos == nullptr || a.q == nullptr || a.gates == nullptr || a.out == nullptr ||
      a.idx == nullptr || a.idx_count == nullptr || a.idx_forced == nullptr)
    throw Error(SPECSV_EINVAL, "null argument");
  if (kv.k == nullptr || kv.v == nullptr || kv.ck == nullptr || kv.ck16 == nullptr ||
      kv.cv == nullptr)
    throw Error(SPECSV_EINVAL, "null cache pointer");
  if (kv.rows < 1) throw Error(SPECSV_EINVAL, "rows must be >= 1 (the pending root is committed)");
  if ((kv.ckd == nullptr) != (kv.ckexp == nullptr))
    throw Error(SPECSV_EINVAL, "ckd and ckexp must both be set or both be NULL");
  if (kv.capacity < kv.rows) throw Error(SPECSV_EINVAL, "rows exceed the cache capacity");
  if (a.kv_head_count < 0 || a.kv_head_begin < 0 ||
      (int64_t)a.kv_head_begin + a.kv_head_count > c.n_kv_heads ||
      (a.kv_head_count == 0 && a.kv_head_begin != 0))
    throw Error(SPECSV_EINVAL, "KV-head range outside [0, n_kv_heads)");
  if (kv.rows > (int64_t)kMaxUnionWords * 32 * c.l_sel)
    throw Error(SPECSV_EUNSUPPORTED, "context exceeds this build's selection-block bitmap");
  const int64_t want_blocks = kv.rows >= c.l ? (kv.rows - c.l) / c.d + 1 : 0;
  if (kv.blocks < 0 || kv.blocks > want_blocks)
    throw Error(SPECSV_EINVAL, "compressed block count exceeds the committed rows");
  const int32_t gamma = a.n_queries - 1;
  if (gamma > 0 && (a.tree_k == nullptr || a.tree_v == nullptr || a.tree_mask == nullptr ||
                    a.mask_words < (gamma + 63) / 64))
    throw Error(SPECSV_EINVAL, "draft rows / tree mask missing");
  if (a.pos[0] < 0 || a.pos[0] > kv.rows - 1)
    throw Error(SPECSV_EINVAL, "root position must be a committed row");
  for (int32_t q = 1; q < a.n_queries; ++q) {
    if (a.pos[q] <= a.pos[0]) throw Error(SPECSV_EINVAL, "draft positions must follow the root");
    if (a.pos[q] - a.pos[0] > c.routing_lag)  // engine.cpp:479-480
      throw Error(SPECSV_EINVAL, "step: draft depth exceeds routing lag");
  }
  // the deepest query sees the most selection blocks; in DFS flat order that
  // need not be the last one, so bound every query
  int64_t max_pos = a.pos[0];
  for (int32_t q = 1; q < a.n_queries; ++q) max_pos = std::max(max_pos, a.pos[q]);
  if (selection_block_count(c, routing_visible_len(c, max_pos)) > kMaxAvail)
    throw Error(SPECSV_EUNSUPPORTED, "too many selection blocks for the Top-n kernel");
}

RouteParams make_route_params(const specsv_nsa_config& c, const specsv_layer_kv& kv,
                              const specsv_verify_args& a, const Layout& L, char* ws,
                              const std::vector<int32_t>& routed) {
  RouteParams p;
  std::memset(&p, 0, sizeof(p));
  p.q = a.q;
  p.ck = kv.ck;
  p.trace = g_trace;
  p.idx = a.idx;
  p.idx_count = a.idx_count;
  p.idx_forced = a.idx_forced;
  p.nr = static_cast<int32_t>(routed.size());
  p.nq = a.n_queries;
  p.Hq = (int32_t)c.n_q_heads;
  p.Hkv = (int32_t)c.n_kv_heads;
  p.G = (int32_t)(c.n_q_heads / c.n_kv_heads);
  p.dh = (int32_t)c.d_head;
  p.n = (int32_t)c.n;
  p.l = (int32_t)c.l;
  p.d = (int32_t)c.d;
  p.l_sel = (int32_t)c.l_sel;
  p.blocks = (int32_t)kv.blocks;
  p.scale = 1.0 / std::sqrt(static_cast<double>(c.d_head));
  int64_t mmax = 0;
  std::vector<bool> is_routed(a.n_queries, false);
  for (size_t s = 0; s < routed.size(); ++s) {
    const int32_t q = routed[s];
    is_routed[q] = true;
    const int64_t vis = routing_visible_len(c, a.pos[q]);
    p.slot_q[s] = q;
    p.slot_mvis[s] = (int32_t)visible_blocks(c, kv.blocks, vis);
    p.slot_avail[s] = (int32_t)selection_block_count(c, vis);
    mmax = std::max<int64_t>(mmax, p.slot_mvis[s]);
  }
  for (int32_t q = 0; q < a.n_queries; ++q)
    if (!is_routed[q]) p.unrouted[p.n_unrouted++] = q;
  p.m_pad = (int32_t)align_up((size_t)mmax, kRouteTile);
  p.ntiles = p.m_pad / kRouteTile;
  p.gsh = reinterpret_cast<double*>(ws + L.E_off);
  p.g_stride = (int32_t)(((kRouteTile - 1) * c.d + c.l - 1) / c.l_sel + 1);
  p.TM = reinterpret_cast<double*>(ws + L.TM_off);
  p.TD = reinterpret_cast<double*>(ws + L.TD_off);
  p.part = reinterpret_cast<double*>(ws + L.F_off);
  p.sel_pad = (int32_t)L.sel_pad;
  p.counters = reinterpret_cast<int32_t*>(ws + L.cnt_off);
  p.slot_done = p.counters + 4;
  return p;
}

void run_route(const specsv_nsa_config& c, const specsv_layer_kv& kv, const specsv_verify_args& a,
               void* ws, size_t ws_bytes, cudaStream_t stream);
bool use_route3(const specsv_layer_kv& kv);
void make_route3_req(const specsv_nsa_config& c, const specsv_layer_kv& kv, const specsv_verify_args& a,
                     const Layout& L, char* base, const std::vector<int32_t>& routed, int32_t* cnt,
                     bool spread, Route3Req& R);
void fill_route3_common(const specsv_nsa_config& c, const Layout& L, char* ws, Route3Launch& P);
int32_t* route3_cnt(const Layout& L, char* ws, int r);

// bytes of one request's routing regions (E, TM, TD, F); a batched routing
// launch places request q's at E_off + q x route_bytes
size_t route_bytes(const Layout& L) { return L.total - L.E_off; }

// routing of the REFRESH requests of a batch: one cooperative launch per
// group of up to kRouteBatch requests whose regions fit the workspace
// (specsv_verify_workspace_size_batched); a group of one is the single path
void run_route_batched(const specsv_nsa_config& c, const specsv_layer_kv* kvs,
                       const specsv_verify_args* args, int32_t batch, void* ws, size_t ws_bytes,
                       cudaStream_t stream) {
  std::vector<int32_t> refresh;
  int32_t max_nq = 1;
  int64_t max_rows = 0;
  for (int32_t b = 0; b < batch; ++b)
    if (args[b].role == SPECSV_ROLE_REFRESH) {
      refresh.push_back(b);
      max_nq = std::max(max_nq, args[b].n_queries);
      max_rows = std::max(max_rows, kvs[b].rows);
    }
  if (refresh.empty()) return;
  const Layout L = layout_for(c, max_nq, max_rows);
  if (ws == nullptr || ws_bytes < L.total) throw Error(SPECSV_ENOSPACE, "workspace too small");
  const size_t cap = 1 + (ws_bytes - L.total) / std::max<size_t>(route_bytes(L), 1);
  const int group = (int)std::min<size_t>({(size_t)kRouteBatch, (size_t)kSyncSets, cap});
  char* w = static_cast<char*>(ws);
  bool all3 = true;
  for (int32_t b : refresh) all3 = all3 && use_route3(kvs[b]);
  if (all3) {
    const int group3 = (int)std::min<size_t>((size_t)kR3Batch, cap);
    thread_local Route3Launch P;
    for (size_t g0 = 0; g0 < refresh.size(); g0 += group3) {
      const int n = (int)std::min<size_t>(group3, refresh.size() - g0);
      std::memset(&P, 0, sizeof(P));
      fill_route3_common(c, L, w, P);
      P.n_req = n;
      for (int q = 0; q < n; ++q) {
        const int32_t b = refresh[g0 + q];
        const auto routed = routed_queries(args[b].n_queries, args[b].pos, args[b].group_size, args[b].mode);
        make_route3_req(c, kvs[b], args[b], L, w + L.E_off + (size_t)q * route_bytes(L), routed,
                        route3_cnt(L, w, q), n == 1, P.req[q]);
      }
      cuda_check(launch_route3(P, stream), "batched route launch");
    }
    return;
  }
  thread_local RouteBatch rb;  // ~20 KB host staging of the launch parameters
  for (size_t g0 = 0; g0 < refresh.size(); g0 += group) {
    const int n = (int)std::min<size_t>(group, refresh.size() - g0);
    if (n == 1) {
      run_route(c, kvs[refresh[g0]], args[refresh[g0]], ws, ws_bytes, stream);
      continue;
    }
    std::memset(&rb, 0, sizeof(rb));
    rb.n_req = n;
    for (int q = 0; q < n; ++q) {
      const int32_t b = refresh[g0 + q];
      const auto routed = routed_queries(args[b].n_queries, args[b].pos, args[b].group_size, args[b].mode);
      rb.req[q] = make_route_params(c, kvs[b], args[b], L, w + (size_t)q * route_bytes(L), routed);
      rb.req[q].counters = reinterpret_cast<int32_t*>(w + L.cnt_off) + (size_t)q * kCntSetInts;
      rb.req[q].slot_done = rb.req[q].counters + 4;
      rb.req[q].trace = nullptr;
    }
    cuda_check(launch_route_batch(rb, stream), "batched route launch");
  }
}

// the routing kernel of a call: route3_kernel (integer tensor pipe, certified
// Top-n) whenever the cache carries digit planes; route_fused_kernel (fp64
// DMMA over ck) otherwise or with SPECSV_ROUTE_LEGACY=1
bool use_route3(const specsv_layer_kv& kv) { return kv.ckd != nullptr && !debug_env().route_legacy; }

// one request's route3 parameters; `base` is its routing region (E_off-relative
// offsets of the layout apply); `spread`: ranges per (chunk, KV head) may grow
// until the units fill the device (a launch of one request)
void make_route3_req(const specsv_nsa_config& c, const specsv_layer_kv& kv, const specsv_verify_args& a,
                     const Layout& L, char* base, const std::vector<int32_t>& routed, int32_t* cnt,
                     bool spread, Route3Req& R) {
  std::memset(&R, 0, sizeof(R));
  encode_ckd_map(&R.tm_ckd, kv.ckd, kv.blocks, c.n_kv_heads, c.d_head);
  R.ckexp = kv.ckexp;
  R.q = a.q;
  R.ck = kv.ck;
  R.idx = a.idx;
  R.idx_count = a.idx_count;
  R.idx_forced = a.idx_forced;
  R.nr = static_cast<int32_t>(routed.size());
  R.blocks = (int32_t)kv.blocks;
  R.sel_pad = (int32_t)L.sel_pad;
  R.cnt = cnt;
  int64_t amax = 0;
  std::vector<bool> is_routed(a.n_queries, false);
  for (size_t s = 0; s < routed.size(); ++s) {
    const int32_t q = routed[s];
    is_routed[q] = true;
    const int64_t vis = routing_visible_len(c, a.pos[q]);
    R.slot_q[s] = q;
    R.slot_mvis[s] = (int32_t)visible_blocks(c, kv.blocks, vis);
    R.slot_avail[s] = (int32_t)selection_block_count(c, vis);
    amax = std::max<int64_t>(amax, R.slot_avail[s]);
  }
  for (int32_t q = 0; q < a.n_queries; ++q)
    if (!is_routed[q]) R.unrouted[R.n_unrouted++] = q;
  R.avail_max = (int32_t)amax;
  R.nchunks = (int32_t)route3_nchunks(c, R.nr);
  const int64_t per = R.nchunks * c.n_kv_heads;
  if (per > kR3CntPerReq - 176) throw Error(SPECSV_EUNSUPPORTED, "route3: too many row chunks x KV heads");
  int64_t nranges = std::max<int64_t>(1, (amax + route3_spr_max(c) - 1) / route3_spr_max(c));
  if (spread) nranges = std::max<int64_t>(nranges, route3_grid() / per);
  const int64_t spr = std::max<int64_t>(1, (amax + nranges - 1) / nranges);
  nranges = std::max<int64_t>(1, (amax + spr - 1) / spr);
  if (nranges > route3_nranges_bound(c, L.sel_pad))
    throw Error(SPECSV_EUNSUPPORTED, "route3: selection-block ranges exceed the workspace bound");
  R.nranges = (int32_t)nranges;
  R.spr = (int32_t)spr;
  const size_t rel = L.E_off;  // region offsets are relative to the request's routing region
  R.den = reinterpret_cast<double*>(base + (L.r3_den_off - rel));
  R.gspill = reinterpret_cast<double*>(base + (L.r3_spill_off - rel));
  R.contrib = reinterpret_cast<double*>(base + (L.r3_contrib_off - rel));
  R.exact = reinterpret_cast<double*>(base + (L.r3_exact_off - rel));
}

void fill_route3_common(const specsv_nsa_config& c, const Layout& L, char* ws, Route3Launch& P) {
  P.Hq = (int32_t)c.n_q_heads;
  P.Hkv = (int32_t)c.n_kv_heads;
  P.G = (int32_t)(c.n_q_heads / c.n_kv_heads);
  P.n = (int32_t)c.n;
  P.l = (int32_t)c.l;
  P.d = (int32_t)c.d;
  P.l_sel = (int32_t)c.l_sel;
  P.spc = (int32_t)route3_spc(c);
  P.bps = (int32_t)((c.l_sel - 1 + c.l - 1) / c.d + 1);  // blocks_of: hi - lo + 1 at most
  if (P.bps > kR3MaxBps) throw Error(SPECSV_EUNSUPPORTED, "route3: too many compressed blocks per selection block");
  P.scale = 1.0 / std::sqrt(static_cast<double>(c.d_head));
  P.c_sl = 1.4426950408889634073599 / std::sqrt(static_cast<double>(c.d_head));
  int32_t* cnt = reinterpret_cast<int32_t*>(ws + L.r3cnt_off);
  P.exit_cnt = cnt;
  P.fallbacks = cnt + 4;
  P.force_exact = debug_env().force_exact ? 1 : 0;  // tests: the exact re-scoring path
  P.debug = debug_env().route3_debug;
  P.trace = g_trace;
  if (c.d_head != kR3Tile) throw Error(SPECSV_EUNSUPPORTED, "route3: d_head must be 128");
}

// counter set `r` of a route3 launch
int32_t* route3_cnt(const Layout& L, char* ws, int r) {
  return reinterpret_cast<int32_t*>(ws + L.r3cnt_off) + 8 + (size_t)r * kR3CntPerReq;
}

void run_route(const specsv_nsa_config& c, const specsv_layer_kv& kv, const specsv_verify_args& a,
               void* ws, size_t ws_bytes, cudaStream_t stream) {
  const Layout L = layout_for(c, a.n_queries, kv.rows);
  if (ws == nullptr || ws_bytes < L.total) throw Error(SPECSV_ENOSPACE, "workspace too small");
  const auto routed = routed_queries(a.n_queries, a.pos, a.group_size, a.mode);
  if (use_route3(kv)) {
    thread_local Route3Launch P;  // ~33 KB host staging of the launch parameters
    std::memset(&P, 0, sizeof(P));
    char* w = static_cast<char*>(ws);
    fill_route3_common(c, L, w, P);
    P.n_req = 1;
    make_route3_req(c, kv, a, L, w + L.E_off, routed, route3_cnt(L, w, 0), true, P.req[0]);
    cuda_check(launch_route3(P, stream), "route launch");
    return;
  }
  RouteParams p = make_route_params(c, kv, a, L, static_cast<char*>(ws), routed);
  cuda_check(launch_route(p, stream, true), "route launch");
}

// everything of one request's attend launch but its workspace slices
void fill_attend_params(AttendParams& p, const specsv_nsa_config& c, const specsv_layer_kv& kv,
                        const specsv_verify_args& a, int S) {
  std::memset(&p, 0, sizeof(p));
  const int64_t H = c.n_kv_heads, dh = c.d_head;
  const int32_t gamma = a.n_queries - 1;
  encode_rows_map(&p.tm_k, kv.k, kv.rows, H, dh);
  encode_rows_map(&p.tm_v, kv.v, kv.rows, H, dh);
  encode_rows_map(&p.tm_ck, kv.ck16, kv.blocks, H, dh);
  encode_rows_map(&p.tm_cv, kv.cv, kv.blocks, H, dh);
  encode_rows_map(&p.tm_tk, gamma > 0 ? a.tree_k : kv.k, std::max(gamma, 1), H, dh);
  encode_rows_map(&p.tm_tv, gamma > 0 ? a.tree_v : kv.v, std::max(gamma, 1), H, dh);
  p.k_raw = static_cast<const uint16_t*>(kv.k);
  p.q = a.q;
  p.gates = a.gates;
  p.out = a.out;
  p.idx = a.idx;
  p.idx_count = a.idx_count;
  p.trace = g_trace;
  p.idx_early = a.role == SPECSV_ROLE_REUSE ? 1 : 0;
  p.debug_flags = (debug_env().force_robust ? 1 : 0) | debug_env().attend_debug;  // tests / timing experiments
  const int qc = qc_size_for(c);
  const int nchunks = (a.n_queries + qc - 1) / qc;
  p.nq = a.n_queries;
  p.gamma = gamma;
  p.Hq = (int32_t)c.n_q_heads;
  p.Hkv = (int32_t)H;
  p.G = (int32_t)(c.n_q_heads / H);
  p.n_sel = (int32_t)c.n;
  p.rows = (int32_t)kv.rows;
  p.blocks = (int32_t)kv.blocks;
  p.l = (int32_t)c.l;
  p.d = (int32_t)c.d;
  p.l_sel = (int32_t)c.l_sel;
  p.w = (int32_t)c.w;
  p.lag = (int32_t)c.routing_lag;
  p.qc_size = qc;
  p.n_splits = S;
  p.kvh0 = a.kv_head_count > 0 ? a.kv_head_begin : 0;
  p.nkvh = head_count(c, a);
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)dh));
  const auto src = source_rows(c, a.n_queries, a.pos, a.group_size, a.mode);
  for (int32_t q = 0; q < a.n_queries; ++q) {
    p.pos[q] = (int32_t)a.pos[q];
    p.src_row[q] = src[q];
    p.tree_mask[q] = (q < gamma) ? a.tree_mask[(int64_t)q * a.mask_words] : 0ull;
    const int64_t vis = routing_visible_len(c, a.pos[q]);
    p.qbound[q] = (int32_t)std::min<int64_t>(vis, kv.rows);
    p.qwlo[q] = (int32_t)std::max<int64_t>(0, a.pos[q] - c.w + 1);
    p.qwhi[q] = (int32_t)std::min<int64_t>(a.pos[q], kv.rows - 1);
    p.qmvis[q] = (int32_t)visible_blocks(c, kv.blocks, vis);
  }
  for (int ch = 0; ch < nchunks; ++ch) {
    int32_t mv = 0, wlo = INT32_MAX, whi = -1;
    for (int32_t q = ch * qc; q < std::min<int32_t>(a.n_queries, (ch + 1) * qc); ++q) {
      mv = std::max(mv, p.qmvis[q]);
      wlo = std::min(wlo, p.qwlo[q]);
      whi = std::max(whi, p.qwhi[q]);
    }
    p.ch_ncmp[ch] = (mv + 127) / 128;
    p.ch_wlo[ch] = wlo;
    p.ch_whi[ch] = whi;
  }
}

// request r's partial slice (units of the widest request in the launch) and
// barrier-word set r
void set_attend_ws(AttendParams& p, const Layout& L, char* ws, int r, int chunks, int S, int64_t H) {
  const int64_t units = (int64_t)chunks * H * S;
  float* base = reinterpret_cast<float*>(ws + L.attend_off);
  p.ws = base + r * units * (3 * kAttendCols * 2 + 3 * kAttendCols * kAttendDh);
  p.ws_o_offset = units * (3 * kAttendCols * 2);
  int32_t* sync = reinterpret_cast<int32_t*>(ws + L.sync_off) + (int64_t)r * L.max_chunks * H * 2;
  p.ws_sync_offset = reinterpret_cast<float*>(sync) - p.ws;
}

void run_attend(const specsv_nsa_config& c, const specsv_layer_kv& kv, const specsv_verify_args& a,
                void* ws, size_t ws_bytes, cudaStream_t stream, bool after_route = false) {
  const int S = splits_for(c, a.n_queries, head_count(c, a),
                           after_route ? debug_env().attend_splits_refresh : 0);
  const Layout L = layout_for(c, a.n_queries, kv.rows);
  if (ws == nullptr || ws_bytes < L.total) throw Error(SPECSV_ENOSPACE, "workspace too small");
  AttendParams p;
  fill_attend_params(p, c, kv, a, S);
  const int nchunks = (a.n_queries + p.qc_size - 1) / p.qc_size;
  if (S > 1) check_coresident(S * p.nkvh * nchunks, "attend launch");
  set_attend_ws(p, L, static_cast<char*>(ws), 0, nchunks, S, c.n_kv_heads);
  cuda_check(launch_attend(p, nchunks, stream), "attend launch");
}

// One attend launch per kAttendBatch requests: S splits per head with
// R x S <= 18 (the workspace's partial region) and, when S > 1, the grid
// co-resident (cooperative); S = 1 needs no cross-CTA merge and may span waves.
void run_attend_batched(const specsv_nsa_config& c, const specsv_layer_kv* kvs,
                        const specsv_verify_args* args, int32_t batch, void* ws, size_t ws_bytes,
                        cudaStream_t stream) {
  const int qc = qc_size_for(c);
  const int64_t H = c.n_kv_heads;
  thread_local AttendBatch b;  // ~31 KB host staging of the launch parameters (copied at launch)
  for (int32_t b0 = 0; b0 < batch; b0 += kAttendBatch) {
    const int R = std::min<int32_t>(kAttendBatch, batch - b0);
    int32_t max_nq = 1;
    int64_t max_rows = 0;
    for (int r = 0; r < R; ++r) {
      max_nq = std::max(max_nq, args[b0 + r].n_queries);
      max_rows = std::max(max_rows, kvs[b0 + r].rows);
    }
    int heads = 1;
    for (int r = 0; r < R; ++r) heads = std::max(heads, head_count(c, args[b0 + r]));
    const int chunks = (max_nq + qc - 1) / qc;
    const Layout L = layout_for(c, max_nq, max_rows);
    if (ws == nullptr || ws_bytes < L.total) throw Error(SPECSV_ENOSPACE, "workspace too small");
    const int groups = heads * chunks * R;
    const int S = std::max(1, std::min({18 / R, coresident_for_device() / groups, 18}));
    std::memset(&b, 0, sizeof(b));
    b.n_req = R;
    b.n_chunks = chunks;
    for (int r = 0; r < R; ++r) {
      fill_attend_params(b.req[r], c, kvs[b0 + r], args[b0 + r], S);
      set_attend_ws(b.req[r], L, static_cast<char*>(ws), r, chunks, S, H);
    }
    if (S > 1) check_coresident(S * groups, "batched attend launch");
    cuda_check(launch_attend_batch(b, S, heads, S > 1, stream), "batched attend launch");
  }
}

}  // namespace
}  // namespace specsv_b200

using namespace specsv_b200;

extern "C" {

int32_t specsv_abi_version(void) { return SPECSV_ABI_VERSION; }

int32_t specsv_debug_route3_counter_offset(const specsv_nsa_config* cfg, int32_t n_queries,
                                           int64_t max_rows) {
  if (cfg == nullptr || n_queries < 1) return -1;
  return (int32_t)(layout_for(*cfg, n_queries, max_rows).r3cnt_off / sizeof(int32_t)) + 4;
}

specsv_status specsv_debug_attend_trace(unsigned long long* buf) {
  g_trace = buf;
  return SPECSV_OK;
}

const char* specsv_last_error(void) { return last_error().c_str(); }

specsv_status specsv_validate_config(const specsv_nsa_config* cfg) {
  return guarded([&] {
    if (cfg == nullptr) throw Error(SPECSV_EINVAL, "null config");
    validate_config(*cfg);
    check_build_limits(*cfg);
  });
}

size_t specsv_verify_workspace_size(const specsv_nsa_config* cfg, int32_t n_queries,
                                    int64_t max_rows) {
  if (cfg == nullptr || n_queries < 1) return 0;
  return layout_for(*cfg, n_queries, max_rows).total;
}

size_t specsv_verify_workspace_size_batched(const specsv_nsa_config* cfg, int32_t n_queries,
                                            int64_t max_rows, int32_t batch) {
  if (cfg == nullptr || n_queries < 1 || batch < 1) return 0;
  const Layout L = layout_for(*cfg, n_queries, max_rows);
  const int32_t r = std::min<int32_t>(batch, std::min(kRouteBatch, kSyncSets));
  return L.total + (size_t)(r - 1) * route_bytes(L);
}

specsv_status specsv_nsa_route(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                               const specsv_verify_args* args, void* ws, size_t ws_bytes,
                               specsv_stream_t stream) {
  return guarded([&] {
    if (!cfg || !kv || !args) throw Error(SPECSV_EINVAL, "null argument");
    validate_config(*cfg);
    check_build_limits(*cfg);
    validate_args(*cfg, *kv, *args);
    run_route(*cfg, *kv, *args, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
  });
}

specsv_status specsv_nsa_attend_fused(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                                      const specsv_verify_args* args, void* ws, size_t ws_bytes,
                                      specsv_stream_t stream) {
  return guarded([&] {
    if (!cfg || !kv || !args) throw Error(SPECSV_EINVAL, "null argument");
    validate_config(*cfg);
    check_build_limits(*cfg);
    validate_args(*cfg, *kv, *args);
    run_attend(*cfg, *kv, *args, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
  });
}

specsv_status specsv_nsa_verify(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                                const specsv_verify_args* args, void* ws, size_t ws_bytes,
                                specsv_stream_t stream) {
  return guarded([&] {
    if (!cfg || !kv || !args) throw Error(SPECSV_EINVAL, "null argument");
    validate_config(*cfg);
    check_build_limits(*cfg);
    validate_args(*cfg, *kv, *args);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const bool refresh = args->role == SPECSV_ROLE_REFRESH;
    if (refresh) run_route(*cfg, *kv, *args, ws, ws_bytes, s);
    run_attend(*cfg, *kv, *args, ws, ws_bytes, s, refresh);
  });
}

specsv_status specsv_nsa_verify_batched(const specsv_nsa_config* cfg, const specsv_layer_kv* kvs,
                                        const specsv_verify_args* args, int32_t batch, void* ws,
                                        size_t ws_bytes, specsv_stream_t stream) {
  return guarded([&] {
    if (!cfg || !kvs || !args || batch < 0) throw Error(SPECSV_EINVAL, "null argument");
    validate_config(*cfg);
    check_build_limits(*cfg);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // validate the whole batch before the first launch: a bad request must not
    // leave the ones before it half-verified
    for (int32_t b = 0; b < batch; ++b) validate_args(*cfg, kvs[b], args[b]);
    run_route_batched(*cfg, kvs, args, batch, ws, ws_bytes, s);
    run_attend_batched(*cfg, kvs, args, batch, ws, ws_bytes, s);
  });
}

specsv_status specsv_nsa_scores(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                                const specsv_verify_args* args, int32_t query, double* scores,
                                void* ws, size_t ws_bytes, specsv_stream_t stream) {
  return guarded([&] {
    if (!cfg || !kv || !args || !scores) throw Error(SPECSV_EINVAL, "null argument");
    validate_config(*cfg);
    check_build_limits(*cfg);
    validate_args(*cfg, *kv, *args);
    if (query < 0 || query >= args->n_queries) throw Error(SPECSV_EINVAL, "query out of range");
    const Layout L = layout_for(*cfg, args->n_queries, kv->rows);
    if (ws == nullptr || ws_bytes < L.total) throw Error(SPECSV_ENOSPACE, "workspace too small");
    std::vector<int32_t> routed{query};
    RouteParams p = make_route_params(*cfg, *kv, *args, L, static_cast<char*>(ws), routed);
    cuda_check(launch_scores_only(p, scores, 0, reinterpret_cast<cudaStream_t>(stream)),
               "scores launch");
  });
}

specsv_status specsv_select_blocks(const specsv_nsa_config* cfg, const double* scores,
                                   int64_t visible_len, int32_t* idx, int32_t* count,
                                   uint32_t* forced, specsv_stream_t stream) {
  return guarded([&] {
    if (!cfg || !scores || !idx || !count || !forced) throw Error(SPECSV_EINVAL, "null argument");
    validate_config(*cfg);
    if (cfg->n > 64) throw Error(SPECSV_EUNSUPPORTED, "n must be <= 64");
    const int64_t avail = selection_block_count(*cfg, visible_len);
    if (avail > kMaxAvail) throw Error(SPECSV_EUNSUPPORTED, "too many selection blocks");
    cuda_check(launch_select(scores, (int)avail, (int)cfg->n, idx, count, forced,
                             reinterpret_cast<cudaStream_t>(stream)),
               "select launch");
  });
}

specsv_status specsv_compress_append(const specsv_nsa_config* cfg, const specsv_layer_kv* kv,
                                     int64_t first_block, int64_t last_block,
                                     const float* pos_embed, specsv_stream_t stream) {
  return guarded([&] {
    if (!cfg || !kv) throw Error(SPECSV_EINVAL, "null argument");
    validate_config(*cfg);
    if (cfg->d_head > 1024) throw Error(SPECSV_EUNSUPPORTED, "d_head too large");
    if (kv->rows < 0 || kv->rows > kv->capacity)
      throw Error(SPECSV_EINVAL, "rows exceed the cache capacity");
    const int64_t want = kv->rows >= cfg->l ? (kv->rows - cfg->l) / cfg->d + 1 : 0;
    if (first_block < 0 || last_block > want || first_block > last_block)
      throw Error(SPECSV_EINVAL, "block range outside the committed rows");
    if (!kv->k || !kv->v || !kv->ck || !kv->ck16 || !kv->cv)
      throw Error(SPECSV_EINVAL, "null cache pointer");
    if ((kv->ckd == nullptr) != (kv->ckexp == nullptr))
      throw Error(SPECSV_EINVAL, "ckd and ckexp must both be set or both be NULL");
    cuda_check(launch_compress(kv->k, kv->v, pos_embed, kv->ck, kv->ck16, kv->cv, kv->ckd, kv->ckexp,
                               first_block, last_block, (int)cfg->n_kv_heads, (int)cfg->d_head, (int)cfg->l,
                               (int)cfg->d, reinterpret_cast<cudaStream_t>(stream)),
               "compress launch");
  });
}

specsv_status specsv_resolve_layer_roles(const int64_t* reuse_set, int64_t n_reuse,
                                         int64_t n_layers, int32_t* roles, int64_t* source) {
  return guarded([&] {
    if ((n_reuse > 0 && !reuse_set) || !roles || !source) throw Error(SPECSV_EINVAL, "null argument");
    resolve_layer_roles(reuse_set, n_reuse, n_layers, roles, source);
  });
}

specsv_status specsv_clamp_inherited(const specsv_nsa_config* cfg, const int32_t* src,
                                     uint32_t src_forced, int32_t count, int64_t causal_bound,
                                     int32_t* out, uint32_t* out_forced, int32_t* out_count) {
  return guarded([&] {
    if (!cfg || (count > 0 && !src) || !out || !out_count) throw Error(SPECSV_EINVAL, "null argument");
    *out_count = clamp_inherited(*cfg, src, src_forced, count, causal_bound, out, out_forced);
  });
}

specsv_status specsv_load_stats(const specsv_nsa_config* cfg, int64_t rows, int32_t n_queries,
                                const int64_t* pos, const uint64_t* tree_mask, int32_t mask_words,
                                int32_t group_size, int32_t mode, int32_t role, const int32_t* idx,
                                const int32_t* idx_count, specsv_load_stats_t* out) {
  return guarded([&] {
    if (!cfg || !pos || !idx || !idx_count || !out) throw Error(SPECSV_EINVAL, "null argument");
    if (n_queries > 1 && !tree_mask) throw Error(SPECSV_EINVAL, "null tree mask");
    load_stats(*cfg, rows, n_queries, pos, tree_mask, mask_words, group_size, mode, role, idx,
               idx_count, out);
  });
}

specsv_status specsv_algorithmic_bytes(const specsv_nsa_config* cfg, int64_t rows,
                                       int32_t n_queries, const int64_t* pos, int32_t role,
                                       const int32_t* idx, const int32_t* idx_count, int32_t mode,
                                       int32_t group_size, int64_t* bytes) {
  return guarded([&] {
    if (!cfg || !pos || !idx || !idx_count || !bytes) throw Error(SPECSV_EINVAL, "null argument");
    *bytes = algorithmic_bytes(*cfg, rows, n_queries, pos, role, idx, idx_count, mode, group_size);
  });
}

}  // extern "C"
