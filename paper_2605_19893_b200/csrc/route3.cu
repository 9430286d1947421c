// route3.cu -- refresh-layer routing on sm_100a's integer tensor pipe:
// compressed-block selection scores and Top-n with forced blocks, for up to
// kR3Batch requests in one cooperative launch.
//
// Replaces nsa::selection_scores + nsa::select_blocks
// (src/nsa_attention.cpp:38-136) for every query that constructs indices.
//
// Logits.  The reference forms logit = dot(q_h, ck_i) / sqrt(dh) in double
// from fp32 operands (nsa_attention.cpp:51-56).  Here every q row and every
// key row is a 31-bit fixed-point integer on its own power-of-two grid
// (X = round(x 2^(30 - e)), |x| < 2^e the row maximum), split into four signed
// base-256 digits.  Digit products are exact s8 x s8 -> s32 tcgen05 MMAs
// (kind::i8, M = 128 blocks, N = 48 (query, head) rows, K = 128): the 13
// digit pairs of weight >= 256^2 accumulate exactly into five TMEM columns
// sets by weight class, which the epilogue recombines in int64.  The result
// differs from the exact fp32-operand dot by at most 2^-21.9 |q|_max |k|_max
// (grid rounding plus the three dropped low pairs), a bound carried per row.
//
// Scores.  Per unit and row: tile max, e = 2^(logit - max) in fp64, tile sum
// and the tile's selection-block sums G_b = sum_i overlap(i, b) e_i.  One
// grid barrier later every unit normalises its rows (max / denominator over
// all tiles of the row), folds the GQA heads of each slot, and writes the KV
// head's share per selection block.  A second arrival gates the Top-n tasks
// (one per (request, slot)): score_b = sum over KV heads and tiles of the
// shares / (Hq l) -- the reference's sum over heads and blocks of
// p * overlap / l (nsa_attention.cpp:57-78), regrouped.
//
// Certification.  Each logit error bound delta (log2 units) makes every
// probability exact to a factor 2^(+-2 delta), so every score is within a
// relative eps = 2 ln2 delta_max of its exact value.  The Top-n (forced
// {0, avail-2, avail-1} plus the best by (score desc, id asc),
// nsa_attention.cpp:94-136) is accepted when the last pick and the best
// non-pick are separated by more than eps; otherwise the task re-scores its
// query exactly in fp64 (the reference's arithmetic, regrouped) and selects on
// those scores.  The indices therefore equal the reference's whatever the
// inputs; the re-scoring path is exercised by tests (force_exact).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "attend.h"
#include "sm100.cuh"

namespace specsv_b200 {
namespace {

using namespace sm100;

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kTB = kR3Tile;   // compressed blocks per unit
constexpr int kDh = 128;
constexpr int kN = kR3Rows;    // q rows per unit
constexpr int kAcc = 5;        // digit-pair weight classes 256^2 .. 256^6
constexpr uint32_t kTmemCols = 256;
constexpr int kTopnGroups = kThreads / 4;

// shared memory map (bytes from the 1024-aligned base)
constexpr uint32_t kOffStage = 0;                    // 2 x fp32 key tile [128][128] (TMA)
constexpr uint32_t kStageBytes = kTB * kDh * 4;      // 65536
constexpr uint32_t kOffKs = 2 * kStageBytes;         // key digits [4][128 rows x 128 B], SW128
constexpr uint32_t kKsSlice = kTB * 128;             // 16384
constexpr uint32_t kOffQs = kOffKs + 4 * kKsSlice;   // q digits [4][48 rows x 128 B], SW128
constexpr uint32_t kQsSlice = kN * 128;              // 6144
constexpr uint32_t kOffMisc = kOffQs + 4 * kQsSlice;
static_assert(kN * kTB * 8 <= 4 * kKsSlice, "fp64 logits alias the key digits");
static_assert(kQsSlice % 1024 == 0, "SW128 atoms");
static_assert((size_t)kMaxAvail * 12 <= 2 * kStageBytes, "Top-n arrays alias the key stages");

struct Misc {
  uint64_t tma_full[2], mma_done;
  uint32_t tmem_base;
  int32_t kexp[kTB];
  float kmax[kTB];
  int32_t qexp[kN];
  float qmax[kN];
  double F[kN];       // phase C: this unit's tile weight per row
  double E[kN];       // phase C: row error bound (log2 units)
  double red_m[kWarps][4], red_s[kWarps][4];  // exact path: per-warp (max, sum)
  double fin_m[4], fin_s[4];
  double gbest_s[kTopnGroups];
  int32_t gbest_i[kTopnGroups];
  int32_t picks[64];
  double lb_s, sk, sk1;
  int32_t lb_i, nsurv, certified;
  uint32_t fbits;
  double red_w[kWarps];
};
constexpr size_t kSmemBytes = kOffMisc + sizeof(Misc) + 1024;
static_assert(kSmemBytes <= 232448, "shared memory budget");

__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// e^x for x <= 0, ~2 ulp (x = n ln2 + r, Taylor to degree 12); x < -708 -> 0
__device__ __forceinline__ double exp_nonpos(double x) {
  if (!(x >= -708.0)) return 0.0;
  const double n = rint(x * 1.4426950408889634);
  double r = fma(n, -6.93147180369123816490e-01, x);
  r = fma(n, -1.90821492927058770002e-10, r);
  double p = 2.08767569878680989792e-09;
  p = fma(p, r, 2.50521083854417187751e-08);
  p = fma(p, r, 2.75573192239858906526e-07);
  p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05);
  p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03);
  p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02);
  p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return __hiloint2double(__double2hiint(p) + (static_cast<int>(n) << 20), __double2loint(p));
}

// 2^x for x <= 0 (x in log2 units), ~2 ulp: x = n + f, f in [-1/2, 1/2],
// 2^f = e^(f ln2) by Taylor to degree 11 (|f ln2| <= 0.347: < 1e-17)
__device__ __forceinline__ double exp2_nonpos(double x) {
  if (!(x >= -1020.0)) return 0.0;
  const double n = rint(x);
  const double r = (x - n) * 6.93147180559945309417e-01;
  double p = 2.50521083854417187751e-08;
  p = fma(p, r, 2.75573192239858906526e-07);
  p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05);
  p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03);
  p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02);
  p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return __hiloint2double(__double2hiint(p) + (static_cast<int>(n) << 20), __double2loint(p));
}

__device__ __forceinline__ double pow2i(int k) {  // 2^k, |k| <= 1022
  return __longlong_as_double(static_cast<long long>(1023 + k) << 52);
}

// tokens shared by compressed block i ([i d, i d + l)) and selection block b
__device__ __forceinline__ int overlap(int i, int b, int d, int l, int l_sel) {
  const int lo = max(i * d, b * l_sel), hi = min(i * d + l, (b + 1) * l_sel);
  return hi > lo ? hi - lo : 0;
}

// compressed blocks overlapping selection block b: [lo, hi]
__device__ __forceinline__ void blocks_of(int b, int d, int l, int l_sel, int& lo, int& hi) {
  const int num = b * l_sel - l;  // i > num / d
  lo = num >= 0 ? num / d + 1 : 0;
  hi = ((b + 1) * l_sel - 1) / d;
}

// four signed base-256 digits of round(x 2^shift) (|x 2^shift| <= 2^30):
// byte s of the result is the digit of weight 256^s
__device__ __forceinline__ uint32_t digits4(float x, float sc) {
  const int X = __float2int_rn(x * sc);
  return (static_cast<uint32_t>(X) + 0x80808080u) ^ 0x80808080u;
}

// row `row` (4 consecutive elements per lane, a 128-element row per warp) of
// a digit-sliced K-major SW128 operand: slice s at base + s * slice_bytes
__device__ __forceinline__ void write_digit_row(uint8_t* base, uint32_t slice_bytes, int row, int lane,
                                                float4 v, int e) {
  const int shift = 30 - e;
  float sc;
  if (shift >= -126 && shift <= 127) {
    sc = __int_as_float((127 + shift) << 23);
  } else {  // extreme row magnitudes: scale in two exact steps
    v.x = ldexpf(v.x, shift - shift / 2);
    v.y = ldexpf(v.y, shift - shift / 2);
    v.z = ldexpf(v.z, shift - shift / 2);
    v.w = ldexpf(v.w, shift - shift / 2);
    sc = ldexpf(1.0f, shift / 2);
  }
  const uint32_t w0 = digits4(v.x, sc), w1 = digits4(v.y, sc), w2 = digits4(v.z, sc),
                 w3 = digits4(v.w, sc);
  const uint32_t off = sw128_off(row, lane >> 2) + 4 * (lane & 3);
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const uint32_t sel = s | ((s + 4) << 4);
    const uint32_t lo = __byte_perm(w0, w1, sel), hi = __byte_perm(w2, w3, sel);
    *reinterpret_cast<uint32_t*>(base + s * slice_bytes + off) = __byte_perm(lo, hi, 0x5410);
  }
}

struct UnitInfo {
  int req, kvh, chunk, tile, r0, nrows;
};

__device__ __forceinline__ UnitInfo unit_info(const Route3Launch& P, int u) {
  int r = 0;
  while (r + 1 < P.n_req && u >= P.unit_start[r + 1]) ++r;
  const Route3Req& R = P.req[r];
  int lu = u - P.unit_start[r];
  UnitInfo U;
  U.req = r;
  U.tile = lu % R.ntiles;
  lu /= R.ntiles;
  U.kvh = lu % P.Hkv;
  U.chunk = lu / P.Hkv;
  U.r0 = U.chunk * P.chunk_rows;
  U.nrows = min(P.chunk_rows, R.nr * P.G - U.r0);
  return U;
}

__device__ __forceinline__ int64_t unit_gsh_offset(const Route3Launch& P, const UnitInfo& U, int u) {
  return (int64_t)(u - P.unit_start[U.req]) * kN * P.span;
}

__device__ __forceinline__ void issue_unit_tma(const Route3Launch& P, int u, uint8_t* dst, uint64_t* bar) {
  const UnitInfo U = unit_info(P, u);
  mbar_expect_tx(bar, kStageBytes);
  tma_load_3d(dst, &P.req[U.req].tm_ck, 0, U.kvh, U.tile * kTB, bar);
}

// q rows of a unit -> digit slices (all 16 warps, three rows each; every
// row's load is in flight before the first reduction)
__device__ void stage_q(const Route3Launch& P, const UnitInfo& U, uint8_t* smem, Misc& m) {
  const Route3Req& R = P.req[U.req];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kPer = (kN + kWarps - 1) / kWarps;
  float4 v[kPer];
#pragma unroll
  for (int z = 0; z < kPer; ++z) {
    const int j = warp + z * kWarps;
    v[z] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < U.nrows) {
      const int row = U.r0 + j, slot = row / P.G, h = U.kvh * P.G + row % P.G;
      v[z] = __ldg(reinterpret_cast<const float4*>(R.q + ((int64_t)R.slot_q[slot] * P.Hq + h) * kDh) + lane);
    }
  }
#pragma unroll
  for (int z = 0; z < kPer; ++z) {
    const int j = warp + z * kWarps;
    if (j >= kN) break;
    const float mx = warp_max_f(fmaxf(fmaxf(fabsf(v[z].x), fabsf(v[z].y)), fmaxf(fabsf(v[z].z), fabsf(v[z].w))));
    int e = 0;
    frexpf(mx, &e);  // mx < 2^e
    write_digit_row(smem + kOffQs, kQsSlice, j, lane, v[z], e);
    if (lane == 0) {
      m.qexp[j] = e;
      m.qmax[j] = mx;
    }
  }
}

// the staged fp32 key tile -> digit slices (8 rows per warp)
__device__ void slice_keys(const float* st, uint8_t* smem, Misc& m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 2
  for (int r = warp; r < kTB; r += kWarps) {
    const float4 v = reinterpret_cast<const float4*>(st + r * kDh)[lane];
    const float mx = warp_max_f(fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    int e = 0;
    frexpf(mx, &e);
    write_digit_row(smem + kOffKs, kKsSlice, r, lane, v, e);
    if (lane == 0) {
      m.kexp[r] = e;
      m.kmax[r] = mx;
    }
  }
}

// ------------------------------------------------------------------ Top-n
// (score desc, id asc): true when (sa, ia) ranks before (sb, ib)
__device__ __forceinline__ bool ranks_before(double sa, int ia, double sb, int ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// select_blocks (nsa_attention.cpp:94-136) over sel[0, avail): forced blocks,
// then the `want` best others into m.picks.  Also records the last pick's
// score (m.sk) and the best non-pick's (m.sk1, -inf if none) and sets
// m.certified = the two are separated by more than eps (relative).
__device__ void select_topn(const double* sel, int* surv, int avail, int n, double eps, Misc& m) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int f1 = avail - 2 > 0 ? avail - 2 : -1;
  const int f2 = avail - 1 > 0 ? avail - 1 : -1;
  const int nforced = avail > 0 ? 1 + (f1 > 0) + (f2 > 0 && f2 != f1) : 0;
  const int target = n < avail ? n : avail;
  const int want = target - nforced;
  const int ncand = avail - nforced;
  auto cand = [&](int b, double& sc) {
    const bool ok = b < avail && b != 0 && b != f1 && b != f2;
    sc = ok ? sel[b] : -INFINITY;
    return ok;
  };
  if (tid == 0) {
    m.nsurv = 0;
    m.lb_s = -INFINITY;
    m.lb_i = 0x7fffffff;
    m.sk = INFINITY;
    m.sk1 = -INFINITY;
  }
  __syncthreads();
  if (want > 0) {
    double bs = -INFINITY;  // 1. best of each 4-lane group
    int bi = 0x7fffffff;
    for (int b = tid; b < avail; b += kThreads) {
      double sc;
      if (cand(b, sc) && ranks_before(sc, b, bs, bi)) {
        bs = sc;
        bi = b;
      }
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ranks_before(os, oi, bs, bi)) {
        bs = os;
        bi = oi;
      }
    }
    if ((lane & 3) == 0) {
      m.gbest_s[tid >> 2] = bs;
      m.gbest_i[tid >> 2] = bi;
    }
    __syncthreads();
    {  // 2. the group maximum of rank want-1: a lower bound of the want-th best
      const int g = tid >> 2, part = tid & 3;
      const double ms = m.gbest_s[g];
      const int mi = m.gbest_i[g];
      int rank = 0;
      for (int o = part; o < kTopnGroups; o += 4)
        rank += ranks_before(m.gbest_s[o], m.gbest_i[o], ms, mi) ? 1 : 0;
      rank += __shfl_xor_sync(0xffffffffu, rank, 1);
      rank += __shfl_xor_sync(0xffffffffu, rank, 2);
      if (part == 0 && want <= kTopnGroups && rank == want - 1 && ms != -INFINITY) {
        m.lb_s = ms;
        m.lb_i = mi;
      }
    }
    __syncthreads();
    const double ls = m.lb_s;  // 3. survivors: a prefix of the global order
    const int li = m.lb_i;
    for (int b = tid; b < avail; b += kThreads) {
      double sc;
      if (cand(b, sc) && (ranks_before(sc, b, ls, li) || (sc == ls && b == li))) surv[atomicAdd(&m.nsurv, 1)] = b;
    }
    __syncthreads();
    const int ns = m.nsurv;  // 4. exact ranks among the survivors
    for (int k = tid; k < ns; k += kThreads) {
      const int b = surv[k];
      const double sb = sel[b];
      int rank = 0;
      for (int o = 0; o < ns; ++o) {
        const int c = surv[o];
        rank += ranks_before(sel[c], c, sb, b) ? 1 : 0;
      }
      if (rank < want) m.picks[nforced + rank] = b;
      if (rank == want - 1) m.sk = sb;
      if (rank == want) m.sk1 = sb;
    }
    __syncthreads();
    if (ns <= want && ncand > want) {  // 5. the best non-survivor is the best non-pick
      double bo = -INFINITY;
      for (int b = tid; b < avail; b += kThreads) {
        double sc;
        if (cand(b, sc) && !(ranks_before(sc, b, ls, li) || (sc == ls && b == li))) bo = fmax(bo, sc);
      }
      bo = warp_max_d(bo);
      if (lane == 0) m.red_w[warp] = bo;
      __syncthreads();
      if (tid == 0) {
        double v = -INFINITY;
        for (int w = 0; w < kWarps; ++w) v = fmax(v, m.red_w[w]);
        m.sk1 = v;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    const double a = m.sk, b = m.sk1;
    m.certified = (want <= 0 || ncand <= want || b == -INFINITY || (a - b) > eps * (a + b)) ? 1 : 0;
  }
  __syncthreads();
}

// the selected row, ascending (a rank-and-scatter over distinct block ids)
__device__ void write_row(const Misc& cm, Misc& m, int avail, int n, int32_t* idx_row, int32_t* count,
                          uint32_t* forced_bits) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid >= 32) return;
  const int f1 = avail - 2 > 0 ? avail - 2 : -1;
  const int f2 = avail - 1 > 0 ? avail - 1 : -1;
  const int cnt = (n < avail ? n : avail) > 0 ? (n < avail ? n : avail) : 0;
  if (lane == 0) {
    m.fbits = 0u;
    if (avail > 0) {
      int c = 0;
      m.picks[c++] = 0;
      if (f1 > 0) m.picks[c++] = f1;
      if (f2 > 0 && f2 != f1) m.picks[c++] = f2;
    }
  }
  __syncwarp();
  for (int a = lane; a < cnt; a += 32) {
    const int v = cm.picks[a];
    int rank = 0;
    for (int o = 0; o < cnt; ++o) rank += cm.picks[o] < v ? 1 : 0;
    idx_row[rank] = v;
    if ((v == 0 || v == f1 || v == f2) && rank < 32) atomicOr(&m.fbits, 1u << rank);
  }
  for (int a = cnt + lane; a < n; a += 32) idx_row[a] = -1;
  __syncwarp();
  if (lane == 0) {
    *count = cnt;
    *forced_bits = m.fbits;
  }
}

// ------------------------------------------------------------------ exact path
// fp64 scores of one slot, the reference's arithmetic (nsa_attention.cpp:38-80)
// regrouped: per KV head, up to four of its q heads at a time, a pass for the
// softmax maximum and denominator, then per selection block the overlapping
// blocks' probabilities.  One CTA; only for queries the certified path cannot
// decide (or forced by tests).
__device__ void exact_scores(const Route3Launch& P, const Route3Req& R, int slot, double* sel,
                             double* qrows, Misc& m) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qi = R.slot_q[slot], mv = R.slot_mvis[slot], avail = R.slot_avail[slot];
  const int G = P.G, Hkv = P.Hkv;
  const double inv = 1.0 / ((double)P.Hq * (double)P.l);
  for (int b = tid; b < avail; b += kThreads) sel[b] = 0.0;
  for (int kvh = 0; kvh < Hkv; ++kvh) {
    for (int g0 = 0; g0 < G; g0 += 4) {
      const int ng = min(4, G - g0);
      __syncthreads();
      for (int e = tid; e < ng * kDh; e += kThreads)
        qrows[e] = (double)R.q[((int64_t)qi * P.Hq + kvh * G + g0 + e / kDh) * kDh + e % kDh];
      __syncthreads();
      auto logits = [&](int i, double (&l)[4]) {
        const float4* kr = reinterpret_cast<const float4*>(R.ck + ((int64_t)i * Hkv + kvh) * kDh);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int x4 = 0; x4 < kDh / 4; ++x4) {
          const float4 k4 = __ldg(kr + x4);
          const double kx[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int gg = 0; gg < 4; ++gg)
              if (gg < ng) acc[gg] = fma(qrows[gg * kDh + 4 * x4 + c], kx[c], acc[gg]);
        }
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) l[gg] = acc[gg] * P.scale;
      };
      double mx[4], sm[4];
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        mx[gg] = -INFINITY;
        sm[gg] = 0.0;
      }
      for (int i = tid; i < mv; i += kThreads) {  // pass 1: running (max, sum) per head
        double l[4];
        logits(i, l);
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
          if (l[gg] > mx[gg]) {
            sm[gg] = sm[gg] * exp_nonpos(mx[gg] - l[gg]) + 1.0;
            mx[gg] = l[gg];
          } else {
            sm[gg] += exp_nonpos(l[gg] - mx[gg]);
          }
        }
      }
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {  // fixed-order reduction: xor tree, then warps in order
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const double om = __shfl_xor_sync(0xffffffffu, mx[gg], o);
          const double os = __shfl_xor_sync(0xffffffffu, sm[gg], o);
          const double M = fmax(mx[gg], om);
          sm[gg] = (M == -INFINITY) ? 0.0 : sm[gg] * exp_nonpos(mx[gg] - M) + os * exp_nonpos(om - M);
          mx[gg] = M;
        }
        if (lane == 0) {
          m.red_m[warp][gg] = mx[gg];
          m.red_s[warp][gg] = sm[gg];
        }
      }
      __syncthreads();
      if (tid < 4) {
        double M = -INFINITY, S = 0.0;
        for (int w = 0; w < kWarps; ++w) {
          const double wm = m.red_m[w][tid], ws = m.red_s[w][tid];
          const double nm = fmax(M, wm);
          S = (nm == -INFINITY) ? 0.0 : S * exp_nonpos(M - nm) + ws * exp_nonpos(wm - nm);
          M = nm;
        }
        m.fin_m[tid] = M;
        m.fin_s[tid] = S;
      }
      __syncthreads();
      for (int b = tid; b < avail; b += kThreads) {  // pass 2: per selection block
        int lo, hi;
        blocks_of(b, P.d, P.l, P.l_sel, lo, hi);
        hi = min(hi, mv - 1);
        double s = 0.0;
        for (int i = lo; i <= hi; ++i) {
          double l[4];
          logits(i, l);
          const double w = (double)overlap(i, b, P.d, P.l, P.l_sel);
#pragma unroll
          for (int gg = 0; gg < 4; ++gg)
            if (gg < ng && m.fin_s[gg] > 0.0) s += exp_nonpos(l[gg] - m.fin_m[gg]) / m.fin_s[gg] * w;
        }
        sel[b] += s * inv;
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ kernel
__device__ __forceinline__ void stamp(const Route3Launch& P, int k) {
  if (P.trace != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.trace[kRouteTraceBase + blockIdx.x * 16 + k] = t;
  }
}

__global__ void __launch_bounds__(kThreads, 1) route3_kernel(const __grid_constant__ Route3Launch P) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  Misc& m = *reinterpret_cast<Misc*>(smem + kOffMisc);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x, nctas = gridDim.x;
  int* bar = P.counters;
  griddep_wait();  // inputs (q) may come from the launch just before (PDL)
  stamp(P, 0);
  const int units = P.unit_start[P.n_req];
  if (tid == 0) {
    mbar_init(&m.tma_full[0], 1);
    mbar_init(&m.tma_full[1], 1);
    mbar_init(&m.mma_done, 1);
    fence_mbar_init();
    for (int k = 0; k < 2 && cta + k * nctas < units; ++k)
      issue_unit_tma(P, cta + k * nctas, smem + kOffStage + k * kStageBytes, &m.tma_full[k]);
  }
  if (cta == nctas - 1) {  // queries that reuse a representative's set get count -1
    for (int r = 0; r < P.n_req; ++r) {
      const Route3Req& R = P.req[r];
      for (int e = tid; e < R.n_unrouted * (P.n + 1); e += kThreads) {
        const int qq = R.unrouted[e / (P.n + 1)], a = e % (P.n + 1);
        if (a == P.n) {
          R.idx_count[qq] = -1;
          R.idx_forced[qq] = 0u;
        } else {
          R.idx[(int64_t)qq * P.n + a] = -1;
        }
      }
    }
  }
  if (warp == 0 && cta < units) tmem_alloc<kTmemCols>(&m.tmem_base);
  __syncthreads();
  tc_fence_after();

  // ================= phase A: units (logits, tile statistics, G) =================
  int staged = -1;  // (request, KV head, chunk) whose q digits are in shared memory
  int k = 0;
  for (int u = cta; u < units; u += nctas, ++k) {
    const UnitInfo U = unit_info(P, u);
    const Route3Req& R = P.req[U.req];
    const int qkey = (U.req * 128 + U.chunk) * 128 + U.kvh;
    if (qkey != staged) {
      stage_q(P, U, smem, m);
      staged = qkey;
    }
    if (k < 2) stamp(P, 6 + 5 * k);
    const int sb = k & 1;
    mbar_wait(&m.tma_full[sb], (k >> 1) & 1);
    if (k < 2) stamp(P, 7 + 5 * k);
    slice_keys(reinterpret_cast<const float*>(smem + kOffStage + sb * kStageBytes), smem, m);
    fence_proxy_async_smem();
    __syncthreads();
    if (k < 2) stamp(P, 8 + 5 * k);
    if (tid == 0 && u + 2 * nctas < units)  // the stage is free: prefetch two units ahead
      issue_unit_tma(P, u + 2 * nctas, smem + kOffStage + sb * kStageBytes, &m.tma_full[sb]);
    if (warp == 0) {
      tc_fence_after();
      constexpr uint32_t idesc = idesc_s8(kTB, kN);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            if (s + t < 2) continue;
            const int cls = s + t - 2;
            const bool first = kk == 0 && s == (s + t - 3 > 0 ? s + t - 3 : 0);
            umma_i8_warp(m.tmem_base + cls * kN,
                         desc_sw128(sbase + kOffKs + t * kKsSlice + 32 * kk, 16, 1024),
                         desc_sw128(sbase + kOffQs + s * kQsSlice + 32 * kk, 16, 1024), idesc,
                         first ? 0u : 1u);
          }
      umma_commit_warp(&m.mma_done);
    }
    __syncwarp();
    mbar_wait(&m.mma_done, k & 1);
    tc_fence_after();
    if (k < 2) stamp(P, 9 + 5 * k);
    double* L = reinterpret_cast<double*>(smem + kOffKs);  // [kN][kTB] log2-unit logits (aliases the digits)
    if (warp < 12) {
      const int qd = warp & 3, cg = warp >> 2;
      const int i = 32 * qd + lane;
      uint32_t a[kAcc][16];
#pragma unroll
      for (int c = 0; c < kAcc; ++c)
        tmem_ld16(m.tmem_base + (static_cast<uint32_t>(32 * qd) << 16) + c * kN + 16 * cg, a[c]);
      tmem_wait_ld();
      const int gblk = U.tile * kTB + i;
      const int ke = m.kexp[i];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int j = 16 * cg + jj;
        double val = -INFINITY;
        if (j < U.nrows && gblk < R.slot_mvis[(U.r0 + j) / P.G]) {
          long long h = (int)a[4][jj];
          h = h * 256 + (int)a[3][jj];
          h = h * 256 + (int)a[2][jj];
          h = h * 256 + (int)a[1][jj];
          h = h * 256 + (int)a[0][jj];
          val = (double)h * pow2i(m.qexp[j] + ke - 44) * P.c_sl;
        }
        L[j * kTB + i] = val;
      }
    }
    tc_fence_before();
    __syncthreads();
    if (k < 2) stamp(P, 10 + 5 * k);
    // per row: tile max, e = 2^(logit - max), tile sum, selection-block sums
    {
      float akm = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) akm = fmaxf(akm, m.kmax[4 * lane + c]);
      akm = warp_max_f(akm);
      const int rows_head = R.nr * P.G;
      double* gsh = R.gsh + unit_gsh_offset(P, U, u);
      for (int j = warp; j < U.nrows; j += kWarps) {
        double* Lj = L + j * kTB;
        double v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = Lj[lane + 32 * c];
        const double mx = warp_max_d(fmax(fmax(v[0], v[1]), fmax(v[2], v[3])));
        double td = 0.0;
        if (mx != -INFINITY) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double e = v[c] == -INFINITY ? 0.0 : exp2_nonpos(v[c] - mx);
            Lj[lane + 32 * c] = e;
            td += e;
          }
        }
        td = warp_sum_d(td);
        __syncwarp();
        const int b0 = U.tile * P.spt;
        for (int bl = lane; bl < P.span; bl += 32) {
          double g = 0.0;
          if (mx != -INFINITY) {
            int lo, hi;
            blocks_of(b0 + bl, P.d, P.l, P.l_sel, lo, hi);
            lo = max(lo, U.tile * kTB);
            hi = min(hi, U.tile * kTB + kTB - 1);
            for (int i = lo; i <= hi; ++i)
              g += (double)overlap(i, b0 + bl, P.d, P.l, P.l_sel) * Lj[i - U.tile * kTB];
          }
          gsh[j * P.span + bl] = g;
        }
        if (lane == 0) {
          double* st = R.stats + ((int64_t)(U.kvh * rows_head + U.r0 + j) * R.ntiles + U.tile) * 4;
          st[0] = mx;
          st[1] = td;
          // logit error bound (log2 units): grid rounding + dropped digit pairs
          // <= 2^-21.9 |q|max |k|max, with a factor-2 margin
          st[2] = P.c_sl * (double)m.qmax[j] * (double)akm * 4.76837158203125e-07;  // 2^-21
        }
      }
    }
    __syncthreads();  // L / digits / staging reuse by the next unit
  }
  if (warp == 0 && cta < units) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(m.tmem_base);
  }
  stamp(P, 1);

  // ================= grid barrier: every tile statistic is out =================
  __syncthreads();
  if (tid == 0) {
    red_add_release_gpu(bar + 0, 1);
    while (ld_acquire_gpu(bar + 0) < nctas) {
    }
  }
  __syncthreads();
  stamp(P, 2);

  // ================= phase C: normalise, fold GQA heads, per-KV-head shares =================
  for (int u = cta; u < units; u += nctas) {
    const UnitInfo U = unit_info(P, u);
    const Route3Req& R = P.req[U.req];
    const int rows_head = R.nr * P.G;
    for (int j = warp; j < U.nrows; j += kWarps) {
      // every tile's statistics of the row in registers (one L2 round trip)
      const double* sj = R.stats + (int64_t)(U.kvh * rows_head + U.r0 + j) * R.ntiles * 4;
      constexpr int kTpl = 8;  // tiles per lane: ntiles <= 256 (kMaxAvail selection blocks)
      double m2v[kTpl], tdv[kTpl];
      double mx = -INFINITY, bmax = 0.0;
#pragma unroll
      for (int z = 0; z < kTpl; ++z) {
        const int t = lane + 32 * z;
        m2v[z] = -INFINITY;
        tdv[z] = 0.0;
        if (t < R.ntiles) {
          const double2 a = __ldcg(reinterpret_cast<const double2*>(sj) + 2 * t);
          const double2 c = __ldcg(reinterpret_cast<const double2*>(sj) + 2 * t + 1);
          m2v[z] = a.x;
          tdv[z] = a.y;
          bmax = fmax(bmax, c.x);
        }
        mx = fmax(mx, m2v[z]);
      }
      mx = warp_max_d(mx);
      bmax = warp_max_d(bmax);
      double den = 0.0;
      if (mx != -INFINITY)
#pragma unroll
        for (int z = 0; z < kTpl; ++z)
          if (m2v[z] != -INFINITY) den += tdv[z] * exp2_nonpos(m2v[z] - mx);
      den = warp_sum_d(den);
      if (lane == (U.tile & 31)) {
        double ownv = -INFINITY;
#pragma unroll
        for (int z = 0; z < kTpl; ++z)
          if (z == (U.tile >> 5)) ownv = m2v[z];
        m.F[j] = (ownv == -INFINITY || !(den > 0.0)) ? 0.0 : exp2_nonpos(ownv - mx) / den;
        m.E[j] = bmax;
      }
    }
    __syncthreads();
    const int s0 = U.r0 / P.G, ns = U.nrows / P.G;
    const double* gsh = R.gsh + unit_gsh_offset(P, U, u);
    for (int e = tid; e < ns * P.span; e += kThreads) {
      const int sl = e / P.span, bl = e % P.span;
      double c = 0.0;
      for (int g = 0; g < P.G; ++g) c += m.F[sl * P.G + g] * gsh[(sl * P.G + g) * P.span + bl];
      R.contrib[(((int64_t)(s0 + sl) * P.Hkv + U.kvh) * R.ntiles + U.tile) * P.span + bl] = c;
    }
    if (U.tile == 0)
      for (int sl = tid; sl < ns; sl += kThreads) {
        double e = 0.0;
        for (int g = 0; g < P.G; ++g) e = fmax(e, m.E[sl * P.G + g]);
        R.eps[(int64_t)(s0 + sl) * P.Hkv + U.kvh] = e;
      }
    __syncthreads();
  }
  stamp(P, 3);

  // ================= Top-n tasks after every share is out =================
  const int tasks = P.task_start[P.n_req];
  __syncthreads();
  if (tid == 0) red_add_release_gpu(bar + 1, 1);
  griddep_launch();  // the next launch may start placing CTAs as this grid drains
  if (cta < tasks) {
    if (tid == 0)
      while (ld_acquire_gpu(bar + 1) < nctas) {
      }
    __syncthreads();
    stamp(P, 4);
    double* sel = reinterpret_cast<double*>(smem + kOffStage);                // [kMaxAvail]
    int* surv = reinterpret_cast<int*>(smem + kOffStage + 8 * kMaxAvail);    // [kMaxAvail]
    double* qrows = reinterpret_cast<double*>(smem + kOffStage + 12 * kMaxAvail);  // [4][128]
    for (int t = cta; t < tasks; t += nctas) {
      int r = 0;
      while (r + 1 < P.n_req && t >= P.task_start[r + 1]) ++r;
      const Route3Req& R = P.req[r];
      const int slot = t - P.task_start[r];
      const int avail = R.slot_avail[slot];
      const double inv = 1.0 / ((double)P.Hq * (double)P.l);
      const double* cb = R.contrib + (int64_t)slot * P.Hkv * R.ntiles * P.span;
      for (int b = tid; b < avail; b += kThreads) {
        const int t_hi = min(R.ntiles - 1, b / P.spt);
        const int t_lo = max(0, (b - P.span + P.spt) / P.spt);
        double v[8][2];  // every share of the block in flight at once
#pragma unroll
        for (int kvh = 0; kvh < 8; ++kvh)
#pragma unroll
          for (int z = 0; z < 2; ++z) {
            const int tt = t_lo + z;
            v[kvh][z] = (kvh < P.Hkv && tt <= t_hi)
                            ? __ldcg(cb + ((int64_t)kvh * R.ntiles + tt) * P.span + (b - tt * P.spt))
                            : 0.0;
          }
        double s = 0.0;  // KV heads ascending, tiles ascending
#pragma unroll
        for (int kvh = 0; kvh < 8; ++kvh) {
          if (kvh >= P.Hkv) break;
          s += v[kvh][0];
          s += v[kvh][1];
          for (int tt = t_lo + 2; tt <= t_hi; ++tt)
            s += __ldcg(cb + ((int64_t)kvh * R.ntiles + tt) * P.span + (b - tt * P.spt));
        }
        for (int kvh = 8; kvh < P.Hkv; ++kvh)
          for (int tt = t_lo; tt <= t_hi; ++tt)
            s += __ldcg(cb + ((int64_t)kvh * R.ntiles + tt) * P.span + (b - tt * P.spt));
        sel[b] = s * inv;
      }
      double dl = 0.0;
      if (tid < P.Hkv && R.ntiles > 0) dl = __ldcg(R.eps + (int64_t)slot * P.Hkv + tid);
      dl = warp_max_d(dl);
      if (tid == 0) m.red_w[0] = dl;
      __syncthreads();
      // relative score error <= 2 ln2 delta (+ fp64 rounding), with margin
      const double eps = 1.5 * 2.0 * 0.6931471805599453 * m.red_w[0] + 1e-12;
      select_topn(sel, surv, avail, P.n, eps, m);
      if (!m.certified || P.force_exact) {
        if (tid == 0 && P.fallbacks != nullptr) atomicAdd(P.fallbacks, 1);
        exact_scores(P, R, slot, sel, qrows, m);
        select_topn(sel, surv, avail, P.n, 0.0, m);
      }
      const int q = R.slot_q[slot];
      write_row(m, m, avail, P.n, R.idx + (int64_t)q * P.n, R.idx_count + q, R.idx_forced + q);
      __syncthreads();
    }
  }
  stamp(P, 5);
  __syncthreads();
  if (tid == 0 && atom_add_acq_rel_gpu(bar + 2, 1) == nctas - 1) {  // the last CTA out resets
    atomicExch(bar + 0, 0);
    atomicExch(bar + 1, 0);
    atomicExch(bar + 2, 0);
  }
}

int sm_count3() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& slot = cache[dev < 64 ? dev : 63];
  int sms = slot.load(std::memory_order_relaxed);
  if (sms == 0) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev < 64) slot.store(sms, std::memory_order_relaxed);
  }
  return sms;
}

}  // namespace

cudaError_t launch_route3(Route3Launch& p, cudaStream_t s) {
  p.unit_start[0] = 0;
  p.task_start[0] = 0;
  for (int r = 0; r < p.n_req; ++r) {
    const Route3Req& R = p.req[r];
    p.unit_start[r + 1] = p.unit_start[r] + p.Hkv * R.nchunks * R.ntiles;
    p.task_start[r + 1] = p.task_start[r] + R.nr;
  }
  const int work = std::max(p.unit_start[p.n_req], p.task_start[p.n_req]);
  const int ctas = std::max(1, std::min(sm_count3(), work));
  cudaError_t e = cudaFuncSetAttribute(route3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeCooperative;  // grid barriers: every CTA co-resident
  attr[na++].val.cooperative = 1;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, route3_kernel, p);
}

}  // namespace specsv_b200
