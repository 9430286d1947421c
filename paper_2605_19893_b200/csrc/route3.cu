// route3.cu -- refresh-layer routing on sm_100a's integer tensor pipe:
// compressed-block selection scores and Top-n with forced blocks, for up to
// kR3Batch requests in one cooperative launch.
//
// Replaces nsa::selection_scores + nsa::select_blocks
// (src/nsa_attention.cpp:38-136) for every query that constructs indices.
//
// Work unit = (request, row chunk, KV head, range of <= 64 selection blocks):
// one CTA, the range's <= 256 compressed blocks streamed ONCE by TMA as key
// digit planes written at compression time (compress.cu), all of the chunk's
// (slot, GQA head) rows multiplied against them.  At the bench shape (64K,
// 9 routed queries, 8 KV heads) that is 8 heads x 18 ranges = 144 units, one
// per SM.
//
// Logits.  The reference forms logit = dot(q_h, ck_i) / sqrt(dh) in double
// from fp32 operands (nsa_attention.cpp:51-56).  Here every q row and key row
// is a 31-bit fixed-point integer on its own power-of-two grid
// (X = round(x 2^(30 - e)), max |x| < 2^e) split into four signed base-256
// digits; the 13 digit pairs of weight >= 256^2 are exact s8 x s8 -> s32
// tcgen05 MMAs (kind::i8, M = 128 blocks, N = 48 rows, K = 128) summed per
// weight class in TMEM and recombined in int64.  The logit differs from the
// exact fp32-operand dot by < 2^(eq + ek - 22.98) (grid rounding plus the
// three dropped low pairs).
//
// Scores without a max pass.  p_hi = e_hi / DEN_h with e = 2^(logit log2 e)
// taken against the fixed reference 0 in fp64 (logits beyond +-960 log2
// units send the query to the exact path), so a range's sums are additive
// across ranges: per row j the range computes the selection-block sums
// g_jb = sum_i overlap(i, b) e_ij and its share of the denominator
// den_j = sum_b g_jb (every visible block's tokens sum to l over the
// selection blocks, so summing over all ranges gives l x DEN).  One exchange
// of the per-range den rows per (chunk, KV head), then every unit writes its
// KV head's normalised share contrib_b = sum_{g in G} g_(q,g),b / den_(q,g),
// and the Top-n task of each slot sums the KV heads in ascending order:
// score_b = sum_h sum_i p_hi overlap(i, b) / (l Hq) -- the reference's sum
// over heads and blocks of p * overlap / l / Hq (nsa_attention.cpp:57-78),
// regrouped (P3: <= 1e-13 relative).
//
// Certification.  A logit error bound delta (log2 units) makes every e exact
// to a factor 2^(+-delta), so every score is within a relative
// eps = 2 ln2 delta_max (x1.5 margin, plus 2e-10 for the fp64 exp and sums)
// of its exact value.  The Top-n (forced {0, avail-2, avail-1} plus the best
// by (score desc, id asc), nsa_attention.cpp:94-136) is accepted when the last
// pick and the best non-pick are separated by more than eps; otherwise the
// task re-scores its query exactly in fp64 (the reference's arithmetic,
// regrouped) and selects on those scores.  The indices therefore equal the
// reference's whatever the inputs; the re-scoring path is exercised by tests
// (force_exact).
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
constexpr int kDh = 128;
constexpr int kN = kR3Rows;   // rows per unit (MMA N)
constexpr int kTB = kR3Tile;  // compressed blocks per MMA tile
constexpr int kAcc = 5;       // digit-pair weight classes 256^2 .. 256^6
constexpr int kWarpMma = 12;
constexpr uint32_t kTmemCols = 512;  // 2 tiles x 5 classes x 48 columns
constexpr int kTopnGroups = kThreads / 4;
constexpr uint32_t kExStage = 32768;  // exact path: bytes per key stage (whole blocks, all KV heads)
constexpr int kMaxHq = 128;           // q heads (build limit)
constexpr uint32_t kExQOff = 3 * kExStage;  // exact path: fp64 q of every head, after three stages
constexpr int kExQS = kDh + 4;               // its row stride in doubles (KV heads' rows on other banks)
static_assert(kN == 4 * 12, "epilogue: 4 TMEM lane quadrants x 4 column groups of 12 (16 warps)");
static_assert(kR3MaxSpr == 64, "two selection blocks per lane in the row sums");

// counter words of one request (Route3Req::cnt)
constexpr int kCntDen = 0;     // [nchunks x Hkv] arrivals of a (chunk, KV head)'s ranges
constexpr int kCntTop = 272;   // [nchunks] arrivals of a chunk's units after their shares
constexpr int kCntBound = 352;  // [nr] 64-bit: the slot's logit error bound (log2 units, fp64 bits;
                                //      +inf: exact path), max over its rows and units
constexpr int kCntLock = 496;   // the exact path's scratch lock
static_assert(kCntBound + 2 * kMaxQueries <= kCntLock && kCntLock < kR3CntPerReq, "counter set");
constexpr unsigned long long kBoundFlag = 0x7FF0000000000000ULL;  // +inf

// shared memory map (bytes from the 1024-aligned base)
constexpr uint32_t kPlaneBytes = kTB * 128;                // one digit plane of one tile (SW128)
constexpr uint32_t kTileBytes = 4 * kPlaneBytes;           // 64 KB; then the tile's e values [48][128] fp64
constexpr uint32_t kOffQs = 2 * kTileBytes;                // q digits [4][48 rows x 128 B], SW128
constexpr uint32_t kQsSlice = kN * 128;                    // 6144
constexpr int kES = 64;  // e values: [256 rows][64] fp64 over both tiles' plane regions, column
                         // j stored at j ^ (row & 15) (conflict-free row stores and column reads)
constexpr int kGS = kN + 1;                                // selection-block sums: [64][kGS] fp64
constexpr uint32_t kOffG = kOffQs + 4 * kQsSlice;          // g [kR3MaxSpr][kGS] fp64
constexpr uint32_t kOffMisc = kOffG + kR3MaxSpr * kGS * 8;
static_assert(kTB * kES * 8 == kTileBytes, "e values: tile t's rows alias tile t's planes");
static_assert(kQsSlice % 1024 == 0, "SW128 atoms");
static_assert((size_t)kMaxAvail * 12 + 4 * kDh * 8 + 66 * 4 <= 2 * kTileBytes, "Top-n arrays alias the planes");
static_assert((size_t)kMaxAvail * 12 + 2048 * 8 <= 2 * kTileBytes, "survivor scores after sel and surv");

struct Misc {
  uint64_t tma_full[2], mma_done[2], ex_full[3];
  uint32_t tmem_base;
  int32_t flag, kemax, nkmax;
  int32_t qexp[kN];
  int32_t qinex[kN];    // q elements the grid rounds, per row
  int32_t colmvis[kN];  // visible compressed blocks of the column's slot (0: no column)
  double qsc[kN];       // c_sl 2^(qe - 44): logit (log2 units) per unit of h 2^ke
  double invD[kN];
  int32_t kexp[kR3MaxBlk];  // row exponents of the unit's blocks
  double T16[16];       // 2^(k/16)
  int32_t glo[kR3MaxSpr];                 // first compressed block overlapping each selection block
  double gw[kR3MaxBps][kR3MaxSpr];        // its blocks' token overlaps (0 past the last one)
  // Top-n / exact path
  double red_m[kWarps][4], red_s[kWarps][4];
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


// 2^(k/16), k = 0..15, correctly rounded
__constant__ double kT16[16] = {1.0, 1.0442737824274138, 1.0905077326652577, 1.1387886347566916,
                                1.189207115002721, 1.241857812073484, 1.2968395546510096, 1.3542555469368927,
                                1.4142135623730951, 1.4768261459394993, 1.5422108254079407, 1.6104903319492543,
                                1.681792830507429, 1.7562521603732995, 1.8340080864093424, 1.9152065613971474};

// 2^L for |L| < 512 in fp64 (relative error < 5e-11, inside the 2e-10 term of
// the certification bound): 16 L rounded to an integer k16 by the
// 1.5 2^52 shifter, 2^(k16 / 16) from the table and the exponent field,
// 2^r (|r| <= 1/32) by a degree-4 polynomial in r
__device__ __forceinline__ double exp2_fast(double L, const double* T16) {
  const double kShift = 6755399441055744.0;  // 1.5 x 2^52
  const double t = fma(L, 16.0, kShift);
  const double k16 = t - kShift;
  const int ki = __double2loint(t);
  const double r = fma(k16, -0.0625, L);
  double p = 9.6181291076284772e-03;        // ln2^4 / 4!
  p = fma(p, r, 5.5504108664821580e-02);
  p = fma(p, r, 2.4022650695910071e-01);
  p = fma(p, r, 6.9314718055994531e-01);
  p = fma(p, r, 1.0);
  const double v = p * T16[ki & 15];
  return __hiloint2double(__double2hiint(v) + ((ki >> 4) << 20), __double2loint(v));
}

// int32 -> double on the fp64 pipe (no conversion unit): 2^52 + 2^31 + x, minus the bias
__device__ __forceinline__ double i2d(int x) {
  return __hiloint2double(0x43300000, x ^ 0x80000000) - 4503601774854144.0;
}
// int64 with |x| < 2^51 -> double: 1.5 2^52 + x, minus the bias
__device__ __forceinline__ double l2d(long long x) {
  return __longlong_as_double(x + 0x4338000000000000LL) - 6755399441055744.0;
}
// x 2^k for x = 0 or a normal x whose result stays normal (the exponent field)
__device__ __forceinline__ double scale2(double x, int k) {
  const int hi = __double2hiint(x);
  return __hiloint2double((hi & 0x7ff00000) ? hi + (k << 20) : hi, __double2loint(x));
}

struct Unit {
  int req, lu, chunk, kvh, range;
  int s0, nslots, nrows;  // slots [s0, s0 + nslots) of the chunk; rows = nslots x G
  int b0, b1;             // selection blocks [b0, b1)
  int row0, nblk;         // compressed blocks [row0, row0 + nblk)
};

template <class LaunchT>
__device__ __forceinline__ Unit unit_of(const LaunchT& P, int u) {
  int r = 0;
  while (r + 1 < P.n_req && u >= P.unit_start[r + 1]) ++r;
  const Route3Req& R = P.req[r];
  Unit U;
  U.req = r;
  U.lu = u - P.unit_start[r];
  int x = U.lu;
  U.range = x % R.nranges;
  x /= R.nranges;
  U.kvh = x % P.Hkv;
  U.chunk = x / P.Hkv;
  U.s0 = U.chunk * P.spc;
  U.nslots = min(P.spc, R.nr - U.s0);
  U.nrows = U.nslots * P.G;
  U.b0 = U.range * R.spr;
  U.b1 = min(U.b0 + R.spr, R.avail_max);
  int lo, hi, lo1, hi1;
  blocks_of(U.b0, P.d, P.l, P.l_sel, lo, hi);
  blocks_of(max(U.b1 - 1, U.b0), P.d, P.l, P.l_sel, lo1, hi1);
  U.row0 = lo;
  U.nblk = U.b1 > U.b0 ? min(hi1, R.blocks - 1) - lo + 1 : 0;
  return U;
}

// the unit's q rows (16 warps, three rows each), loaded first so the loads are
// in flight across the rest of the unit's setup
template <class LaunchT>
__device__ __forceinline__ void load_q(const LaunchT& P, const Route3Req& R, const Unit& U, float4 (&v)[3]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int z = 0; z < 3; ++z) {
    const int j = warp + z * kWarps;
    v[z] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < U.nrows) {
      const int slot = U.s0 + j / P.G, h = U.kvh * P.G + j % P.G;
      v[z] = __ldg(reinterpret_cast<const float4*>(R.q + ((int64_t)R.slot_q[slot] * P.Hq + h) * kDh) + lane);
    }
  }
}

// ... -> digit slices, plus per-column tables
template <class LaunchT>
__device__ __forceinline__ void digit_q(const LaunchT& P, const Route3Req& R, const Unit& U,
                                        const float4 (&v)[3], uint8_t* smem, Misc& m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  static_assert(kN == 3 * kWarps, "three q rows per warp");
#pragma unroll
  for (int z = 0; z < 3; ++z) {
    const int j = warp + z * kWarps;
    const float mx = warp_max_f(fmaxf(fmaxf(fabsf(v[z].x), fabsf(v[z].y)), fmaxf(fabsf(v[z].z), fabsf(v[z].w))));
    int e = 0;
    if (mx > 0.f) frexpf(mx, &e);  // mx < 2^e
    write_digit_row(smem + kOffQs, kQsSlice, j, lane, v[z], e);
    int inex = 0;  // elements the 31-bit grid rounds (the rest it represents exactly)
    {
      const float xs[4] = {v[z].x, v[z].y, v[z].z, v[z].w};
      const int shift = 30 - e;
      const bool plain = shift >= -126 && shift <= 127;
      const float sc = plain ? __int_as_float((127 + shift) << 23) : 1.0f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float sx = plain ? xs[c] * sc : ldexpf(xs[c], shift);  // exact (a power of two)
        inex += (float)__float2int_rn(sx) != sx ? 1 : 0;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) inex += __shfl_xor_sync(0xffffffffu, inex, o);
    if (lane == 0) {
      m.qinex[j] = inex;
      m.qexp[j] = e;
      m.qsc[j] = P.c_sl * pow2i(e - 44);
      m.colmvis[j] = j < U.nrows ? R.slot_mvis[U.s0 + j / P.G] : 0;
    }
  }
}

// one unit's key digit planes -> the two tile stages (an empty second tile just arrives)
__device__ __forceinline__ void issue_unit_tma(const Route3Req& R, const Unit& U, uint8_t* smem, Misc& m) {
  const uint64_t pol = l2_evict_first_policy();  // the digit planes are read once per launch
  const int ntile = U.nblk > kTB ? 2 : 1;
  for (int t = 0; t < 2; ++t) {
    if (t < ntile) {
      mbar_expect_tx(&m.tma_full[t], kTileBytes);
#pragma unroll
      for (int s = 0; s < 4; ++s)
        tma_load_4d_hint(smem + t * kTileBytes + s * kPlaneBytes, &R.tm_ckd, 0, s, U.kvh, U.row0 + t * kTB,
                         &m.tma_full[t], pol);
    } else {
      mbar_arrive(&m.tma_full[t]);
    }
  }
}

template <class LaunchT>
__device__ __forceinline__ void stamp(const LaunchT& P, int k) {
#ifdef SPECSV_TRACE_TILES  // phase stamps: diagnostics build only (see attend.cu)
  if (P.trace != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.trace[kRouteTraceBase + blockIdx.x * 16 + k] = t;
  }
#endif
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
// GL lanes per group (2 candidates each at avail <= 2 x kThreads): groups of
// 16 lanes rank 32 group bests (2 comparisons per thread), groups of 8 rank
// 64 (8 comparisons; groups of 4: 128 bests, 32 comparisons).  The bound needs
// want < groups: want <= n - 1, so 16 lanes for n <= 32 and 8 lanes up to the
// build limit n <= 64 (check_build_limits).
// The survivors' scores are copied next to their ids (surv_s, up to
// kSurvCap), so the exact ranking reads two independent arrays instead of
// sel[surv[o]]; with COMPACT false it reads sel[surv[o]] (the earlier form).
constexpr int kSurvCap = 2048;
template <int GL, bool COMPACT>
__device__ void select_topn_impl(const double* sel, int* surv, double* surv_s, int avail, int n, double eps,
                                 Misc& m, unsigned long long* tr) {
  constexpr int kGroups = kThreads / GL;
  static_assert(kGroups <= kTopnGroups, "group bests");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long c0 = clock64();
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
    for (int off = 1; off < GL; off <<= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ranks_before(os, oi, bs, bi)) {
        bs = os;
        bi = oi;
      }
    }
    if ((lane & (GL - 1)) == 0) {
      m.gbest_s[tid / GL] = bs;
      m.gbest_i[tid / GL] = bi;
    }
    __syncthreads();
    {  // 2. the group maximum of rank `want`: at least want + 1 candidates rank at or
       //    before it, so the survivors hold the picks AND the best non-pick
      const int g = tid / GL, part = tid & (GL - 1);
      const double ms = m.gbest_s[g];
      const int mi = m.gbest_i[g];
      int rank = 0;
#pragma unroll
      for (int o = part; o < kGroups; o += GL)
        rank += ranks_before(m.gbest_s[o], m.gbest_i[o], ms, mi) ? 1 : 0;
#pragma unroll
      for (int off = 1; off < GL; off <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, off);
      if (part == 0 && want < kGroups && rank == want && ms != -INFINITY) {
        m.lb_s = ms;
        m.lb_i = mi;
      }
    }
    __syncthreads();
    if (tr != nullptr && tid == 0) tr[11] = clock64() - c0;
    const double ls = m.lb_s;  // 3. survivors: a prefix of the global order
    const int li = m.lb_i;
    for (int b = tid; b < avail; b += kThreads) {
      double sc;
      if (cand(b, sc) && (ranks_before(sc, b, ls, li) || (sc == ls && b == li))) {
        const int slot = atomicAdd(&m.nsurv, 1);
        surv[slot] = b;
        if (COMPACT && slot < kSurvCap) surv_s[slot] = sc;
      }
    }
    __syncthreads();
    const int ns = m.nsurv;  // 4. exact ranks among the survivors
    if (COMPACT && ns <= kSurvCap) {
      for (int k = tid; k < ns; k += kThreads) {
        const int b = surv[k];
        const double sb = surv_s[k];
        int rank = 0;
#pragma unroll 4
        for (int o = 0; o < ns; ++o) rank += ranks_before(surv_s[o], surv[o], sb, b) ? 1 : 0;
        if (rank < want) m.picks[nforced + rank] = b;
        if (rank == want - 1) m.sk = sb;
        if (rank == want) m.sk1 = sb;
      }
    } else {
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
    }
    __syncthreads();
    if (ns <= want && ncand > want) {  // 5. (a survivor set without a non-pick: the best non-survivor)
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

// route3 debug bit 5 (32): the earlier form (groups of 4 lanes, sel[surv[o]])
__device__ __forceinline__ void select_topn(const double* sel, int* surv, int avail, int n, double eps, Misc& m,
                                            int debug, unsigned long long* tr = nullptr) {
  double* surv_s = const_cast<double*>(sel) + 12 * kMaxAvail / 8;  // after sel and surv
  if (debug & 32)
    select_topn_impl<4, false>(sel, surv, surv_s, avail, n, eps, m, tr);
  else if (n <= 32)  // want <= n - 1 < 32 groups of 16 lanes
    select_topn_impl<16, true>(sel, surv, surv_s, avail, n, eps, m, tr);
  else  // want <= 63 < 64 groups of 8 lanes
    select_topn_impl<8, true>(sel, surv, surv_s, avail, n, eps, m, tr);
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
// regrouped, for queries the certified path cannot decide (or forced by
// tests).  One CTA: (1) every visible block's logit for every q head (fp32
// operands, fp64 products and sums) from the compressed keys streamed as
// contiguous 32 KB chunks (all KV heads of whole blocks) by bulk copies
// through kExStages shared-memory stages, stored once to the request's scratch
// [Hq][blocks] in L2, per-head running maxima; (2) e = exp(logit - max) stored
// back, denominators in a fixed order; (3) per selection block the overlapping
// blocks' probabilities.  The scratch is one per request: slots that fall
// back take it in turn (a spin lock; the path is rare).
constexpr int kExStages = 3;
__device__ __forceinline__ uint32_t ex_stage_off(int s) { return (uint32_t)s * kExStage; }  // over the idle sel/surv arrays

template <class LaunchT>
__device__ void exact_scores(const LaunchT& P, const Route3Req& R, int slot, double* sel, uint8_t* smem,
                             Misc& m, int& ex_seq) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qi = R.slot_q[slot], mv = R.slot_mvis[slot], avail = R.slot_avail[slot];
  const int Hq = P.Hq, Hkv = P.Hkv, G = P.G;
  const double inv = 1.0 / ((double)Hq * (double)P.l);
  const int bpc = max(1, (int)(kExStage / ((uint32_t)Hkv * kDh * 4)));  // blocks per chunk
  const int nch = (mv + bpc - 1) / bpc;
  double* q64 = reinterpret_cast<double*>(smem + kExQOff);  // [Hq][kExQS] fp64 (exact copies)
  double* Lg = R.exact;                                      // [Hq][blocks]
  if (tid == 0) {  // the request's scratch, one fallback at a time
    while (atomicCAS(&R.cnt[kCntLock], 0, 1) != 0) __nanosleep(1000);
    __threadfence();
  }
  __syncthreads();
  stamp(P, 9);
  auto issue = [&](int c) {  // chunk c -> stage (ex_seq + c) % kExStages
    const int sq = ex_seq + c, st = sq % kExStages;
    const int i0 = c * bpc, nb = min(bpc, mv - i0);
    const uint32_t bytes = (uint32_t)nb * Hkv * kDh * 4;
    mbar_expect_tx(&m.ex_full[st], bytes);
    bulk_g2s(smem + ex_stage_off(st), R.ck + (int64_t)i0 * Hkv * kDh, bytes, &m.ex_full[st]);
  };
  // KV-head groups whose q heads (<= 64) fit the fp64 q rows; the keys stream once per group
  const int kvg = max(1, 64 / G);
  for (int kv0 = 0; kv0 < Hkv; kv0 += kvg) {
    const int kv1 = min(Hkv, kv0 + kvg);
    __syncthreads();  // the previous group's q rows and stages are consumed
    for (int e = tid; e < (kv1 - kv0) * G * kDh; e += kThreads)
      q64[(e / kDh) * kExQS + e % kDh] = (double)R.q[((int64_t)qi * Hq + kv0 * G) * kDh + e];
    if (tid == 0)
      for (int c = 0; c < min(kExStages, nch); ++c) issue(c);
    __syncthreads();  // q visible
    // ---- pass 1: item = (block of the chunk, KV head, 8-way dims part): each key element
    // is converted to fp64 once and meets the G q heads of its KV head; the 8 parts of a
    // (block, KV head) are 8 consecutive lanes (fixed-order shuffle sum)
    const int part = tid & 7;
    const int nkv = kv1 - kv0;
    for (int c = 0; c < nch; ++c) {
      const int sq = ex_seq + c, st = sq % kExStages;
      mbar_wait(&m.ex_full[st], (sq / kExStages) & 1);
      const float* kst = reinterpret_cast<const float*>(smem + ex_stage_off(st));
      const int i0 = c * bpc, nb = min(bpc, mv - i0);
      for (int item = tid >> 3; item < nb * nkv; item += kThreads / 8) {
        const int it = item / nkv, kvl = item % nkv, kvh = kv0 + kvl;
        // dims part + 8 x: the 8 parts read consecutive words (no bank conflicts)
        const float* kr = kst + ((int64_t)it * Hkv + kvh) * kDh + part;
        double kx[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) kx[x] = (double)kr[8 * x];
        for (int g0 = 0; g0 < G; g0 += 4) {
          double acc[4];
#pragma unroll
          for (int gg = 0; gg < 4; ++gg) {
            acc[gg] = 0.0;
            if (g0 + gg < G) {
              const double* qr = q64 + (kvl * G + g0 + gg) * kExQS + part;
#pragma unroll
              for (int x = 0; x < 16; ++x) acc[gg] = fma(qr[8 * x], kx[x], acc[gg]);
            }
          }
#pragma unroll
          for (int gg = 0; gg < 4; ++gg)
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) acc[gg] += __shfl_xor_sync(0xffffffffu, acc[gg], o);
          if (part == 0)
#pragma unroll
            for (int gg = 0; gg < 4; ++gg)
              if (g0 + gg < G) Lg[(int64_t)(kvh * G + g0 + gg) * R.blocks + i0 + it] = acc[gg] * P.scale;
        }
      }
      __syncthreads();  // the stage is consumed
      if (tid == 0 && c + kExStages < nch) issue(c + kExStages);
    }
    ex_seq += nch;
  }
  double* Mh = reinterpret_cast<double*>(smem + kExQOff);  // q no longer needed: [kMaxHq] den
  __syncthreads();
  stamp(P, 10);
  // ---- pass 2 (warp w: heads w, w + 16, ..): the head's maximum, then e = exp(logit - max)
  // stored back and the denominator (lanes, then the warp tree: a fixed order)
  for (int h = warp; h < Hq; h += kWarps) {
    double* lh = Lg + (int64_t)h * R.blocks;
    double M = -INFINITY;
    for (int i = lane; i < mv; i += 32) M = fmax(M, __ldcg(lh + i));
    M = warp_max_d(M);
    double sm = 0.0;
    for (int i = lane; i < mv; i += 32) {
      const double e = exp_nonpos(__ldcg(lh + i) - M);
      lh[i] = e;
      sm += e;
    }
    sm = warp_sum_d(sm);
    if (lane == 0) Mh[kMaxHq + h] = sm;
  }
  __syncthreads();
  stamp(P, 11);
  // ---- pass 3: per selection block
  for (int b = tid; b < avail; b += kThreads) {
    int lo, hi;
    blocks_of(b, P.d, P.l, P.l_sel, lo, hi);
    hi = min(hi, mv - 1);
    double acc = 0.0;
    for (int h = 0; h < Hq; ++h) {
      const double D = Mh[kMaxHq + h];
      if (!(D > 0.0)) continue;
      double sh = 0.0;
      for (int i = lo; i <= hi; ++i)
        sh += __ldcg(Lg + (int64_t)h * R.blocks + i) * (double)overlap(i, b, P.d, P.l, P.l_sel);
      acc += sh / D;
    }
    sel[b] = acc * inv;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    atomicExch(&R.cnt[kCntLock], 0);
  }
}

// ------------------------------------------------------------------ kernel
template <int NR>
__global__ void __launch_bounds__(kThreads, 1) route3_kernel(const __grid_constant__ Route3LaunchT<NR> P) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  Misc& m = *reinterpret_cast<Misc*>(smem + kOffMisc);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x, nctas = gridDim.x;
  double* g = reinterpret_cast<double*>(smem + kOffG);  // [kR3MaxSpr][kGS]
  const int units = P.unit_start[P.n_req];
  if (tid == 0) {
    for (int t = 0; t < 2; ++t) {
      mbar_init(&m.tma_full[t], 1);
      mbar_init(&m.mma_done[t], 1);
    }
    for (int t = 0; t < 3; ++t) mbar_init(&m.ex_full[t], 1);
    fence_mbar_init();
  }
  // The first unit's key planes and block exponents are cache data (complete in
  // stream order before this call): they go out before the wait for the
  // previous launch, so they stream under its tail.  q comes after the wait.
  // a unit's setup that needs no q: counters, selection-block weights, zeroed sums,
  // block exponents (issue_unit_tma goes first, by thread 0)
  auto setup_unit = [&](const Unit& U, const Route3Req& R) {
    const int kpack = tid < U.nblk ? __ldg(R.ckexp + (int64_t)(U.row0 + tid) * P.Hkv + U.kvh) : 0;
    if (tid == 0) {
      m.flag = 0;
      m.kemax = -100000;
      m.nkmax = 0;
    }
    {  // compressed blocks overlapping each selection block of the range, and their token overlaps
      const int bl = tid & (kR3MaxSpr - 1), kg = tid / kR3MaxSpr;
      const int b = U.b0 + bl;
      int lo, hi;
      blocks_of(b, P.d, P.l, P.l_sel, lo, hi);
      hi = min(hi, U.row0 + U.nblk - 1);
      if (kg == 0) m.glo[bl] = lo;
      for (int kq = kg; kq < kR3MaxBps; kq += kThreads / kR3MaxSpr)
        m.gw[kq][bl] = lo + kq <= hi ? (double)overlap(lo + kq, b, P.d, P.l, P.l_sel) : 0.0;
    }
    for (int e = tid; e < kR3MaxSpr * kGS; e += kThreads) g[e] = 0.0;  // (selection blocks past nsel stay 0)
    __syncthreads();  // counter resets before the exponent maxima
    static_assert(kR3MaxBlk <= kThreads, "one block exponent per thread");
    if (tid < kR3MaxBlk) {
      const bool has = tid < U.nblk;
      const int ke = (int)(int16_t)(kpack & 0xFFFF), knx = (kpack >> 16) & 0xFF;  // exponent, rounded elements
      m.kexp[tid] = has ? ke : 0;
      if (has) {
        atomicMax(&m.kemax, ke);
        if (knx) atomicMax(&m.nkmax, knx);
      }
    }
  };
  // The first unit's key planes, block exponents and weights are cache data
  // (complete in stream order before this call): they go out before the wait
  // for the previous launch, under its tail.  q comes after the wait.
  if (tid < 16) m.T16[tid] = kT16[tid];
  if (cta < units) {
    const Unit U = unit_of(P, cta);
    const Route3Req& R = P.req[U.req];
    if (tid == 0) issue_unit_tma(R, U, smem, m);
    setup_unit(U, R);
  }
  // the previous launch (PDL) may still read what this one writes.  (q could
  // be read before the wait too -- a verify input, nsa_verify.h -- but loading
  // it under the previous launch's tail measured 0.3% slower in the step)
  griddep_wait();
  stamp(P, 0);
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = m.tmem_base;

  // ================= phase 1: logits, e, selection-block sums, den rows =================
  int k = 0;
  for (int u = cta; u < units; u += nctas, ++k) {
    const Unit U = unit_of(P, u);
    const Route3Req& R = P.req[U.req];
    const uint32_t par = k & 1;
    const int ntile = U.nblk > kTB ? 2 : 1;
    if (k > 0) {
      if (tid == 0) issue_unit_tma(R, U, smem, m);
      setup_unit(U, R);
    }
    float4 qv[3];
    load_q(P, R, U, qv);
    digit_q(P, R, U, qv, smem, m);
    fence_proxy_async_smem();  // q digits: generic-proxy writes read by the MMA
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (k == 0) stamp(P, 1);

    if (warp == kWarpMma) {  // both tiles' MMAs as their planes land
      // B = the q digit planes s >= s_lo stacked along N (rows s x 48 + j), so
      // one MMA multiplies key plane tt by every q plane it needs and writes
      // class c = s + tt at TMEM column block c - 2 (classes 2..6 = weights
      // 256^2..256^6; the lower pairs are dropped).  Per K step: (tt 2: s 0-3,
      // blocks 0-3, initialising), (tt 3, s 3: block 4, initialising), then
      // (tt 3: s 0-2), (tt 1: s 1-3), (tt 0: s 2-3) accumulate.
      const uint32_t qb = sbase + kOffQs;
      for (int t = 0; t < 2; ++t) {
        mbar_wait(&m.tma_full[t], par);
        if (t < ntile) {
          tc_fence_after();
          const uint32_t kb = sbase + t * kTileBytes, d0 = tmem + t * kAcc * kN;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t ko = 32 * kk;
            umma_i8_warp(d0, desc_sw128(kb + 2 * kPlaneBytes + ko, 16, 1024), desc_sw128(qb + ko, 16, 1024),
                         idesc_s8(kTB, 4 * kN), kk ? 1u : 0u);
            umma_i8_warp(d0 + 4 * kN, desc_sw128(kb + 3 * kPlaneBytes + ko, 16, 1024),
                         desc_sw128(qb + 3 * kQsSlice + ko, 16, 1024), idesc_s8(kTB, kN), kk ? 1u : 0u);
            umma_i8_warp(d0 + 1 * kN, desc_sw128(kb + 3 * kPlaneBytes + ko, 16, 1024), desc_sw128(qb + ko, 16, 1024),
                         idesc_s8(kTB, 3 * kN), 1u);
            umma_i8_warp(d0, desc_sw128(kb + 1 * kPlaneBytes + ko, 16, 1024),
                         desc_sw128(qb + 1 * kQsSlice + ko, 16, 1024), idesc_s8(kTB, 3 * kN), 1u);
            umma_i8_warp(d0, desc_sw128(kb + ko, 16, 1024), desc_sw128(qb + 2 * kQsSlice + ko, 16, 1024),
                         idesc_s8(kTB, 2 * kN), 1u);
          }
        }
        umma_commit_warp(&m.mma_done[t]);  // (no MMAs for a missing tile: arrives at once)
      }
    }
    const int qd = warp & 3, cg = warp >> 2;  // TMEM lane quadrant, 12-column group
    for (int t = 0; t < 2; ++t) {
      if (t >= ntile) {  // the empty commit's phase
        if (12 * cg < U.nrows) mbar_wait(&m.mma_done[t], par);
        continue;
      }
      if (12 * cg < U.nrows) {
        // ---- epilogue: recombine the classes, logit, e = 2^logit -> e values [256][64]
        mbar_wait(&m.mma_done[t], par);
        tc_fence_after();
        if (k == 0) stamp(P, 9 + t);
        uint32_t a[kAcc][12];
#pragma unroll
        for (int c = 0; c < kAcc; ++c) {
          const uint32_t ta = tmem + ((uint32_t)(32 * qd) << 16) + (t * kAcc + c) * kN + 12 * cg;
          tmem_ld8(ta, a[c]);
          tmem_ld4(ta + 8, a[c] + 8);
        }
        tmem_wait_ld();
        const int il = 32 * qd + lane, i = t * kTB + il;
        const int gb = U.row0 + i;
        const int ke_row = m.kexp[i];
        double* E = reinterpret_cast<double*>(smem);
        bool ovf = false;
        // branch-free so the 12 independent chains interleave: logits first,
        // then e = 2^logit (clamped into the exponent range; out-of-range
        // logits flag the query for the exact path)
        double Lv[12];
#pragma unroll
        for (int jj = 0; jj < 12; ++jj) {
          // h = a6 2^32 + a5 2^24 + a4 2^16 + a3 2^8 + a2 (classes 2..6; |a_c|
          // <= pairs x 2^21): the top two in int32 (< 2^30), the bottom three in
          // int64 (< 2^40), one fp64 FMA (rounding 2^-53 relative)
          const double hi = i2d((int)a[3][jj] + ((int)a[4][jj] << 8));
          const long long lo = (long long)(int)a[2][jj] * 65536 + (long long)(int)a[1][jj] * 256 + (int)a[0][jj];
          Lv[jj] = scale2(fma(hi, 16777216.0, l2d(lo)) * m.qsc[12 * cg + jj], ke_row);
        }
        const bool row_ok = i < U.nblk;
#pragma unroll
        for (int jj = 0; jj < 12; ++jj) {
          const int j = 12 * cg + jj;
          const bool valid = row_ok && gb < m.colmvis[j];
          // |logit| >= 512 log2 units: outside the fp64 exp's range here -- the
          // query goes to the exact path
          ovf |= valid && (__double2hiint(Lv[jj]) & 0x7fffffff) >= 0x40800000;
          const double e = exp2_fast(Lv[jj], m.T16);
          E[i * kES + (j ^ (i & 15))] = valid ? e : 0.0;
        }
        if (__any_sync(0xffffffffu, ovf) && lane == 0) m.flag = 1;
      }
    }
    tc_fence_before();
    __syncthreads();
    if (k == 0) stamp(P, 2);
    {  // ---- selection-block sums: thread (row j, eight consecutive selection
       // blocks), eight independent chains; the rows of one column read along a
       // warp are consecutive (conflict-free)
      const double* E = reinterpret_cast<const double*>(smem);
      const int nsel = U.b1 - U.b0;
      const int ngrp = (nsel + 7) / 8;
      for (int item = tid; item < U.nrows * ngrp; item += kThreads) {
        const int j = item % U.nrows, bl0 = 8 * (item / U.nrows);
        int rr[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) rr[z] = m.glo[min(bl0 + z, kR3MaxSpr - 1)] - U.row0;
        double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int kq = 0; kq < P.bps; ++kq)
#pragma unroll
          for (int z = 0; z < 8; ++z) {
            const int r = min(rr[z] + kq, U.nblk - 1);  // (weights past a block's last row are 0; rows
                                                         //  below nblk are written, zero when masked)
            acc[z] = fma(m.gw[kq][min(bl0 + z, kR3MaxSpr - 1)], E[r * kES + (j ^ (r & 15))], acc[z]);
          }
#pragma unroll
        for (int z = 0; z < 8; ++z)
          if (bl0 + z < nsel) g[(bl0 + z) * kGS + j] = acc[z];
      }
    }
    __syncthreads();
    if (k == 0) stamp(P, 3);
    // ---- this range's denominator rows, error exponents, spill, arrival
    {
      double* den = R.den + ((int64_t)(U.chunk * P.Hkv + U.kvh) * R.nranges + U.range) * kN;
      if (tid < kN) {  // four partial sums, then in order
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        for (int bl = 0; bl < kR3MaxSpr; bl += 4)
#pragma unroll
          for (int z = 0; z < 4; ++z) v[z] += g[(bl + z) * kGS + tid];
        den[tid] = (v[0] + v[1]) + (v[2] + v[3]);
      }
      if (tid < U.nrows) {
        // |logit error| <= 2^(eq + ek - 31) (rounded q elements + rounded k elements + 2.01):
        // grid rounding of the rounded elements only, plus the three dropped low digit
        // pairs (< 2^(eq + ek - 29.99)); per unit the largest ek and k count, x2 margin
        const double bnd = m.flag ? __longlong_as_double((long long)kBoundFlag)
                                  : P.c_sl * pow2i(max(-1000, min(1000, m.qexp[tid] + m.kemax - 30))) *
                                        ((double)(m.nkmax + m.qinex[tid]) + 2.01);
        atomicMax(reinterpret_cast<unsigned long long*>(R.cnt + kCntBound) + U.s0 + tid / P.G,
                  (unsigned long long)__double_as_longlong(bnd));
      }
      if (u + nctas < units) {  // not this CTA's last unit: phase 2 reloads g from L2
        double* sp = R.gspill + (int64_t)U.lu * kR3MaxSpr * kGS;
        for (int e = tid; e < kR3MaxSpr * kGS; e += kThreads) sp[e] = g[e];
      }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) red_add_release_gpu(&R.cnt[kCntDen + U.chunk * P.Hkv + U.kvh], 1);
  }
  if (warp == 0 && cta < units) tmem_dealloc<kTmemCols>(tmem);
  if (k > 0) stamp(P, 4);

  // ================= phase 2: denominators, per-KV-head shares =================
  for (int u = cta; u < units; u += nctas) {
    const Unit U = unit_of(P, u);
    const Route3Req& R = P.req[U.req];
    const bool last = u + nctas >= units;
    if (tid == 0) {
      const int* c = &R.cnt[kCntDen + U.chunk * P.Hkv + U.kvh];
      while (ld_acquire_gpu(c) < R.nranges) {
      }
    }
    __syncthreads();
    if (u == cta) stamp(P, 5);
    double* st = reinterpret_cast<double*>(smem);                // [nranges][48] den rows
    double* gs = last ? g : reinterpret_cast<double*>(smem + kTileBytes);  // this unit's g
    const double* src = R.den + (int64_t)(U.chunk * P.Hkv + U.kvh) * R.nranges * kN;
    for (int e0 = tid; e0 < R.nranges * kN; e0 += 4 * kThreads) {  // loads first: one round trip
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = e0 + u * kThreads < R.nranges * kN ? __ldcg(src + e0 + u * kThreads) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e0 + u * kThreads < R.nranges * kN) st[e0 + u * kThreads] = x[u];
    }
    if (!last) {
      const double* sp = R.gspill + (int64_t)U.lu * kR3MaxSpr * kGS;
      for (int e = tid; e < kR3MaxSpr * kGS; e += kThreads) gs[e] = __ldcg(sp + e);
    }
    __syncthreads();
    if (tid < kN) {
      double D = 0.0;  // ranges in ascending order
      for (int r = 0; r < R.nranges; ++r) D += st[r * kN + tid];
      m.invD[tid] = D > 0.0 ? 1.0 / D : 0.0;
      if (tid < U.nrows && D > 0.0 && D < 0x1p-900)  // e values may have lost bits: exact path
        atomicMax(reinterpret_cast<unsigned long long*>(R.cnt + kCntBound) + U.s0 + tid / P.G, kBoundFlag);
    }
    __syncthreads();
    const int nsel = U.b1 - U.b0;
    for (int e = tid; e < U.nslots * nsel; e += kThreads) {
      const int sl = e / nsel, bl = e % nsel;
      double c = 0.0;
      for (int h = 0; h < P.G; ++h) c = fma(gs[bl * kGS + sl * P.G + h], m.invD[sl * P.G + h], c);
      // the KV heads' shares meet in one score row per slot (fp64 atomics: the
      // summation order varies, inside the certified bound; the Top-n task
      // reads the row and zeroes it for the next launch)
      atomicAdd(R.contrib + (int64_t)(U.s0 + sl) * R.sel_pad + U.b0 + bl, c);
    }
    __syncthreads();
    if (tid == 0) red_add_release_gpu(&R.cnt[kCntTop + U.chunk], 1);
  }
  stamp(P, 6);
  const int tasks = P.task_start[P.n_req];
  // The denominator counters are reset once no unit polls them: by the last
  // Top-n task through its wait below (every unit of every chunk has then
  // published its shares, after its denominator wait), so no CTA spends an
  // atomic round trip here.  Without tasks (or debug bit 6 (64)): by the
  // last CTA through phase 2.
  const bool den_by_tasks = tasks > 0 && !(P.debug & 64);
  if (!den_by_tasks && tid == 0 && atom_add_acq_rel_gpu(P.exit_cnt, 1) == nctas - 1) {
    // the last CTA through phase 2: no unit polls a denominator counter any more
    for (int r = 0; r < P.n_req; ++r)
      for (int i = 0; i < P.req[r].nchunks * P.Hkv; ++i) P.req[r].cnt[kCntDen + i] = 0;
    st_release_gpu(P.exit_cnt, 0);
  }

  // ================= phase 3: one Top-n task per routed slot =================
  griddep_launch();  // the next launch may start placing CTAs as this grid drains
  double* sel = reinterpret_cast<double*>(smem);                          // [kMaxAvail]
  int* surv = reinterpret_cast<int*>(smem + 8 * kMaxAvail);                // [kMaxAvail]
  int ex_seq = 0;  // exact-path chunks loaded by this CTA so far (the stage barriers' phases)
  for (int t = nctas - 1 - cta; t < tasks; t += nctas) {
    int r = 0;
    while (r + 1 < P.n_req && t >= P.task_start[r + 1]) ++r;
    const Route3Req& R = P.req[r];
    const int slot = t - P.task_start[r];
    const int chunk = slot / P.spc;
    if (tid == 0) {
      const int* c = &R.cnt[kCntTop + chunk];
      while (ld_acquire_gpu(c) < P.Hkv * R.nranges) {
      }
    }
    __syncthreads();
    stamp(P, 7);
    const int avail = R.slot_avail[slot];
    const double inv = 1.0 / (double)P.Hq;
    if (tid == 0 && atom_add_acq_rel_gpu(P.exit_cnt + 1, 1) == tasks - 1) {
      // the last task through its wait: no task polls a chunk counter any more
      // (nor any unit a denominator counter: every chunk has a task)
      for (int rr = 0; rr < P.n_req; ++rr) {
        for (int i = 0; i < P.req[rr].nchunks; ++i) P.req[rr].cnt[kCntTop + i] = 0;
        if (den_by_tasks)
          for (int i = 0; i < P.req[rr].nchunks * P.Hkv; ++i) P.req[rr].cnt[kCntDen + i] = 0;
      }
      st_release_gpu(P.exit_cnt + 1, 0);
    }
    double* sc = R.contrib + (int64_t)slot * R.sel_pad;
    unsigned long long* bslot = reinterpret_cast<unsigned long long*>(R.cnt + kCntBound) + slot;
    const unsigned long long bb = __ldcg(bslot);
    // the score row in one round trip: every load of this thread before any store
    for (int b0 = tid; b0 < avail; b0 += 4 * kThreads) {
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = b0 + u * kThreads < avail ? __ldcg(sc + b0 + u * kThreads) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (b0 + u * kThreads < avail) {
          sel[b0 + u * kThreads] = x[u] * inv;
          sc[b0 + u * kThreads] = 0.0;
        }
    }
    __syncthreads();
    stamp(P, 14);
    if (tid == 0) *bslot = 0ull;  // every atomicMax of this launch is in
    // relative score error <= 2 ln2 delta (+ fp64 exp / summation rounding), with margin
    const bool flagged = bb >= kBoundFlag;
    const double delta = flagged ? 0.0 : __longlong_as_double((long long)bb);
    const double eps = 1.5 * 2.0 * 0.6931471805599453 * delta + 2e-10;
#ifdef SPECSV_TRACE_TILES
    const long long c0 = clock64();
    select_topn(sel, surv, avail, P.n, eps, m, P.debug,
                P.trace != nullptr ? P.trace + kRouteTraceBase + blockIdx.x * 16 : nullptr);
    stamp(P, 15);
    if (P.trace != nullptr && tid == 0) P.trace[kRouteTraceBase + blockIdx.x * 16 + 12] = clock64() - c0;
    if (P.debug & 1) {  // diagnostics: the selection again (warm instruction cache)
      select_topn(sel, surv, avail, P.n, eps, m, P.debug);
      stamp(P, 13);
    }
#else
    select_topn(sel, surv, avail, P.n, eps, m, P.debug);
#endif
    if (flagged || !m.certified || P.force_exact) {
      if (tid == 0 && P.fallbacks != nullptr) atomicAdd(P.fallbacks, 1);
      exact_scores(P, R, slot, sel, smem, m, ex_seq);
      select_topn(sel, surv, avail, P.n, 0.0, m, P.debug);
    }
    const int q = R.slot_q[slot];
    write_row(m, m, avail, P.n, R.idx + (int64_t)q * P.n, R.idx_count + q, R.idx_forced + q);
    __syncthreads();
  }
  stamp(P, 8);
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

template <int NR>
cudaError_t launch_route3_n(const Route3LaunchT<NR>& p, int ctas, cudaStream_t s) {
  static std::atomic<int> done[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& d = done[dev < 64 ? dev : 63];
  if (!d.load(std::memory_order_acquire)) {  // the shared-memory opt-in, once per device
    const cudaError_t e = cudaFuncSetAttribute(route3_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    d.store(1, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  // CTAs wait on each other's arrivals, so every CTA must be resident (the
  // host sizes the grid to one CTA per SM).  Under programmatic dependent
  // launch the cooperative attribute is dropped, as for the attend launch:
  // CTAs are then placed as the previous launch's CTAs retire, and all of them
  // become resident because nothing the previous launch waits on depends on
  // this grid (with the attribute, eager launches started ~2-3 us later).
  // (debug bit 4 keeps it, for A/B timing)
  if (!pdl_enabled() || (p.debug & 16)) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na++].val.cooperative = 1;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, route3_kernel<NR>, p);
}

}  // namespace

int route3_grid() { return sm_count3(); }

cudaError_t launch_route3(Route3Launch& p, cudaStream_t s) {
  p.unit_start[0] = 0;
  p.task_start[0] = 0;
  for (int r = 0; r < p.n_req; ++r) {
    const Route3Req& R = p.req[r];
    p.unit_start[r + 1] = p.unit_start[r] + p.Hkv * R.nchunks * R.nranges;
    p.task_start[r + 1] = p.task_start[r] + R.nr;
  }
  const int work = std::max(p.unit_start[p.n_req], p.task_start[p.n_req]);
  const int ctas = std::max(1, std::min(sm_count3(), work));
  if (p.n_req == 1 && !(p.debug & 4)) {  // the one-request parameter block (debug bit 2: the full one)
    thread_local Route3LaunchT<1> one;
    static_cast<Route3Common&>(one) = static_cast<const Route3Common&>(p);
    one.req[0] = p.req[0];
    one.unit_start[0] = p.unit_start[0];
    one.unit_start[1] = p.unit_start[1];
    one.task_start[0] = p.task_start[0];
    one.task_start[1] = p.task_start[1];
    return launch_route3_n(one, ctas, s);
  }
  return launch_route3_n(p, ctas, s);
}

}  // namespace specsv_b200
