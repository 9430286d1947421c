/*
 * nsa_oracle.c -- TEST INFRASTRUCTURE ONLY (see nsa_oracle.h).
 *
 * Plain-C restatement of the reference's NSA verify hot path.  Compile with
 * -O2 -ffp-contract=off so every double operation rounds exactly where the
 * reference's does (CMakeLists.txt:14-16).  Citations are relative to
 * /root/reference/proj.
 */
#include "nsa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

const char* or_impl_name(void) { return "oracle-c"; }

/* config.hpp:38-51 */
int or_validate(const or_config* c) {
  if (c->l <= 0) return OR_EINVAL;
  if (c->d <= 0 || c->d > c->l) return OR_EINVAL;
  if (c->l_sel <= 0 || c->l_sel % c->d != 0) return OR_EINVAL;
  if (c->n < 3) return OR_EINVAL;
  if (c->w <= 0) return OR_EINVAL;
  if (c->n_q_heads <= 0 || c->n_kv_heads <= 0 || c->n_q_heads % c->n_kv_heads != 0)
    return OR_EINVAL;
  if (c->d_head <= 0) return OR_EINVAL;
  if (c->n_layers <= 0) return OR_EINVAL;
  if (c->routing_lag < 0) return OR_EINVAL;
  if (c->w < c->routing_lag) return OR_EINVAL;
  return OR_OK;
}

/* config.hpp:55-58 */
static int64_t routing_visible_len(const or_config* c, int64_t pos) {
  int64_t v = pos + 1 - c->routing_lag;
  return v > 0 ? v : 0;
}

/* rng.hpp:17-29 */
uint64_t or_rng_fill_symmetric(uint64_t state, float a, float* out, int64_t count) {
  for (int64_t i = 0; i < count; ++i) {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z = z ^ (z >> 31);
    double unit = (double)(z >> 11) * 0x1.0p-53;
    out[i] = (float)((2.0 * unit - 1.0) * (double)a);
  }
  return state;
}

/* kernels_scalar.cpp:12-26: four interleaved lanes, (s0+s2)+(s1+s3), tail */
double or_dot_f32(const float* a, const float* b, int64_t n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 += (double)a[i + 0] * (double)b[i + 0];
    s1 += (double)a[i + 1] * (double)b[i + 1];
    s2 += (double)a[i + 2] * (double)b[i + 2];
    s3 += (double)a[i + 3] * (double)b[i + 3];
  }
  double r = (s0 + s2) + (s1 + s3);
  for (; i < n; ++i) r += (double)a[i] * (double)b[i];
  return r;
}

/* cache.hpp:84-86 */
int64_t or_compressed_block_count(int64_t n_rows, const or_config* c) {
  return n_rows >= c->l ? (n_rows - c->l) / c->d + 1 : 0;
}

/* cache.hpp:77-81 */
static int64_t visible_blocks(const or_config* c, int64_t block_count, int64_t visible_len) {
  if (visible_len < c->l) return 0;
  int64_t by_len = (visible_len - c->l) / c->d + 1;
  return by_len < block_count ? by_len : block_count;
}

/* attention.hpp:18-21 */
static int64_t selection_block_count(const or_config* c, int64_t visible_len) {
  return visible_len > 0 ? (visible_len + c->l_sel - 1) / c->l_sel : 0;
}

/* nsa_cache.cpp:14-32 (pool_block) driven by extend_compressed_layer :45-66 */
int64_t or_build_compressed(const or_config* c, const float* k, const float* v,
                            int64_t committed_len, const float* pe, float* ck, float* cv) {
  const int64_t dh = c->d_head, H = c->n_kv_heads;
  const int64_t want = or_compressed_block_count(committed_len, c);
  double* acc_k = (double*)malloc(sizeof(double) * dh);
  double* acc_v = (double*)malloc(sizeof(double) * dh);
  const double inv_l = 1.0 / (double)c->l;
  for (int64_t b = 0; b < want; ++b) {
    for (int64_t h = 0; h < H; ++h) {
      for (int64_t j = 0; j < dh; ++j) acc_k[j] = acc_v[j] = 0.0;
      const int64_t start = b * c->d;
      for (int64_t o = 0; o < c->l; ++o) {
        const float* kr = k + ((start + o) * H + h) * dh;
        const float* vr = v + ((start + o) * H + h) * dh;
        for (int64_t j = 0; j < dh; ++j) acc_k[j] += (double)kr[j];
        if (pe != NULL)
          for (int64_t j = 0; j < dh; ++j) acc_k[j] += (double)pe[o * dh + j];
        for (int64_t j = 0; j < dh; ++j) acc_v[j] += (double)vr[j];
      }
      float* ok = ck + (b * H + h) * dh;
      float* ov = cv + (b * H + h) * dh;
      for (int64_t j = 0; j < dh; ++j) {
        ok[j] = (float)(acc_k[j] * inv_l);
        ov[j] = (float)(acc_v[j] * inv_l);
      }
    }
  }
  free(acc_k);
  free(acc_v);
  return want;
}

static double logit_scale(const or_config* c) { return 1.0 / sqrt((double)c->d_head); }

/* nsa_attention.cpp:38-80 */
int64_t or_selection_scores(const or_config* c, const float* q, const float* ck, int64_t blocks,
                            int64_t visible_len, double* sel) {
  const int64_t sel_count = selection_block_count(c, visible_len);
  for (int64_t b = 0; b < sel_count; ++b) sel[b] = 0.0;
  const int64_t m = visible_blocks(c, blocks, visible_len);
  if (m == 0) return sel_count;
  const double scale = logit_scale(c);
  const int64_t group = c->n_q_heads / c->n_kv_heads;
  const int64_t dh = c->d_head, H = c->n_kv_heads;
  double* mass = (double*)calloc((size_t)m, sizeof(double));
  double* logits = (double*)malloc(sizeof(double) * (size_t)m);
  for (int64_t h = 0; h < c->n_q_heads; ++h) {
    const float* qh = q + h * dh;
    const int64_t kvh = h / group;
    double mx = -INFINITY;
    for (int64_t i = 0; i < m; ++i) {
      logits[i] = or_dot_f32(qh, ck + (i * H + kvh) * dh, dh) * scale;
      mx = mx < logits[i] ? logits[i] : mx; /* std::max(mx, x) */
    }
    double den = 0.0;
    for (int64_t i = 0; i < m; ++i) den += exp(logits[i] - mx);
    for (int64_t i = 0; i < m; ++i) mass[i] += exp(logits[i] - mx) / den;
  }
  const double inv_heads = 1.0 / (double)c->n_q_heads;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t lo = i * c->d, hi = lo + c->l;
    for (int64_t b = lo / c->l_sel; b * c->l_sel < hi; ++b) {
      const int64_t olo = lo > b * c->l_sel ? lo : b * c->l_sel;
      const int64_t ohi = hi < (b + 1) * c->l_sel ? hi : (b + 1) * c->l_sel;
      if (ohi <= olo) continue;
      sel[b] += mass[i] * inv_heads * (double)(ohi - olo) / (double)c->l;
    }
  }
  free(mass);
  free(logits);
  return sel_count;
}

/* nsa_attention.cpp:82-92 */
static int64_t forced_blocks(const or_config* c, int64_t visible_len, int64_t* out) {
  const int64_t avail = selection_block_count(c, visible_len);
  if (avail == 0) return 0;
  int64_t n = 0;
  out[n++] = 0;
  if (avail - 2 > 0) out[n++] = avail - 2;
  if (avail - 1 > 0 && avail - 1 != avail - 2) out[n++] = avail - 1;
  /* already ascending; dedupe (avail - 2 == 0 is excluded above) */
  return n;
}

static const double* g_sort_scores;
static int cmp_rest(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  if (g_sort_scores[a] != g_sort_scores[b]) return g_sort_scores[a] > g_sort_scores[b] ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}
static int cmp_i64(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* nsa_attention.cpp:94-136 */
int64_t or_select_blocks(const or_config* c, const double* scores, int64_t n,
                         int64_t visible_len, const int64_t* forced_in, int64_t n_forced,
                         int64_t* idx_out, uint8_t* forced_out) {
  const int64_t avail = selection_block_count(c, visible_len);
  if (avail == 0) return 0;
  int64_t derived[3];
  if (forced_in == NULL) {
    n_forced = forced_blocks(c, visible_len, derived);
    forced_in = derived;
  }
  const int64_t target = n < avail ? n : avail;
  uint8_t* is_forced = (uint8_t*)calloc((size_t)avail, 1);
  int64_t* chosen = (int64_t*)malloc(sizeof(int64_t) * (size_t)(avail + n_forced + 1));
  int64_t nc = 0;
  for (int64_t i = 0; i < n_forced; ++i) {
    int64_t b = forced_in[i];
    if (b >= 0 && b < avail && !is_forced[b]) {
      is_forced[b] = 1;
      chosen[nc++] = b;
    }
  }
  int64_t* rest = (int64_t*)malloc(sizeof(int64_t) * (size_t)avail);
  int64_t nr = 0;
  for (int64_t b = 0; b < avail; ++b)
    if (!is_forced[b]) rest[nr++] = b;
  /* the (score desc, id asc) order is total, so the sort is unique */
  g_sort_scores = scores;
  qsort(rest, (size_t)nr, sizeof(int64_t), cmp_rest);
  for (int64_t i = 0; i < nr && nc < target; ++i) chosen[nc++] = rest[i];
  qsort(chosen, (size_t)nc, sizeof(int64_t), cmp_i64);
  for (int64_t i = 0; i < nc; ++i) {
    idx_out[i] = chosen[i];
    if (forced_out) forced_out[i] = is_forced[chosen[i]];
  }
  free(is_forced);
  free(chosen);
  free(rest);
  return nc;
}

/* nsa_attention.cpp:22-36; p = [out[dh], run_max, run_den] */
static void online_update(double* p, int64_t dh, double logit, const float* v) {
  double* run_max = p + dh;
  double* run_den = p + dh + 1;
  if (logit <= *run_max) {
    const double w = exp(logit - *run_max);
    *run_den += w;
    for (int64_t i = 0; i < dh; ++i) p[i] += w * (double)v[i];
  } else {
    const double scale = exp(*run_max - logit);
    *run_den = *run_den * scale + 1.0;
    for (int64_t i = 0; i < dh; ++i) p[i] *= scale;
    for (int64_t i = 0; i < dh; ++i) p[i] += 1.0 * (double)v[i];
    *run_max = logit;
  }
}

static void partial_init(double* p, int64_t dh) {
  for (int64_t i = 0; i < dh; ++i) p[i] = 0.0;
  p[dh] = -INFINITY;
  p[dh + 1] = 0.0;
}

/* nsa_attention.cpp:138-159 */
void or_branch_compressed(const or_config* c, const float* q, const float* ck, const float* cv,
                          int64_t blocks, int64_t visible_len, double* parts) {
  const double scale = logit_scale(c);
  const int64_t group = c->n_q_heads / c->n_kv_heads;
  const int64_t m = visible_blocks(c, blocks, visible_len);
  const int64_t dh = c->d_head, H = c->n_kv_heads;
  for (int64_t h = 0; h < c->n_q_heads; ++h) {
    double* p = parts + h * (dh + 2);
    partial_init(p, dh);
    const float* qh = q + h * dh;
    const int64_t kvh = h / group;
    for (int64_t i = 0; i < m; ++i) {
      const double logit = or_dot_f32(qh, ck + (i * H + kvh) * dh, dh) * scale;
      online_update(p, dh, logit, cv + (i * H + kvh) * dh);
    }
  }
}

/* nsa_attention.cpp:161-189 */
void or_branch_selected(const or_config* c, const float* q, const float* k, const float* v,
                        int64_t rows, const int64_t* blocks, int64_t n_blocks,
                        const uint8_t* ownership, int64_t token_bound, double* parts) {
  const double scale = logit_scale(c);
  const int64_t group = c->n_q_heads / c->n_kv_heads;
  const int64_t bound = token_bound < rows ? token_bound : rows;
  const int64_t dh = c->d_head, H = c->n_kv_heads;
  for (int64_t h = 0; h < c->n_q_heads; ++h) {
    double* p = parts + h * (dh + 2);
    partial_init(p, dh);
    const float* qh = q + h * dh;
    const int64_t kvh = h / group;
    for (int64_t bi = 0; bi < n_blocks; ++bi) {
      if (ownership != NULL && !ownership[bi]) continue;
      const int64_t lo = blocks[bi] * c->l_sel;
      const int64_t hi = lo + c->l_sel < bound ? lo + c->l_sel : bound;
      for (int64_t t = lo; t < hi; ++t) {
        const double logit = or_dot_f32(qh, k + (t * H + kvh) * dh, dh) * scale;
        online_update(p, dh, logit, v + (t * H + kvh) * dh);
      }
    }
  }
}

/* nsa_attention.cpp:191-222 */
void or_branch_window(const or_config* c, const float* q, const float* k, const float* v,
                      int64_t rows, int64_t pos, int64_t committed_len, const float* tree_k,
                      const float* tree_v, const int32_t* admitted, int64_t n_admitted,
                      double* parts) {
  (void)rows;
  const double scale = logit_scale(c);
  const int64_t group = c->n_q_heads / c->n_kv_heads;
  const int64_t lo = pos - c->w + 1 > 0 ? pos - c->w + 1 : 0;
  const int64_t hi = pos < committed_len - 1 ? pos : committed_len - 1;
  const int64_t dh = c->d_head, H = c->n_kv_heads;
  for (int64_t h = 0; h < c->n_q_heads; ++h) {
    double* p = parts + h * (dh + 2);
    partial_init(p, dh);
    const float* qh = q + h * dh;
    const int64_t kvh = h / group;
    for (int64_t t = lo; t <= hi; ++t) {
      const double logit = or_dot_f32(qh, k + (t * H + kvh) * dh, dh) * scale;
      online_update(p, dh, logit, v + (t * H + kvh) * dh);
    }
    if (tree_k != NULL) {
      for (int64_t a = 0; a < n_admitted; ++a) {
        const int64_t r = admitted[a];
        const double logit = or_dot_f32(qh, tree_k + (r * H + kvh) * dh, dh) * scale;
        online_update(p, dh, logit, tree_v + (r * H + kvh) * dh);
      }
    }
  }
}

/* nsa_attention.cpp:224-237 */
void or_merge_partials(int64_t dh, const double* a, const double* b, double* r) {
  if (a[dh + 1] == 0.0) {
    memcpy(r, b, sizeof(double) * (size_t)(dh + 2));
    return;
  }
  if (b[dh + 1] == 0.0) {
    memcpy(r, a, sizeof(double) * (size_t)(dh + 2));
    return;
  }
  const double mx = a[dh] < b[dh] ? b[dh] : a[dh];
  const double sa = exp(a[dh] - mx), sb = exp(b[dh] - mx);
  r[dh] = mx;
  r[dh + 1] = a[dh + 1] * sa + b[dh + 1] * sb;
  for (int64_t i = 0; i < dh; ++i) r[i] = a[i] * sa + b[i] * sb;
}

/* nsa_attention.cpp:239-251 */
void or_gated_combine(int64_t dh, const double* cmp, const double* slc, const double* win,
                      const double* g, double* out) {
  for (int64_t i = 0; i < dh; ++i) out[i] = 0.0;
  const double* parts[3] = {cmp, slc, win};
  for (int b = 0; b < 3; ++b) {
    const double* p = parts[b];
    if (p[dh + 1] == 0.0) continue;
    for (int64_t i = 0; i < dh; ++i) out[i] += g[b] * (p[i] / p[dh + 1]);
  }
}

/* group_attend.cpp:20-40 */
int64_t or_merged_schedule(const int64_t* sets, const int64_t* counts, int64_t n_sets,
                           int64_t stride, int64_t* uniq, uint8_t* own) {
  int64_t total = 0;
  for (int64_t s = 0; s < n_sets; ++s) total += counts[s];
  int64_t* all = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total + 1));
  int64_t na = 0;
  for (int64_t s = 0; s < n_sets; ++s)
    for (int64_t i = 0; i < counts[s]; ++i) all[na++] = sets[s * stride + i];
  qsort(all, (size_t)na, sizeof(int64_t), cmp_i64);
  int64_t nu = 0;
  for (int64_t i = 0; i < na; ++i)
    if (nu == 0 || all[i] != uniq[nu - 1]) uniq[nu++] = all[i];
  free(all);
  if (own != NULL) {
    for (int64_t s = 0; s < n_sets; ++s) {
      uint8_t* row = own + s * nu;
      memset(row, 0, (size_t)nu);
      int64_t j = 0;
      for (int64_t i = 0; i < counts[s]; ++i) {
        const int64_t b = sets[s * stride + i];
        while (uniq[j] < b) ++j;
        row[j] = 1;
      }
    }
  }
  return nu;
}

/* group_attend.cpp:42-57 */
static int64_t overlap_count(const int64_t* a, int64_t na, const int64_t* b, int64_t nb) {
  int64_t s = 0, i = 0, j = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (a[i] > b[j]) ++j;
    else { ++s; ++i; ++j; }
  }
  return s;
}

/* group_attend.cpp:112-119 */
int64_t or_representative_index(const int64_t* positions, int64_t n) {
  if (n <= 0) return -1;
  int64_t rep = 0;
  for (int64_t i = 1; i < n; ++i)
    if (positions[i] >= positions[rep]) rep = i;
  return rep;
}

/* layer_roles.cpp:37-50 */
int64_t or_clamp_inherited(const or_config* c, const int64_t* src, const uint8_t* src_forced,
                           int64_t count, int64_t causal_bound, int64_t* out,
                           uint8_t* out_forced) {
  int64_t n = 0;
  for (int64_t i = 0; i < count; ++i) {
    if (src[i] * c->l_sel >= causal_bound) continue;
    out[n] = src[i];
    if (out_forced) out_forced[n] = src_forced ? src_forced[i] : 0;
    ++n;
  }
  return n;
}

/* group_attend.cpp:59-73: attend_one for member query qi */
typedef struct layer_ctx {
  const or_config* c;
  const float *k, *v, *ck, *cv, *tree_k, *tree_v;
  int64_t rows, blocks;
} layer_ctx;

static void attend_one(const layer_ctx* L, const float* q, int64_t pos, const int64_t* blocks,
                       int64_t n_blocks, const uint8_t* ownership, const double* gates,
                       const int32_t* admitted, int64_t n_admitted, int use_tree, double* out) {
  const or_config* c = L->c;
  const int64_t dh = c->d_head, Hq = c->n_q_heads;
  const int64_t bound = routing_visible_len(c, pos);
  double* cmp = (double*)malloc(sizeof(double) * (size_t)(Hq * (dh + 2)));
  double* slc = (double*)malloc(sizeof(double) * (size_t)(Hq * (dh + 2)));
  double* win = (double*)malloc(sizeof(double) * (size_t)(Hq * (dh + 2)));
  or_branch_compressed(c, q, L->ck, L->cv, L->blocks, bound, cmp);
  or_branch_selected(c, q, L->k, L->v, L->rows, blocks, n_blocks, ownership, bound, slc);
  or_branch_window(c, q, L->k, L->v, L->rows, pos, L->rows, use_tree ? L->tree_k : NULL,
                   use_tree ? L->tree_v : NULL, admitted, n_admitted, win);
  for (int64_t h = 0; h < Hq; ++h)
    or_gated_combine(dh, cmp + h * (dh + 2), slc + h * (dh + 2), win + h * (dh + 2),
                     gates + h * 3, out + h * dh);
  free(cmp);
  free(slc);
  free(win);
}

/* group_attend.cpp:76-83 */
static int64_t window_rows_attended(const or_config* c, int64_t pos, int64_t rows,
                                    int64_t n_admitted) {
  const int64_t lo = pos - c->w + 1 > 0 ? pos - c->w + 1 : 0;
  const int64_t hi = pos < rows - 1 ? pos : rows - 1;
  int64_t r = hi >= lo ? hi - lo + 1 : 0;
  return r + n_admitted;
}

/* engine.cpp:175-278 (per-layer hot section of run_target_pass) */
int or_verify_layer(const or_config* c, const float* k, const float* v, int64_t rows,
                    const float* ck, const float* cv, int64_t blocks, const float* tree_k,
                    const float* tree_v, int64_t nq, const float* q, const int64_t* pos,
                    const double* gates, const uint64_t* tree_mask, int64_t mask_words,
                    int64_t C, int mode, int role, int64_t* idx, int64_t* idx_count,
                    uint8_t* idx_forced, double* out, or_stats* st) {
  if (or_validate(c) != OR_OK || nq < 1 || C < 1) return OR_EINVAL;
  const int64_t n = c->n, dh = c->d_head, Hq = c->n_q_heads;
  const int64_t qstride = Hq * dh;
  const int64_t gamma = nq - 1;
  const int approx = mode == OR_MODE_APPROX;
  layer_ctx L = {c, k, v, ck, cv, tree_k, tree_v, rows, blocks};
  memset(st, 0, sizeof(*st));

  double* scores = (double*)malloc(sizeof(double) * (size_t)(rows / c->l_sel + 2));
  if (role == OR_ROLE_REFRESH) {
    for (int64_t qi = 0; qi < nq; ++qi) {
      idx_count[qi] = -1;
      for (int64_t i = 0; i < n; ++i) idx[qi * n + i] = -1;
    }
    /* route(q), engine.cpp:176-183 */
#define ROUTE(qi)                                                                        \
  do {                                                                                   \
    const int64_t vis = routing_visible_len(c, pos[qi]);                                 \
    or_selection_scores(c, q + (qi) * qstride, ck, blocks, vis, scores);                 \
    idx_count[qi] = or_select_blocks(c, scores, n, vis, NULL, 0, idx + (qi) * n,         \
                                     idx_forced + (qi) * n);                             \
  } while (0)
    ROUTE(0);
    if (!approx) {
      for (int64_t qi = 1; qi < nq; ++qi) ROUTE(qi);
    } else {
      for (int64_t b = 0; b < gamma; b += C) {
        const int64_t e = b + C < gamma ? b + C : gamma;
        const int64_t rep = or_representative_index(pos + 1 + b, e - b);
        ROUTE(1 + b + rep);
      }
    }
#undef ROUTE
  } else {
    /* engine.cpp:198-208: clamp inherited sets at each query's own bound */
    int64_t tmp[1024];
    uint8_t tmpf[1024];
    for (int64_t qi = 0; qi < nq; ++qi) {
      if (idx_count[qi] < 0) continue;
      const int64_t cnt = or_clamp_inherited(c, idx + qi * n, idx_forced + qi * n, idx_count[qi],
                                             routing_visible_len(c, pos[qi]), tmp, tmpf);
      for (int64_t i = 0; i < cnt; ++i) {
        idx[qi * n + i] = tmp[i];
        idx_forced[qi * n + i] = tmpf[i];
      }
      for (int64_t i = cnt; i < n; ++i) idx[qi * n + i] = -1;
      idx_count[qi] = cnt;
    }
  }
  free(scores);
  if (idx_count[0] < 0) return OR_ESTATE;

  /* root attends alone with its own set, no tree rows (engine.cpp:214-227) */
  attend_one(&L, q, pos[0], idx, idx_count[0], NULL, gates, NULL, 0, 0, out);

  /* groups (engine.cpp:229-276) */
  int32_t* adm = (int32_t*)malloc(sizeof(int32_t) * (size_t)(gamma + 1));
  int64_t* uniq = (int64_t*)malloc(sizeof(int64_t) * (size_t)(C * n + 1));
  uint8_t* own = (uint8_t*)malloc((size_t)(C * C * n + 1));
  for (int64_t b = 0; b < gamma; b += C) {
    const int64_t e = b + C < gamma ? b + C : gamma;
    const int64_t size = e - b;
    const int64_t q0 = 1 + b;
    if (!approx) {
      for (int64_t i = 0; i < size; ++i)
        if (idx_count[q0 + i] < 0) { free(adm); free(uniq); free(own); return OR_ESTATE; }
      const int64_t nu = or_merged_schedule(idx + q0 * n, idx_count + q0, size, n, uniq, own);
      for (int64_t i = 0; i < size; ++i) {
        const int64_t qi = q0 + i;
        int64_t na = 0;
        for (int64_t j = 0; j < gamma; ++j)
          if ((tree_mask[(qi - 1) * mask_words + j / 64] >> (j % 64)) & 1ull) adm[na++] = (int32_t)j;
        attend_one(&L, q + qi * qstride, pos[qi], uniq, nu, own + i * nu, gates + qi * Hq * 3,
                   adm, na, 1, out + qi * qstride);
        st->total_requested_loads += idx_count[qi];
        st->window_token_loads += window_rows_attended(c, pos[qi], rows, na);
        if (i > 0 && st->n_pairs < OR_MAX_PAIRS)
          st->pairwise_overlap[st->n_pairs++] = overlap_count(
              idx + (qi - 1) * n, idx_count[qi - 1], idx + qi * n, idx_count[qi]);
      }
      st->unique_block_loads += nu;
      st->dedup_savings += 0; /* recomputed below */
      st->index_constructions += role == OR_ROLE_REUSE ? 0 : size;
    } else {
      const int64_t rep = q0 + or_representative_index(pos + q0, size);
      if (idx_count[rep] < 0) { free(adm); free(uniq); free(own); return OR_ESTATE; }
      for (int64_t i = 0; i < size; ++i) {
        const int64_t qi = q0 + i;
        int64_t na = 0;
        for (int64_t j = 0; j < gamma; ++j)
          if ((tree_mask[(qi - 1) * mask_words + j / 64] >> (j % 64)) & 1ull) adm[na++] = (int32_t)j;
        attend_one(&L, q + qi * qstride, pos[qi], idx + rep * n, idx_count[rep], NULL,
                   gates + qi * Hq * 3, adm, na, 1, out + qi * qstride);
        st->window_token_loads += window_rows_attended(c, pos[qi], rows, na);
      }
      st->unique_block_loads += idx_count[rep];
      st->total_requested_loads += idx_count[rep] * size;
      st->index_constructions += role == OR_ROLE_REUSE ? 0 : 1;
    }
  }
  st->dedup_savings = st->total_requested_loads - st->unique_block_loads;
  free(adm);
  free(uniq);
  free(own);
  return OR_OK;
}
