/*
 * hc_oracle.c -- CPU restatement of the HCache reference restoration path.
 * TEST INFRASTRUCTURE ONLY (see hc_oracle.h). Citations are relative to the
 * reference tree proj/ (read-only at /root/reference in the build container).
 */
#include "hc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* splitmix64: model.cpp:17-31. next() pre-increments the state by the      */
/* golden gamma, so draw i (0-based) mixes seed + (i+1)*gamma.              */
/* ------------------------------------------------------------------------ */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t hco_splitmix64_at(uint64_t seed, uint64_t index) {
  return mix64(seed + (index + 1) * 0x9E3779B97F4A7C15ull);
}

float hco_symmetric_at(uint64_t seed, uint64_t index, float bound) {
  /* model.cpp:27-30: u in [0,1) from the top 53 bits, then (2u-1)*bound in
   * double, rounded to float. */
  double u = (double)(hco_splitmix64_at(seed, index) >> 11) * 0x1p-53;
  return (float)((2.0 * u - 1.0) * (double)bound);
}

void hco_fill_symmetric(float* out, size_t n, uint64_t seed, uint64_t offset,
                        float bound) {
  for (size_t i = 0; i < n; ++i) out[i] = hco_symmetric_at(seed, offset + i, bound);
}

size_t hco_init_model(int n_layers, int d, int d_ffn, int vocab, uint64_t seed,
                      float* out) {
  /* model.cpp:175-194: bound = 1/sqrt(float(d)); draw order embedding, then
   * per layer wq, wk, wv, wo, fc1, fc2 from one stream. */
  size_t dd = (size_t)d * (size_t)d, df = (size_t)d * (size_t)d_ffn;
  size_t total = (size_t)vocab * (size_t)d + (size_t)n_layers * (4 * dd + 2 * df);
  if (!out) return total;
  float bound = 1.0f / sqrtf((float)d);
  hco_fill_symmetric(out, total, seed, 0, bound);
  return total;
}

/* ------------------------------------------------------------------------ */
/* element codecs                                                           */
/* ------------------------------------------------------------------------ */
uint16_t hco_float_to_half(float f) {
  /* fp16.hpp:10-40 */
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t exp = (x >> 23) & 0xFFu;
  uint32_t man = x & 0x7FFFFFu;
  if (exp == 0xFF) return (uint16_t)(sign | 0x7C00u | (man ? 0x200u : 0));
  int e = (int)exp - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7C00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    man |= 0x800000u;
    int shift = 14 - e;
    uint32_t hm = man >> shift;
    uint32_t rem = man & ((1u << shift) - 1);
    uint32_t halfway = 1u << (shift - 1);
    if (rem > halfway || (rem == halfway && (hm & 1))) ++hm;
    return (uint16_t)(sign | hm);
  }
  uint32_t hm = man >> 13;
  uint32_t rem = man & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (hm & 1))) {
    ++hm;
    if (hm == 0x400u) {
      hm = 0;
      ++e;
      if (e >= 31) return (uint16_t)(sign | 0x7C00u);
    }
  }
  return (uint16_t)(sign | ((uint32_t)e << 10) | hm);
}

float hco_half_to_float(uint16_t h) {
  /* fp16.hpp:42-68 */
  uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1Fu;
  uint32_t man = h & 0x3FFu;
  uint32_t x;
  if (exp == 0) {
    if (man == 0) {
      x = sign;
    } else {
      int e = -1;
      do {
        ++e;
        man <<= 1;
      } while (!(man & 0x400u));
      man &= 0x3FFu;
      x = sign | (uint32_t)(127 - 15 - e) << 23 | (man << 13);
    }
  } else if (exp == 31) {
    x = sign | 0x7F800000u | (man << 13);
  } else {
    x = sign | ((exp - 15 + 127) << 23) | (man << 13);
  }
  float f;
  memcpy(&f, &x, 4);
  return f;
}

uint16_t hco_float_to_bf16(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x7FFFFFu))
    return (uint16_t)((x >> 16) | 0x40u); /* quiet NaN */
  uint32_t lsb = (x >> 16) & 1u;
  x += 0x7FFFu + lsb;
  return (uint16_t)(x >> 16);
}

float hco_bf16_to_float(uint16_t h) {
  uint32_t x = (uint32_t)h << 16;
  float f;
  memcpy(&f, &x, 4);
  return f;
}

void hco_round_to_bf16(float* x, size_t n) {
  for (size_t i = 0; i < n; ++i) x[i] = hco_bf16_to_float(hco_float_to_bf16(x[i]));
}

/* ------------------------------------------------------------------------ */
/* tiny pthread parallel-for over [0, n)                                    */
/* ------------------------------------------------------------------------ */
typedef void (*range_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t begin, end;
} range_job;

static void* range_thunk(void* p) {
  range_job* j = (range_job*)p;
  j->fn(j->ctx, j->begin, j->end);
  return NULL;
}

static void parallel_for(int64_t n, int nthreads, range_fn fn, void* ctx) {
  if (nthreads <= 1 || n < 2) {
    fn(ctx, 0, n);
    return;
  }
  if (nthreads > 256) nthreads = 256;
  if (nthreads > n) nthreads = (int)n;
  pthread_t th[256];
  range_job jobs[256];
  int64_t per = (n + nthreads - 1) / nthreads;
  int launched = 0;
  for (int t = 0; t < nthreads; ++t) {
    int64_t b = (int64_t)t * per, e = b + per;
    if (b >= n) break;
    if (e > n) e = n;
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].begin = b;
    jobs[t].end = e;
    if (pthread_create(&th[t], NULL, range_thunk, &jobs[t]) != 0) {
      fn(ctx, b, e); /* fall back to inline */
      jobs[t].fn = NULL;
    }
    launched = t + 1;
  }
  for (int t = 0; t < launched; ++t)
    if (jobs[t].fn) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------------ */
/* layer_norm: model.cpp:43-61                                              */
/* ------------------------------------------------------------------------ */
void hco_layer_norm(const float* x, int64_t rows, int cols, float* out) {
  for (int64_t i = 0; i < rows; ++i) {
    const float* r = x + i * cols;
    double mean = 0.0;
    for (int c = 0; c < cols; ++c) mean += r[c];
    mean /= (double)cols;
    double var = 0.0;
    for (int c = 0; c < cols; ++c) {
      double d = r[c] - mean;
      var += d * d;
    }
    var /= (double)cols;
    float inv = 1.0f / sqrtf((float)var + 1e-5f);
    float* o = out + i * cols;
    for (int c = 0; c < cols; ++c) o[c] = (r[c] - (float)mean) * inv;
  }
}

/* ------------------------------------------------------------------------ */
/* matmul_wt: matrix.cpp:8-21                                               */
/* ------------------------------------------------------------------------ */
typedef struct {
  const float* x;
  const float* w;
  float* y;
  int k, out;
} mm_ctx;

static void mm_rows(void* p, int64_t b, int64_t e) {
  mm_ctx* c = (mm_ctx*)p;
  for (int64_t i = b; i < e; ++i) {
    const float* xi = c->x + i * c->k;
    float* yi = c->y + i * c->out;
    for (int o = 0; o < c->out; ++o) {
      const float* wo = c->w + (size_t)o * c->k;
      float acc = 0.0f;
      for (int kk = 0; kk < c->k; ++kk) acc += xi[kk] * wo[kk];
      yi[o] = acc;
    }
  }
}

void hco_matmul_wt(const float* x, int64_t m, int k, const float* w, int out,
                   float* y, int nthreads) {
  mm_ctx c = {x, w, y, k, out};
  parallel_for(m, nthreads, mm_rows, &c);
}

/* ------------------------------------------------------------------------ */
/* apply_rope: model.cpp:196-217                                            */
/* ------------------------------------------------------------------------ */
void hco_apply_rope(float* x, int64_t rows, int cols, int n_heads, int start_pos) {
  int d_head = cols / n_heads;
  for (int64_t i = 0; i < rows; ++i) {
    float* r = x + i * cols;
    double pos = (double)(start_pos + i);
    for (int h = 0; h < n_heads; ++h) {
      float* hr = r + h * d_head;
      for (int t = 0; t < d_head / 2; ++t) {
        double freq = pow(10000.0, -2.0 * (double)t / (double)d_head);
        float c = (float)cos(pos * freq);
        float s = (float)sin(pos * freq);
        float a = hr[2 * t];
        float b = hr[2 * t + 1];
        hr[2 * t] = a * c - b * s;
        hr[2 * t + 1] = a * s + b * c;
      }
    }
  }
}

void hco_rope_table(int n_pos, int d_head, float* cos_out, float* sin_out) {
  int half = d_head / 2;
  for (int p = 0; p < n_pos; ++p) {
    double pos = (double)p;
    for (int t = 0; t < half; ++t) {
      double freq = pow(10000.0, -2.0 * (double)t / (double)d_head);
      cos_out[(size_t)p * half + t] = (float)cos(pos * freq);
      sin_out[(size_t)p * half + t] = (float)sin(pos * freq);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* project_hidden_to_kv: model.cpp:219-235                                  */
/* ------------------------------------------------------------------------ */
void hco_project_hidden_to_kv(const float* h, int64_t n, int d, const float* wk,
                              const float* wv, int d_kv, int n_kv_heads,
                              int start_pos, int norm_enabled, int rope_enabled,
                              float* k_out, float* v_out, int nthreads) {
  const float* a = h;
  float* tmp = NULL;
  if (norm_enabled) {
    tmp = (float*)malloc(sizeof(float) * (size_t)n * d);
    hco_layer_norm(h, n, d, tmp);
    a = tmp;
  }
  hco_matmul_wt(a, n, d, wk, d_kv, k_out, nthreads);
  hco_matmul_wt(a, n, d, wv, d_kv, v_out, nthreads);
  if (rope_enabled) hco_apply_rope(k_out, n, d_kv, n_kv_heads, start_pos);
  free(tmp);
}

/* ------------------------------------------------------------------------ */
/* full transformer: model.cpp:38-40 (gelu), 237-356                         */
/* ------------------------------------------------------------------------ */
typedef struct {
  const float *embedding, *wq, *wk, *wv, *wo, *fc1, *fc2;
} layer_view;

static layer_view view_layer(const hco_config* cfg, const float* weights, int L) {
  size_t d = (size_t)cfg->d_hidden, dd = d * d, df = d * (size_t)cfg->d_ffn;
  layer_view v;
  v.embedding = weights;
  const float* base = weights + (size_t)cfg->vocab_size * d + (size_t)L * (4 * dd + 2 * df);
  v.wq = base;
  v.wk = base + dd;
  v.wv = base + 2 * dd;
  v.wo = base + 3 * dd;
  v.fc1 = base + 4 * dd;
  v.fc2 = base + 4 * dd + df;
  return v;
}

typedef struct {
  const float *q, *k, *v;
  float* mix;
  int n, d, dh, n_heads, start_pos;
  float inv_sqrt;
} attn_ctx;

static void attn_rows(void* p, int64_t b, int64_t e) {
  attn_ctx* c = (attn_ctx*)p;
  float* scores = (float*)malloc(sizeof(float) * (size_t)(c->start_pos + c->n + 1));
  for (int64_t i = b; i < e; ++i) {
    int pp = c->start_pos + (int)i;
    for (int head = 0; head < c->n_heads; ++head) {
      const float* qh = c->q + i * c->d + head * c->dh;
      float max_s = -1e30f;
      for (int j = 0; j <= pp; ++j) {
        const float* kh = c->k + (size_t)j * c->d + head * c->dh;
        float s = 0.0f;
        for (int cc = 0; cc < c->dh; ++cc) s += qh[cc] * kh[cc];
        scores[j] = s * c->inv_sqrt;
        max_s = max_s > scores[j] ? max_s : scores[j]; /* std::max(a,b) */
      }
      float denom = 0.0f;
      for (int j = 0; j <= pp; ++j) {
        scores[j] = expf(scores[j] - max_s);
        denom += scores[j];
      }
      float* out = c->mix + i * c->d + head * c->dh;
      for (int j = 0; j <= pp; ++j) {
        float w = scores[j] / denom;
        const float* vh = c->v + (size_t)j * c->d + head * c->dh;
        for (int cc = 0; cc < c->dh; ++cc) out[cc] += w * vh[cc];
      }
    }
  }
  free(scores);
}

static float gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

/* block_forward (model.cpp:102-115) with start_pos 0 and an empty cache, so
 * the layer's cache is exactly the fresh projection. x is updated in place. */
static void block_forward_view(const hco_config* cfg, layer_view lw, float* x, int64_t n,
                               float* k, float* v, int nthreads) {
  int d = cfg->d_hidden, dh = d / cfg->n_heads;
  size_t nd = (size_t)n * d;
  hco_project_hidden_to_kv(x, n, d, lw.wk, lw.wv, d, cfg->n_heads, 0,
                           cfg->norm_enabled, cfg->rope_enabled, k, v, nthreads);
  /* attention_forward (model.cpp:237-288) */
  float* a = (float*)malloc(sizeof(float) * nd);
  if (cfg->norm_enabled) hco_layer_norm(x, n, d, a);
  else memcpy(a, x, sizeof(float) * nd);
  float* q = (float*)malloc(sizeof(float) * nd);
  hco_matmul_wt(a, n, d, lw.wq, d, q, nthreads);
  if (cfg->rope_enabled) hco_apply_rope(q, n, d, cfg->n_heads, 0);
  float* mix = (float*)calloc(nd, sizeof(float));
  attn_ctx ac = {q, k, v, mix, (int)n, d, dh, cfg->n_heads, 0, 1.0f / sqrtf((float)dh)};
  parallel_for(n, nthreads, attn_rows, &ac);
  float* attn = q; /* reuse */
  hco_matmul_wt(mix, n, d, lw.wo, d, attn, nthreads);
  for (size_t i = 0; i < nd; ++i) x[i] += attn[i];
  /* ffn_forward (model.cpp:290-303) */
  if (cfg->norm_enabled) hco_layer_norm(x, n, d, a);
  else memcpy(a, x, sizeof(float) * nd);
  float* h1 = (float*)malloc(sizeof(float) * (size_t)n * cfg->d_ffn);
  hco_matmul_wt(a, n, d, lw.fc1, cfg->d_ffn, h1, nthreads);
  for (size_t i = 0; i < (size_t)n * cfg->d_ffn; ++i) h1[i] = gelu(h1[i]);
  hco_matmul_wt(h1, n, cfg->d_ffn, lw.fc2, d, attn, nthreads);
  for (size_t i = 0; i < nd; ++i) x[i] += attn[i];
  free(h1);
  free(mix);
  free(q);
  free(a);
}

static void block_forward(const hco_config* cfg, const float* weights, int L,
                          float* x, int64_t n, float* k, float* v, int nthreads) {
  block_forward_view(cfg, view_layer(cfg, weights, L), x, n, k, v, nthreads);
}

void hco_block_forward(const hco_config* cfg, const float* wq, const float* wk,
                       const float* wv, const float* wo, const float* fc1,
                       const float* fc2, float* x, int64_t n, float* k_out,
                       float* v_out, int nthreads) {
  layer_view lw = {NULL, wq, wk, wv, wo, fc1, fc2};
  block_forward_view(cfg, lw, x, n, k_out, v_out, nthreads);
}

static void embed(const hco_config* cfg, const float* weights, const int* tokens,
                  int64_t n, float* x) {
  /* model.cpp:82-92 (token range validated by the caller) */
  size_t d = (size_t)cfg->d_hidden;
  for (int64_t i = 0; i < n; ++i)
    memcpy(x + (size_t)i * d, weights + (size_t)tokens[i] * d, sizeof(float) * d);
}

int hco_prefill(const hco_config* cfg, const float* weights, const int* tokens,
                int64_t n, float* layer_inputs, float* k_out, float* v_out,
                float* final_hidden, int nthreads) {
  size_t d = (size_t)cfg->d_hidden, nd = (size_t)n * d;
  float* x = (float*)malloc(sizeof(float) * nd);
  float* kt = (float*)malloc(sizeof(float) * nd);
  float* vt = (float*)malloc(sizeof(float) * nd);
  embed(cfg, weights, tokens, n, x);
  for (int L = 0; L < cfg->n_layers; ++L) {
    if (layer_inputs) memcpy(layer_inputs + (size_t)L * nd, x, sizeof(float) * nd);
    block_forward(cfg, weights, L, x, n, kt, vt, nthreads);
    if (k_out) memcpy(k_out + (size_t)L * nd, kt, sizeof(float) * nd);
    if (v_out) memcpy(v_out + (size_t)L * nd, vt, sizeof(float) * nd);
  }
  if (final_hidden) memcpy(final_hidden, x, sizeof(float) * nd);
  /* argmax_token (model.cpp:67-80) on the last row */
  const float* hid = x + (size_t)(n - 1) * d;
  int best = 0;
  float best_score = -1e30f;
  for (int t = 0; t < cfg->vocab_size; ++t) {
    const float* e = weights + (size_t)t * d;
    float acc = 0.0f;
    for (size_t c = 0; c < d; ++c) acc += e[c] * hid[c];
    if (acc > best_score) {
      best_score = acc;
      best = t;
    }
  }
  free(vt);
  free(kt);
  free(x);
  return best;
}

void hco_prefill_layers(const hco_config* cfg, const float* weights,
                        const int* tokens, int64_t n, int layer_begin,
                        int layer_end, float* k_out, float* v_out, int nthreads) {
  /* model.cpp:349-356: embeds the tokens and runs [lb, le) from that input
   * (the reference feeds the embedding to layer_begin, not layer_begin's true
   * input; restore only ever calls it with lb = 0). */
  size_t d = (size_t)cfg->d_hidden, nd = (size_t)n * d;
  float* x = (float*)malloc(sizeof(float) * nd);
  embed(cfg, weights, tokens, n, x);
  for (int L = layer_begin; L < layer_end; ++L)
    block_forward(cfg, weights, L, x, n, k_out + (size_t)L * nd,
                  v_out + (size_t)L * nd, nthreads);
  free(x);
}

typedef struct {
  float* out;
  uint64_t seed, offset;
  float bound;
} fill_ctx;

static void fill_bf16_range(void* p, int64_t b, int64_t e) {
  fill_ctx* c = (fill_ctx*)p;
  for (int64_t i = b; i < e; ++i)
    c->out[i] = hco_bf16_to_float(
        hco_float_to_bf16(hco_symmetric_at(c->seed, c->offset + (uint64_t)i, c->bound)));
}

void hco_fill_symmetric_bf16(float* out, size_t n, uint64_t seed, uint64_t offset,
                             float bound, int nthreads) {
  fill_ctx c = {out, seed, offset, bound};
  parallel_for((int64_t)n, nthreads, fill_bf16_range, &c);
}

/* ------------------------------------------------------------------------ */
/* chunk indexing: storage.hpp:20; storage.cpp:29-31                        */
/* ------------------------------------------------------------------------ */
int hco_chunk_tokens(void) { return 64; }
int hco_device_for_chunk(int layer, int chunk_idx, int device_count) {
  return (layer + chunk_idx) % device_count;
}
int hco_num_chunks(int n_tokens) { return (n_tokens + 63) / 64; }

/* ------------------------------------------------------------------------ */
/* planner: planner.cpp:34-51 (make), 75-90 (plan), 92-107, 109-128         */
/* ------------------------------------------------------------------------ */
static int valid_timings(const hco_timings* t) {
  return t->io_h > 0 && t->io_kv > 0 && t->c_h > 0 && t->c_token > 0 && t->n_layers >= 1;
}

static void plan_make(int n, int l_h, int comp, hco_plan* p) {
  p->l_h = l_h;
  p->l_o = n - l_h;
  p->complement = p->l_o == 0 ? 0 : comp;
}

int hco_plan_closed_form(const hco_timings* t, hco_plan* out) {
  if (!valid_timings(t)) return -1;
  int n = t->n_layers, comp;
  double lh_real;
  if (t->c_h > t->io_h) {
    comp = 1;
    lh_real = (double)n * t->io_kv / (t->io_kv + t->c_h - t->io_h);
  } else {
    comp = 2;
    lh_real = (double)n * t->c_token / (t->c_token + t->io_h - t->c_h);
  }
  int l_h = (int)ceil(lh_real - 1e-12);
  if (l_h < 0) l_h = 0;
  if (l_h > n) l_h = n;
  plan_make(n, l_h, comp, out);
  return 0;
}

double hco_makespan(const hco_plan* p, const hco_timings* t) {
  double lh = (double)p->l_h, lo = (double)p->l_o;
  double a, b;
  switch (p->complement) {
    case 0:
      a = t->c_h * lh;
      b = t->io_h * lh;
      return a > b ? a : b;
    case 1:
      a = t->c_h * lh;
      b = t->io_h * lh + t->io_kv * lo;
      return a > b ? a : b;
    default:
      a = t->io_h * lh;
      b = t->c_token * lo + t->c_h * lh;
      return a > b ? a : b;
  }
}

int hco_brute_force_plan(const hco_timings* t, hco_plan* out) {
  if (!valid_timings(t)) return -1;
  int have = 0;
  double best_cost = 0;
  for (int lh = 0; lh <= t->n_layers; ++lh) {
    for (int ci = 0; ci < 2; ++ci) {
      hco_plan cand;
      plan_make(t->n_layers, lh, ci == 0 ? 1 : 2, &cand);
      double cost = hco_makespan(&cand, t);
      if (!have || cost < best_cost || (cost == best_cost && cand.l_h > out->l_h)) {
        *out = cand;
        best_cost = cost;
        have = 1;
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* simulate_pipeline: pipeline.cpp:33-104                                   */
/* ------------------------------------------------------------------------ */
int hco_simulate_pipeline(const hco_job* jobs, int n_jobs, int prefetch_depth,
                          hco_event* events, double* total_s, double* fill_s) {
  if (prefetch_depth < 1) return -1;
  int* io_order = (int*)malloc(sizeof(int) * (n_jobs + 1));
  int* staged_order = (int*)malloc(sizeof(int) * (n_jobs + 1));
  int* staged_rank = (int*)malloc(sizeof(int) * (n_jobs + 1));
  double* fetch_end = (double*)calloc(n_jobs + 1, sizeof(double));
  double* compute_end = (double*)calloc(n_jobs + 1, sizeof(double));
  int* computed = (int*)calloc(n_jobs + 1, sizeof(int));
  int n_io = 0, n_staged = 0, n_ev = 0;
  for (int j = 0; j < n_jobs; ++j)
    if (jobs[j].has_io) io_order[n_io++] = j;
  for (int r = 0; r < n_io; ++r)
    if (jobs[io_order[r]].has_compute) staged_order[n_staged++] = io_order[r];
  for (int j = 0; j < n_jobs; ++j) staged_rank[j] = -1;
  for (int r = 0; r < n_staged; ++r) staged_rank[staged_order[r]] = r;
  double io_free = 0, compute_free = 0, fill = 0;
  int next_io = 0;
  for (int j = 0; j <= n_jobs; ++j) {
    /* issue_ready_fetches (pipeline.cpp:62-82), then compute job j */
    while (next_io < n_io) {
      int jj = io_order[next_io];
      double dep = 0;
      if (jobs[jj].has_compute) {
        int r = staged_rank[jj];
        if (r >= prefetch_depth + 1) {
          int blocker = staged_order[r - prefetch_depth - 1];
          if (!computed[blocker]) break;
          dep = compute_end[blocker];
        }
      }
      double start = io_free > dep ? io_free : dep;
      double end = start + jobs[jj].io_s;
      events[n_ev].lane = 0;
      events[n_ev].layer = jobs[jj].layer;
      events[n_ev].job = jj;
      events[n_ev].start_s = start;
      events[n_ev].end_s = end;
      ++n_ev;
      fetch_end[jj] = end;
      io_free = end;
      if (n_ev == 1) fill = end;
      ++next_io;
    }
    if (j == n_jobs) break;
    if (!jobs[j].has_compute) continue;
    double ready = jobs[j].has_io ? fetch_end[j] : 0.0;
    double start = compute_free > ready ? compute_free : ready;
    double end = start + jobs[j].compute_s;
    events[n_ev].lane = 1;
    events[n_ev].layer = jobs[j].layer;
    events[n_ev].job = j;
    events[n_ev].start_s = start;
    events[n_ev].end_s = end;
    ++n_ev;
    compute_end[j] = end;
    computed[j] = 1;
    compute_free = end;
  }
  int ok = next_io == n_io;
  double total = 0;
  for (int e = 0; e < n_ev; ++e)
    if (events[e].end_s > total) total = events[e].end_s;
  /* std::stable_sort by start_s (pipeline.cpp:100-103): insertion sort. */
  for (int a = 1; a < n_ev; ++a) {
    hco_event key = events[a];
    int b = a - 1;
    while (b >= 0 && key.start_s < events[b].start_s) {
      events[b + 1] = events[b];
      --b;
    }
    events[b + 1] = key;
  }
  *total_s = total;
  *fill_s = fill;
  free(io_order);
  free(staged_order);
  free(staged_rank);
  free(fetch_end);
  free(compute_end);
  free(computed);
  return ok ? n_ev : -2;
}

/* ------------------------------------------------------------------------ */
/* trace lengths: trace.cpp:11-39 (Rng), 54-100 (gen_trace Conversation)     */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t s;
} trace_rng;

static uint64_t trng_next(trace_rng* r) {
  uint64_t z = (r->s += 0x9E3779B97F4A7C15ull);
  return mix64(z);
}
static double trng_uniform(trace_rng* r) { return (double)(trng_next(r) >> 11) * 0x1p-53; }
static int trng_geometric(trace_rng* r, double mean) {
  double p = 1.0 / (mean > 1.0 ? mean : 1.0);
  double u = trng_uniform(r);
  if (u < 1e-300) u = 1e-300;
  return 1 + (int)floor(log(u) / log(1.0 - p));
}
static double trng_exponential(trace_rng* r, double rate) {
  double u = trng_uniform(r);
  if (u < 1e-300) u = 1e-300;
  return -log(u) / rate;
}

int hco_conversation_history(int n_sessions, int rounds, double mean_input,
                             double mean_output, double arrival_rate, int vocab,
                             uint64_t seed, int* history_out) {
  (void)vocab;
  trace_rng r = {seed ^ 0xA5A5A5A5DEADBEEFull};
  int k = 0;
  for (int s = 0; s < n_sessions; ++s) {
    (void)trng_exponential(&r, arrival_rate);
    int history = 0;
    for (int rd = 1; rd <= rounds; ++rd) {
      history_out[k++] = history;
      int n_prompt = trng_geometric(&r, mean_input);
      for (int t = 0; t < n_prompt; ++t) (void)trng_next(&r); /* prompt token ids */
      int budget = trng_geometric(&r, mean_output);
      history += n_prompt + budget;
    }
  }
  return k;
}

uint64_t hco_fnv1a(const void* data, size_t n) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}
