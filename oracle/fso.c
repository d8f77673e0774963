/*
 * fso.c — plain, slow, obviously-correct CPU oracle of the decoder math on the
 * FlowSpec tree-verification path.  TEST INFRASTRUCTURE ONLY (see fso.h).
 *
 * Arithmetic is fp64 throughout; values are rounded only where the precision
 * contract stores them:
 *   residual x ............ fp32
 *   q, k, v (after bias+RoPE) bf16 (K/V cache storage)
 *   RMSNorm output, attention output, silu(g)*u (the GEMM inputs): fp32
 *   logits ................ fp32
 * i.e. the bf16 branch differs from the fp32 one only in the weights and in
 * the q/k/v storage; every other step is the plain definition (RMSNorm
 * y = x*inv*g, then the linear layer), pinned against HF transformers in
 * tests/test_oracle_decoder.py (fp32, and bf16 with the same storage points).
 * (fp32 config: fp32 everywhere)
 * Compile with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 *
 * Paper passages followed:
 *   decoder structure ..... PAPER.md:721 (App. B.1): embedding, decoder layers
 *                           of self-attention + FFN + residual, classification head
 *   tree attention ........ PAPER.md:248 (§3.1): each segment carries tree
 *                           position IDs and a tree attention mask; here the mask
 *                           is given explicitly as a per-row visibility list
 *   KV cache pruning ...... PAPER.md:342-347 (§3.3)
 * Model hyper-parameters (RMSNorm eps, rotate-half RoPE, SwiGLU, optional
 * q/k/v bias) follow the public LLaMA2/Qwen2 definitions the paper names
 * — DESIGN.md reading R19.
 */
#include "fso.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- generator */
/* SURVEY.md §8(d) "Generators": splitmix64 finalizer */
uint64_t fso_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

float fso_round_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan: truncate, keep quiet nan */
    if (u & 0x007fffffu) u |= 0x00400000u;
    u &= 0xffff0000u;
  } else {
    u += 0x7fffu + ((u >> 16) & 1u); /* round to nearest even */
    u &= 0xffff0000u;
  }
  memcpy(&x, &u, 4);
  return x;
}

static uint64_t tensor_key(uint64_t seed, uint64_t tid) {
  return fso_mix64(seed ^ (tid * 0xD1B54A32D192ED03ull));
}

/* u = h>>40 (24 bits); i = 2u-(2^24-1) odd, exact in fp32; x = RN32(i*c) */
static float gen_from_key(uint64_t key, uint64_t e, float c, int32_t gain,
                          int32_t bf16) {
  uint64_t h = fso_mix64(key ^ e);
  int32_t u = (int32_t)(h >> 40);
  int32_t i = 2 * u - 16777215;
  float x = (float)i * c;
  if (gain) x = 1.0f + x;
  return bf16 ? fso_round_bf16(x) : x;
}

static float gen_scale(double sigma, int32_t gain) {
  /* centred: U(+-sigma*sqrt3) has std sigma; gain: 1 + U(+-0.1) */
  return gain ? (float)(0.1 / 16777216.0) : (float)(sigma * sqrt(3.0) / 16777216.0);
}

float fso_gen_value(uint64_t seed, uint64_t tid, uint64_t e, double sigma,
                    int32_t gain, int32_t bf16) {
  return gen_from_key(tensor_key(seed, tid), e, gen_scale(sigma, gain), gain, bf16);
}

/* ------------------------------------------------------------------- model */
struct fso_model {
  fso_cfg c;
  int32_t n_tensors_per_layer;
  void** cache; /* [(L+1) * 32] lazily materialised tensors (uint16 bf16 or float) */
};

static int64_t t_rows(const fso_cfg* c, int32_t which) {
  switch (which) {
    case FSO_Q: return (int64_t)c->n_heads * c->head_dim;
    case FSO_K: case FSO_V: return (int64_t)c->n_kv_heads * c->head_dim;
    case FSO_O: return c->d_model;
    case FSO_GATE: case FSO_UP: return c->ffn;
    case FSO_DOWN: return c->d_model;
    case FSO_ATTN_NORM: case FSO_MLP_NORM: case FSO_FINAL_NORM: return 1;
    case FSO_BQ: return 1;
    case FSO_BK: case FSO_BV: return 1;
    case FSO_EMBED: case FSO_HEAD: return c->vocab;
  }
  return -1;
}
static int64_t t_cols(const fso_cfg* c, int32_t which) {
  switch (which) {
    case FSO_Q: case FSO_K: case FSO_V: return c->d_model;
    case FSO_O: return (int64_t)c->n_heads * c->head_dim;
    case FSO_GATE: case FSO_UP: return c->d_model;
    case FSO_DOWN: return c->ffn;
    case FSO_ATTN_NORM: case FSO_MLP_NORM: case FSO_FINAL_NORM: return c->d_model;
    case FSO_BQ: return (int64_t)c->n_heads * c->head_dim;
    case FSO_BK: case FSO_BV: return (int64_t)c->n_kv_heads * c->head_dim;
    case FSO_EMBED: case FSO_HEAD: return c->d_model;
  }
  return -1;
}
static uint64_t t_id(int32_t layer, int32_t which) {
  if (which == FSO_EMBED) return 0xFFFF0ull;
  if (which == FSO_HEAD) return 0xFFFF1ull;
  if (which == FSO_FINAL_NORM) return 0xFFFF2ull;
  return (uint64_t)layer * 16ull + (uint64_t)which;
}
/* SURVEY §8(d) "Scales" */
static double t_sigma(const fso_cfg* c, int32_t which) {
  switch (which) {
    case FSO_O: case FSO_DOWN: return 0.02 / sqrt(2.0 * c->n_layers);
    case FSO_HEAD: return 2.0 / sqrt((double)c->d_model);
    default: return 0.02;
  }
}
static int32_t t_gain(int32_t which) {
  return which == FSO_ATTN_NORM || which == FSO_MLP_NORM || which == FSO_FINAL_NORM;
}

fso_model* fso_model_create(const fso_cfg* cfg) {
  if (!cfg || cfg->n_layers < 1 || cfg->d_model < 1 || cfg->n_heads < 1 ||
      cfg->n_kv_heads < 1 || cfg->n_heads % cfg->n_kv_heads || cfg->head_dim < 2 ||
      (cfg->head_dim & 1) || cfg->ffn < 1 || cfg->vocab < 2)
    return NULL;
  fso_model* m = (fso_model*)calloc(1, sizeof(fso_model));
  m->c = *cfg;
  m->cache = (void**)calloc((size_t)(cfg->n_layers + 1) * 32, sizeof(void*));
  return m;
}

void fso_model_free(fso_model* m) {
  if (!m) return;
  for (int64_t i = 0; i < (int64_t)(m->c.n_layers + 1) * 32; i++) free(m->cache[i]);
  free(m->cache);
  free(m);
}

int64_t fso_tensor_numel(const fso_model* m, int32_t which) {
  return t_rows(&m->c, which) * t_cols(&m->c, which);
}

/* one row of a weight tensor as floats (generated, or read from the cache) */
static void get_row(fso_model* m, int32_t layer, int32_t which, int64_t row,
                    float* out);

static void** cache_slot(fso_model* m, int32_t layer, int32_t which) {
  int32_t l = (which >= FSO_EMBED) ? m->c.n_layers : layer;
  return &m->cache[(int64_t)l * 32 + which];
}

static void materialise(fso_model* m, int32_t layer, int32_t which) {
  void** slot = cache_slot(m, layer, which);
  if (*slot) return;
  int64_t R = t_rows(&m->c, which), C = t_cols(&m->c, which);
  uint64_t key = tensor_key(m->c.seed, t_id(layer, which));
  float cs = gen_scale(t_sigma(&m->c, which), t_gain(which));
  int32_t gain = t_gain(which);
  if (m->c.bf16) {
    uint16_t* p = (uint16_t*)malloc((size_t)(R * C) * 2);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < R; r++)
      for (int64_t k = 0; k < C; k++) {
        float v = gen_from_key(key, (uint64_t)(r * C + k), cs, gain, 1);
        uint32_t u;
        memcpy(&u, &v, 4);
        p[r * C + k] = (uint16_t)(u >> 16);
      }
    *slot = p;
  } else {
    float* p = (float*)malloc((size_t)(R * C) * 4);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < R; r++)
      for (int64_t k = 0; k < C; k++)
        p[r * C + k] = gen_from_key(key, (uint64_t)(r * C + k), cs, gain, 0);
    *slot = p;
  }
}

static void get_row(fso_model* m, int32_t layer, int32_t which, int64_t row,
                    float* out) {
  int64_t C = t_cols(&m->c, which);
  void* cached = *cache_slot(m, layer, which);
  if (cached) {
    if (m->c.bf16) {
      const uint16_t* p = (const uint16_t*)cached + row * C;
      for (int64_t k = 0; k < C; k++) {
        uint32_t u = (uint32_t)p[k] << 16;
        memcpy(&out[k], &u, 4);
      }
    } else {
      memcpy(out, (const float*)cached + row * C, (size_t)C * 4);
    }
    return;
  }
  uint64_t key = tensor_key(m->c.seed, t_id(layer, which));
  float cs = gen_scale(t_sigma(&m->c, which), t_gain(which));
  for (int64_t k = 0; k < C; k++)
    out[k] = gen_from_key(key, (uint64_t)(row * C + k), cs, t_gain(which), m->c.bf16);
}

int32_t fso_gen_tensor(fso_model* m, int32_t layer, int32_t which, float* out) {
  int64_t R = t_rows(&m->c, which), C = t_cols(&m->c, which);
  if (R < 0 || layer < 0 || layer >= m->c.n_layers) return -1;
  if (which == FSO_BQ || which == FSO_BK || which == FSO_BV) {
    if (!m->c.qkv_bias) return -1;
  }
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; r++) get_row(m, layer, which, r, out + r * C);
  return 0;
}

/* ---------------------------------------------------------------- KV store */
struct fso_kv {
  fso_cfg c;
  int32_t max_slots;
  int32_t bf16;
  void* data; /* [layer][which][kvh][slot][head_dim] */
};

static int64_t kv_index(const fso_kv* kv, int32_t layer, int32_t which,
                        int32_t kvh, int32_t slot) {
  return ((((int64_t)layer * 2 + which) * kv->c.n_kv_heads + kvh) * kv->max_slots + slot) *
         kv->c.head_dim;
}

fso_kv* fso_kv_create(const fso_model* m, int32_t max_slots) {
  if (!m || max_slots < 1) return NULL;
  fso_kv* kv = (fso_kv*)calloc(1, sizeof(fso_kv));
  kv->c = m->c;
  kv->max_slots = max_slots;
  kv->bf16 = m->c.bf16;
  size_t n = (size_t)m->c.n_layers * 2 * m->c.n_kv_heads * (size_t)max_slots * m->c.head_dim;
  kv->data = calloc(n, kv->bf16 ? 2 : 4);
  if (!kv->data) { free(kv); return NULL; }
  return kv;
}

void fso_kv_free(fso_kv* kv) {
  if (!kv) return;
  free(kv->data);
  free(kv);
}

static double kv_load(const fso_kv* kv, int64_t idx) {
  if (kv->bf16) {
    uint32_t u = (uint32_t)((const uint16_t*)kv->data)[idx] << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
  }
  return ((const float*)kv->data)[idx];
}

static void kv_store(fso_kv* kv, int64_t idx, float v) {
  if (kv->bf16) {
    float r = fso_round_bf16(v);
    uint32_t u;
    memcpy(&u, &r, 4);
    ((uint16_t*)kv->data)[idx] = (uint16_t)(u >> 16);
  } else {
    ((float*)kv->data)[idx] = v;
  }
}

int32_t fso_kv_get(const fso_kv* kv, int32_t layer, int32_t which, int32_t kvh,
                   int32_t slot, float* out) {
  if (layer < 0 || layer >= kv->c.n_layers || which < 0 || which > 1 || kvh < 0 ||
      kvh >= kv->c.n_kv_heads || slot < 0 || slot >= kv->max_slots)
    return -1;
  int64_t b = kv_index(kv, layer, which, kvh, slot);
  for (int32_t j = 0; j < kv->c.head_dim; j++) out[j] = (float)kv_load(kv, b + j);
  return 0;
}

int32_t fso_kv_move(fso_kv* kv, int32_t layer_begin, int32_t layer_end,
                    const int32_t* from, const int32_t* to, int32_t n) {
  if (layer_begin < 0 || layer_end > kv->c.n_layers || layer_begin > layer_end) return -1;
  for (int32_t i = 0; i < n; i++)
    if (from[i] < 0 || from[i] >= kv->max_slots || to[i] < 0 || to[i] >= kv->max_slots)
      return -1;
  int32_t hd = kv->c.head_dim;
  size_t es = kv->bf16 ? 2 : 4;
  unsigned char* tmp = (unsigned char*)malloc((size_t)n * hd * es + 1);
  for (int32_t l = layer_begin; l < layer_end; l++)
    for (int32_t w = 0; w < 2; w++)
      for (int32_t h = 0; h < kv->c.n_kv_heads; h++) {
        for (int32_t i = 0; i < n; i++) /* all reads first ... */
          memcpy(tmp + (size_t)i * hd * es,
                 (unsigned char*)kv->data + (size_t)kv_index(kv, l, w, h, from[i]) * es,
                 (size_t)hd * es);
        for (int32_t i = 0; i < n; i++) /* ... then all writes */
          memcpy((unsigned char*)kv->data + (size_t)kv_index(kv, l, w, h, to[i]) * es,
                 tmp + (size_t)i * hd * es, (size_t)hd * es);
      }
  free(tmp);
  return 0;
}

int32_t fso_kv_synth(fso_kv* kv, int32_t n, uint64_t kv_seed) {
  if (n < 0 || n > kv->max_slots) return -1;
  int32_t hd = kv->c.head_dim;
  float cs = gen_scale(1.0, 0);
#pragma omp parallel for collapse(2) schedule(static)
  for (int32_t l = 0; l < kv->c.n_layers; l++)
    for (int32_t w = 0; w < 2; w++) {
      uint64_t key = tensor_key(kv_seed, 0x200000ull + (uint64_t)l * 2ull + (uint64_t)w);
      for (int32_t h = 0; h < kv->c.n_kv_heads; h++)
        for (int32_t s = 0; s < n; s++)
          for (int32_t j = 0; j < hd; j++) {
            uint64_t e = (((uint64_t)h << 32) + (uint64_t)s) * (uint64_t)hd + (uint64_t)j;
            kv_store(kv, kv_index(kv, l, w, h, s) + j, gen_from_key(key, e, cs, 0, kv->bf16));
          }
    }
  return 0;
}

/* ----------------------------------------------------------------- forward */
static float store_act(const fso_cfg* c, double v) {
  /* q/k/v storage: fp32, then bf16 under the bf16 contract */
  float f = (float)v;
  return c->bf16 ? fso_round_bf16(f) : f;
}

/* GEMM-input activations (RMSNorm outputs, attention output, silu*up) are
 * stored as fp32 under both contracts (R18) */
static double store_f32(double v) { return (double)(float)v; }

/* Mutation switch for the pin tests only (tests/test_oracle_decoder.py):
 * each value removes one term so the test can show its pin notices. 0 = off. */
static int32_t g_mutant = 0;
void fso_set_mutant(int32_t which) { g_mutant = which; }

/* RMSNorm (LLaMA, PAPER.md:721 decoder layer; HF LlamaRMSNorm):
 *   y = x * inv * g,  inv = 1/sqrt(mean(x^2) + eps), stored as fp32. */
static void rmsnorm(fso_model* m, int32_t layer, int32_t which, int32_t n_rows,
                    const float* x, double* y) {
  const fso_cfg* c = &m->c;
  int32_t d = c->d_model;
  float* g = (float*)malloc((size_t)d * 4);
  get_row(m, layer, which, 0, g);
  for (int32_t r = 0; r < n_rows; r++) {
    double ss = 0.0;
    for (int32_t k = 0; k < d; k++) ss += (double)x[(int64_t)r * d + k] * (double)x[(int64_t)r * d + k];
    double inv = 1.0 / sqrt(ss / d + c->rms_eps);
    if (g_mutant == 1 && which == FSO_FINAL_NORM) inv = 1.0;   /* mutant: no inv on the head */
    if (g_mutant == 2 && which == FSO_ATTN_NORM) inv = 1.0;    /* mutant: no inv before QKV */
    for (int32_t k = 0; k < d; k++)
      y[(int64_t)r * d + k] = store_f32((double)x[(int64_t)r * d + k] * inv * (double)g[k]);
  }
  free(g);
}

/* out[m][r] = sum_k W[r][k] * in[m][k]  (fp64 accumulation, k ascending) */
static void linear(fso_model* m, int32_t layer, int32_t which, int32_t n_rows,
                   const double* in, double* out) {
  int64_t R = t_rows(&m->c, which), C = t_cols(&m->c, which);
#pragma omp parallel
  {
    float* w = (float*)malloc((size_t)C * 4);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < R; r++) {
      get_row(m, layer, which, r, w);
      for (int32_t i = 0; i < n_rows; i++) {
        const double* a = in + (int64_t)i * C;
        double s = 0.0;
        for (int64_t k = 0; k < C; k++) s += (double)w[k] * a[k];
        out[(int64_t)i * R + r] = s;
      }
    }
    free(w);
  }
}

/* HF rotate-half RoPE: (a, b) = (x[i], x[i+hd/2]) ->
 *   (a cos - b sin, b cos + a sin), angle = pos * theta^(-2i/hd) in fp64,
 *   cos/sin rounded to fp32 (precision contract). */
static void rope(const fso_cfg* c, double* v, int32_t pos) {
  int32_t half = c->head_dim / 2;
  for (int32_t i = 0; i < half; i++) {
    double ang = (double)pos * pow(c->rope_theta, -2.0 * i / c->head_dim);
    double cs = (double)(float)cos(ang), sn = (double)(float)sin(ang);
    double a = v[i], b = v[i + half];
    v[i] = a * cs - b * sn;
    v[i + half] = b * cs + a * sn;
  }
}

int32_t fso_forward(fso_model* m, fso_kv* kv, int32_t layer_begin, int32_t layer_end,
                    int32_t n_rows, const int32_t* tokens, const int32_t* pos,
                    const int32_t* slot, const int32_t* vis_off,
                    const int32_t* vis_slot, const float* h_in, float* h_out,
                    float* logits) {
  const fso_cfg* c = &m->c;
  if (n_rows < 1 || layer_begin < 0 || layer_end > c->n_layers || layer_begin > layer_end)
    return -1;
  if (layer_begin == 0 && !tokens) return -1;
  if (layer_begin > 0 && !h_in) return -1;
  if (layer_end > layer_begin && (!kv || !slot || !vis_off || !vis_slot || !pos)) return -1;
  for (int32_t r = 0; r < n_rows; r++) {
    if (layer_begin == 0 && (tokens[r] < 0 || tokens[r] >= c->vocab)) return -1;
    if (layer_end > layer_begin) {
      if (slot[r] < 0 || slot[r] >= kv->max_slots) return -1;
      for (int32_t j = vis_off[r]; j < vis_off[r + 1]; j++)
        if (vis_slot[j] < 0 || vis_slot[j] >= kv->max_slots) return -1;
    }
  }
  const int32_t d = c->d_model, H = c->n_heads, Hkv = c->n_kv_heads, hd = c->head_dim;
  const int32_t G = H / Hkv;
  const int64_t nq = (int64_t)H * hd, nkv = (int64_t)Hkv * hd;

  float* x = (float*)malloc((size_t)n_rows * d * 4); /* fp32 residual */
  if (layer_begin == 0) {
    float* row = (float*)malloc((size_t)d * 4);
    for (int32_t r = 0; r < n_rows; r++) {
      get_row(m, 0, FSO_EMBED, tokens[r], row);
      memcpy(x + (int64_t)r * d, row, (size_t)d * 4);
    }
    free(row);
  } else {
    memcpy(x, h_in, (size_t)n_rows * d * 4);
  }

  int64_t wmax = nq > c->ffn ? nq : c->ffn;
  if (wmax < d) wmax = d;
  double* y = (double*)malloc((size_t)n_rows * d * 8);
  double* q = (double*)malloc((size_t)n_rows * nq * 8);
  double* kk = (double*)malloc((size_t)n_rows * nkv * 8);
  double* vv = (double*)malloc((size_t)n_rows * nkv * 8);
  double* att = (double*)malloc((size_t)n_rows * nq * 8);
  double* g = (double*)malloc((size_t)n_rows * c->ffn * 8);
  double* u = (double*)malloc((size_t)n_rows * c->ffn * 8);
  double* o = (double*)malloc((size_t)n_rows * wmax * 8);
  float* bias = (float*)malloc((size_t)nq * 4);

  for (int32_t l = layer_begin; l < layer_end; l++) {
    /* --- self-attention block --- */
    rmsnorm(m, l, FSO_ATTN_NORM, n_rows, x, y);
    linear(m, l, FSO_Q, n_rows, y, q);
    linear(m, l, FSO_K, n_rows, y, kk);
    linear(m, l, FSO_V, n_rows, y, vv);
    if (c->qkv_bias) {
      get_row(m, l, FSO_BQ, 0, bias);
      for (int32_t r = 0; r < n_rows; r++)
        for (int64_t j = 0; j < nq; j++) q[r * nq + j] += bias[j];
      get_row(m, l, FSO_BK, 0, bias);
      for (int32_t r = 0; r < n_rows; r++)
        for (int64_t j = 0; j < nkv; j++) kk[r * nkv + j] += bias[j];
      get_row(m, l, FSO_BV, 0, bias);
      for (int32_t r = 0; r < n_rows; r++)
        for (int64_t j = 0; j < nkv; j++) vv[r * nkv + j] += bias[j];
    }
    for (int32_t r = 0; r < n_rows; r++) {
      for (int32_t h = 0; h < H; h++) {
        rope(c, q + r * nq + (int64_t)h * hd, pos[r]);
        for (int32_t j = 0; j < hd; j++)
          q[r * nq + (int64_t)h * hd + j] = store_act(c, q[r * nq + (int64_t)h * hd + j]);
      }
      for (int32_t h = 0; h < Hkv; h++) {
        rope(c, kk + r * nkv + (int64_t)h * hd, pos[r]);
        /* K/V of the rows are written to the cache before attention */
        for (int32_t j = 0; j < hd; j++) {
          kv_store(kv, kv_index(kv, l, 0, h, slot[r]) + j, (float)kk[r * nkv + (int64_t)h * hd + j]);
          kv_store(kv, kv_index(kv, l, 1, h, slot[r]) + j, (float)vv[r * nkv + (int64_t)h * hd + j]);
        }
      }
    }
    const double scale = 1.0 / sqrt((double)hd);
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int32_t r = 0; r < n_rows; r++)
      for (int32_t h = 0; h < H; h++) {
        int32_t kvh = h / G; /* GQA: query head h reads kv head floor(h*Hkv/H) */
        int32_t nv = vis_off[r + 1] - vis_off[r];
        double* s = (double*)malloc((size_t)(nv > 0 ? nv : 1) * 8);
        const double* qh = q + (int64_t)r * nq + (int64_t)h * hd;
        double mx = -INFINITY;
        for (int32_t j = 0; j < nv; j++) {
          int64_t kb = kv_index(kv, l, 0, kvh, vis_slot[vis_off[r] + j]);
          double dot = 0.0;
          for (int32_t t = 0; t < hd; t++) dot += qh[t] * kv_load(kv, kb + t);
          s[j] = dot * scale;
          if (s[j] > mx) mx = s[j];
        }
        double den = 0.0;
        for (int32_t j = 0; j < nv; j++) {
          s[j] = exp(s[j] - mx);
          den += s[j];
        }
        double* oh = att + (int64_t)r * nq + (int64_t)h * hd;
        for (int32_t t = 0; t < hd; t++) oh[t] = 0.0;
        for (int32_t j = 0; j < nv; j++) {
          int64_t vb = kv_index(kv, l, 1, kvh, vis_slot[vis_off[r] + j]);
          double p = s[j] / den;
          for (int32_t t = 0; t < hd; t++) oh[t] += p * kv_load(kv, vb + t);
        }
        for (int32_t t = 0; t < hd; t++) oh[t] = store_f32(oh[t]);
        free(s);
      }
    linear(m, l, FSO_O, n_rows, att, o);
    for (int64_t i = 0; i < (int64_t)n_rows * d; i++) x[i] = (float)((double)x[i] + o[i]);

    /* --- SwiGLU FFN block --- */
    rmsnorm(m, l, FSO_MLP_NORM, n_rows, x, y);
    linear(m, l, FSO_GATE, n_rows, y, g);
    linear(m, l, FSO_UP, n_rows, y, u);
    for (int64_t i = 0; i < (int64_t)n_rows * c->ffn; i++) {
      double gv = g[i];
      g[i] = store_f32(gv / (1.0 + exp(-gv)) * u[i]);   /* SiLU(g) * u */
    }
    linear(m, l, FSO_DOWN, n_rows, g, o);
    for (int64_t i = 0; i < (int64_t)n_rows * d; i++) x[i] = (float)((double)x[i] + o[i]);
  }

  if (h_out) memcpy(h_out, x, (size_t)n_rows * d * 4);
  if (layer_end == c->n_layers && logits) {
    rmsnorm(m, 0, FSO_FINAL_NORM, n_rows, x, y);
    int64_t V = c->vocab;
    double* lg = (double*)malloc((size_t)n_rows * V * 8);
    linear(m, 0, FSO_HEAD, n_rows, y, lg);
    for (int64_t i = 0; i < (int64_t)n_rows * V; i++) logits[i] = (float)lg[i];
    free(lg);
  }
  free(x); free(y); free(q); free(kk); free(vv); free(att); free(g); free(u); free(o);
  free(bias);
  return 0;
}

/* materialise all weights up front when cache_weights is set */
int32_t fso_model_materialise(fso_model* m) {
  if (!m->c.cache_weights) return 0;
  for (int32_t l = 0; l < m->c.n_layers; l++)
    for (int32_t w = 0; w <= FSO_BV; w++) {
      if ((w == FSO_BQ || w == FSO_BK || w == FSO_BV) && !m->c.qkv_bias) continue;
      materialise(m, l, w);
    }
  materialise(m, 0, FSO_EMBED);
  materialise(m, 0, FSO_HEAD);
  materialise(m, 0, FSO_FINAL_NORM);
  return 0;
}
