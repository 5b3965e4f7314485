/*
 * TEST INFRASTRUCTURE — CPU fp32 oracle of the per-block batched execution path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library, and only as the checker or the timed CPU baseline; the product path
 * (paper_2404_18322_b200/) never calls it.
 *
 * What it restates. The reference (blocksim) prices a block run instead of computing it:
 * CostModel::block_us sums per-component tables (proj/core/src/costmodel.cpp:96-105) for the
 * components a block holds (attention / ffn, proj/core/include/blocksim/zoo.hpp:12, 29-54);
 * activations cross blocks as bf16 rows of embed_dim_out (act_bytes_per_token = 2*d,
 * costmodel.cpp:129-131) and a block's K/V cache costs 4*d bytes per token per attention
 * component (costmodel.cpp:114-127, pages of kPageTokens = 16, kv.hpp:16). The arithmetic those
 * tables stand for is a Llama-2 decoder layer: RMSNorm ->
 * Q,K,V projections -> rotary embedding (rotate_half) -> causal softmax attention over the
 * block-local K/V of the sequence -> O projection + residual -> RMSNorm -> SwiGLU FFN + residual.
 * The cosine equivalence check restates signature_similarity (proj/core/src/zoo.cpp:78-88).
 *
 * Parity pinning: the reference holds no arithmetic golden vectors for the block forward, so the
 * layer math is pinned against HuggingFace transformers' LlamaDecoderLayer (fixtures generated
 * by scripts/make_golden.py into tests/golden/, checked by tests/test_oracle.py); the cosine is
 * pinned by the reference's own cases (test_zoo.cpp:12-18).
 *
 * Everything is fp32 with weights equal to the bf16-rounded synthetic values (oracle/synth.h).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "synth.h"

typedef struct {
  int n_layers, d_model, n_heads, head_dim, d_ff, max_pos;
  float norm_eps, rope_theta, init_scale;
  uint64_t seed;
  const char* name;
  const char* components; /* 'a' attention / 'f' ffn per zoo component; NULL = n_layers x "af" */
  int ffn_src;            /* > d_ff: FFN = first d_ff channels of a d_ff = ffn_src block's FFN */
} or_block_desc; /* same layout as be_block_desc (include/blockexec.h) */

typedef struct {
  float *wq, *wk, *wv, *wo, *wg, *wu, *wd; /* logical row-major [out][in]; NULL if absent */
} or_layer;

typedef struct {
  or_block_desc desc;
  char name[64];
  char comps[1024];
  int n_att, n_ffn;
  or_layer* layers; /* l-th attention component uses wq..wo, l-th ffn wg..wd */
  float* rope_cos;  /* [max_pos][hd/2] */
  float* rope_sin;
} or_block;

typedef struct {
  int n_layers, d, max_tokens, len;
  float* kv; /* [layer][2][max_tokens][d] */
} or_seq;

/* src_cols: logical row stride of the stream (a column prefix of a wider matrix when > cols) */
static void fill_weight(float* w, size_t rows, size_t cols, uint64_t seed, const char* block,
                        int layer, const char* tensor, float scale, size_t src_cols) {
  char sid[160];
  snprintf(sid, sizeof sid, "weights:%s:%d:%s", block, layer, tensor);
  const uint64_t key = or_stream_key(seed, sid);
#pragma omp parallel for schedule(static)
  for (long long r = 0; r < (long long)rows; ++r)
    for (size_t c = 0; c < cols; ++c)
      w[(size_t)r * cols + c] = or_bf16_round(or_synth_value(key, (uint64_t)r * src_cols + c, scale));
}

or_block* or_block_create(const or_block_desc* d) {
  if (!d || d->n_heads * d->head_dim != d->d_model || d->max_pos <= 0) return NULL;
  or_block* b = (or_block*)calloc(1, sizeof(or_block));
  b->desc = *d;
  snprintf(b->name, sizeof b->name, "%s", d->name ? d->name : "block");
  b->desc.name = b->name;
  if (d->components) {
    snprintf(b->comps, sizeof b->comps, "%s", d->components);
  } else {
    for (int l = 0; l < d->n_layers && 2 * l + 2 < (int)sizeof b->comps; ++l) strcat(b->comps, "af");
  }
  b->desc.components = b->comps;
  for (const char* c = b->comps; *c; ++c) {
    if (*c == 'a') ++b->n_att;
    else if (*c == 'f') ++b->n_ffn;
    else { free(b); return NULL; }
  }
  if (b->n_att + b->n_ffn == 0) { free(b); return NULL; }
  b->desc.n_layers = b->n_att > b->n_ffn ? b->n_att : b->n_ffn;
  const size_t D = d->d_model, F = d->d_ff;
  b->layers = (or_layer*)calloc(b->desc.n_layers, sizeof(or_layer));
  for (int l = 0; l < b->n_att; ++l) {
    or_layer* L = &b->layers[l];
    L->wq = (float*)malloc(D * D * 4);
    L->wk = (float*)malloc(D * D * 4);
    L->wv = (float*)malloc(D * D * 4);
    L->wo = (float*)malloc(D * D * 4);
    if (!L->wq || !L->wk || !L->wv || !L->wo) return NULL;
    fill_weight(L->wq, D, D, d->seed, b->name, l, "wq", d->init_scale, D);
    fill_weight(L->wk, D, D, d->seed, b->name, l, "wk", d->init_scale, D);
    fill_weight(L->wv, D, D, d->seed, b->name, l, "wv", d->init_scale, D);
    fill_weight(L->wo, D, D, d->seed, b->name, l, "wo", d->init_scale, D);
  }
  for (int l = 0; l < b->n_ffn; ++l) {
    or_layer* L = &b->layers[l];
    L->wg = (float*)malloc(F * D * 4);
    L->wu = (float*)malloc(F * D * 4);
    L->wd = (float*)malloc(D * F * 4);
    if (!L->wg || !L->wu || !L->wd) return NULL;
    const size_t F_src = d->ffn_src > d->d_ff ? (size_t)d->ffn_src : F;
    fill_weight(L->wg, F, D, d->seed, b->name, l, "wg", d->init_scale, D);
    fill_weight(L->wu, F, D, d->seed, b->name, l, "wu", d->init_scale, D);
    fill_weight(L->wd, D, F, d->seed, b->name, l, "wd", d->init_scale, F_src);
  }
  const int half = d->head_dim / 2;
  b->rope_cos = (float*)malloc((size_t)d->max_pos * half * 4);
  b->rope_sin = (float*)malloc((size_t)d->max_pos * half * 4);
  for (int p = 0; p < d->max_pos; ++p)
    for (int j = 0; j < half; ++j) {
      const double inv = pow((double)d->rope_theta, -2.0 * j / d->head_dim);
      const double ang = (double)p * inv;
      b->rope_cos[(size_t)p * half + j] = (float)cos(ang);
      b->rope_sin[(size_t)p * half + j] = (float)sin(ang);
    }
  return b;
}

void or_block_free(or_block* b) {
  if (!b) return;
  for (int l = 0; l < b->desc.n_layers; ++l) {
    or_layer* L = &b->layers[l];
    free(L->wq); free(L->wk); free(L->wv); free(L->wo); free(L->wg); free(L->wu); free(L->wd);
  }
  free(b->layers);
  free(b->rope_cos);
  free(b->rope_sin);
  free(b);
}

const float* or_block_weight(const or_block* b, int layer, const char* t) {
  if (!b || layer < 0 || layer >= b->desc.n_layers) return NULL;
  const or_layer* L = &b->layers[layer];
  if (!strcmp(t, "wq")) return L->wq;
  if (!strcmp(t, "wk")) return L->wk;
  if (!strcmp(t, "wv")) return L->wv;
  if (!strcmp(t, "wo")) return L->wo;
  if (!strcmp(t, "wg")) return L->wg;
  if (!strcmp(t, "wu")) return L->wu;
  if (!strcmp(t, "wd")) return L->wd;
  return NULL;
}

/* W[layer][tensor] += delta (logical [rows][cols] fp32): a LoRA adapter's B A folded into the
 * restated weights (the GPU keeps B and A apart; be_exec_lora_batch). */
int or_block_add_delta(or_block* b, int layer, const char* t, const float* delta) {
  float* w = (float*)or_block_weight(b, layer, t);
  if (!w || !delta) return 1;
  const size_t D = b->desc.d_model, F = b->desc.d_ff;
  size_t n = D * D;
  if (!strcmp(t, "wg") || !strcmp(t, "wu") || !strcmp(t, "wd")) n = D * F;
  for (size_t i = 0; i < n; ++i) w[i] += delta[i];
  return 0;
}

or_seq* or_seq_create(const or_block* b, int max_tokens) {
  or_seq* s = (or_seq*)calloc(1, sizeof(or_seq));
  s->n_layers = b->n_att; /* K/V planes: one per attention component */
  s->d = b->desc.d_model;
  s->max_tokens = max_tokens;
  s->kv = (float*)calloc((size_t)s->n_layers * 2 * max_tokens * s->d, 4);
  return s;
}
void or_seq_free(or_seq* s) {
  if (!s) return;
  free(s->kv);
  free(s);
}
int or_seq_len(const or_seq* s) { return s->len; }
/* Fills positions [0, len) of every layer's K/V with synthetic values (CPU-baseline timing:
 * stands in for a prefill the timed sample does not redo). */
void or_seq_fill(or_seq* s, int len, uint64_t seed) {
  if (len > s->max_tokens) len = s->max_tokens;
  const uint64_t key = or_stream_key(seed, "oracle:kvfill");
  const size_t per = (size_t)s->max_tokens * s->d;
#pragma omp parallel for schedule(static)
  for (long long lk = 0; lk < (long long)s->n_layers * 2; ++lk)
    for (size_t i = 0; i < (size_t)len * s->d; ++i)
      s->kv[lk * per + i] = or_synth_value(key, lk * per + i, 1.0f);
  s->len = len;
}
const float* or_seq_kv(const or_seq* s, int layer, int kv) {
  return s->kv + ((size_t)layer * 2 + kv) * s->max_tokens * s->d;
}

/* Y[n][N] = X[n][K] . W[N][K]^T */
static void matmul_nt(const float* X, const float* W, float* Y, int n, int N, int K) {
#pragma omp parallel for schedule(static)
  for (int o = 0; o < N; ++o) {
    const float* w = W + (size_t)o * K;
    for (int t = 0; t < n; ++t) {
      const float* x = X + (size_t)t * K;
      float acc = 0.f;
#pragma omp simd reduction(+ : acc)
      for (int k = 0; k < K; ++k) acc += x[k] * w[k];
      Y[(size_t)t * N + o] = acc;
    }
  }
}

static void rmsnorm(const float* x, float* y, int n, int d, float eps) {
  for (int t = 0; t < n; ++t) {
    double ss = 0.0;
    for (int i = 0; i < d; ++i) ss += (double)x[(size_t)t * d + i] * x[(size_t)t * d + i];
    const float r = (float)(1.0 / sqrt(ss / d + (double)eps));
    for (int i = 0; i < d; ++i) y[(size_t)t * d + i] = x[(size_t)t * d + i] * r;
  }
}

/* rotate_half RoPE on one head vector in place (HF Llama convention) */
static void rope_apply(float* v, int hd, const float* cs, const float* sn) {
  const int half = hd / 2;
  for (int j = 0; j < half; ++j) {
    const float a = v[j], b = v[j + half];
    v[j] = a * cs[j] - b * sn[j];
    v[j + half] = b * cs[j] + a * sn[j];
  }
}

/*
 * Runs n tokens through every layer of the block (the work blocksim prices as block_us).
 * Token i belongs to seqs[tok_seq[i]] at position tok_pos[i]; its K/V are appended there and it
 * attends to positions [0, tok_pos[i]] of its sequence. Returns 0, or -1 on bad input.
 */
int or_block_forward(const or_block* b, or_seq** seqs, int n, const int* tok_seq,
                     const int* tok_pos, const float* x_in, float* x_out, int n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#else
  (void)n_threads;
#endif
  const or_block_desc* D = &b->desc;
  const int d = D->d_model, F = D->d_ff, H = D->n_heads, hd = D->head_dim, half = hd / 2;
  for (int i = 0; i < n; ++i) {
    const or_seq* s = seqs[tok_seq[i]];
    if (tok_pos[i] < 0 || tok_pos[i] >= s->max_tokens || tok_pos[i] >= D->max_pos) return -1;
  }
  float* x = (float*)malloc((size_t)n * d * 4);
  float* xn = (float*)malloc((size_t)n * d * 4);
  float* q = (float*)malloc((size_t)n * d * 4);
  float* k = (float*)malloc((size_t)n * d * 4);
  float* v = (float*)malloc((size_t)n * d * 4);
  float* att = (float*)malloc((size_t)n * d * 4);
  float* o = (float*)malloc((size_t)n * d * 4);
  float* g = (float*)malloc((size_t)n * F * 4);
  float* u = (float*)malloc((size_t)n * F * 4);
  memcpy(x, x_in, (size_t)n * d * 4);
  const float scale = 1.0f / sqrtf((float)hd);

  int ia = 0, jf = 0;
  for (const char* comp = b->comps; *comp; ++comp) {
    if (*comp == 'f') {
      /* ffn component */
      const or_layer* L = &b->layers[jf++];
      rmsnorm(x, xn, n, d, D->norm_eps);
      matmul_nt(xn, L->wg, g, n, F, d);
      matmul_nt(xn, L->wu, u, n, F, d);
      for (size_t i = 0; i < (size_t)n * F; ++i) g[i] = g[i] / (1.0f + expf(-g[i])) * u[i];
      matmul_nt(g, L->wd, o, n, d, F);
      for (size_t i = 0; i < (size_t)n * d; ++i) x[i] += o[i];
      continue;
    }
    const int l = ia++;
    const or_layer* L = &b->layers[l];
    /* attention component */
    rmsnorm(x, xn, n, d, D->norm_eps);
    matmul_nt(xn, L->wq, q, n, d, d);
    matmul_nt(xn, L->wk, k, n, d, d);
    matmul_nt(xn, L->wv, v, n, d, d);
    for (int i = 0; i < n; ++i) {
      const int pos = tok_pos[i];
      const float* cs = b->rope_cos + (size_t)pos * half;
      const float* sn = b->rope_sin + (size_t)pos * half;
      for (int h = 0; h < H; ++h) {
        rope_apply(q + (size_t)i * d + h * hd, hd, cs, sn);
        rope_apply(k + (size_t)i * d + h * hd, hd, cs, sn);
      }
      or_seq* s = seqs[tok_seq[i]];
      float* kc = s->kv + ((size_t)l * 2 + 0) * s->max_tokens * d;
      float* vc = s->kv + ((size_t)l * 2 + 1) * s->max_tokens * d;
      memcpy(kc + (size_t)pos * d, k + (size_t)i * d, (size_t)d * 4);
      memcpy(vc + (size_t)pos * d, v + (size_t)i * d, (size_t)d * 4);
      if (pos + 1 > s->len) s->len = pos + 1;
    }
#pragma omp parallel for schedule(dynamic)
    for (int ih = 0; ih < n * H; ++ih) {
      const int i = ih / H, h = ih % H;
      const int ctx = tok_pos[i] + 1;
      const or_seq* s = seqs[tok_seq[i]];
      const float* kc = s->kv + ((size_t)l * 2 + 0) * s->max_tokens * d;
      const float* vc = s->kv + ((size_t)l * 2 + 1) * s->max_tokens * d;
      const float* qh = q + (size_t)i * d + h * hd;
      float* sc = (float*)malloc((size_t)ctx * 4);
      float mx = -INFINITY;
      for (int p = 0; p < ctx; ++p) {
        const float* kp = kc + (size_t)p * d + h * hd;
        float acc = 0.f;
        for (int e = 0; e < hd; ++e) acc += qh[e] * kp[e];
        sc[p] = acc * scale;
        if (sc[p] > mx) mx = sc[p];
      }
      double sum = 0.0;
      for (int p = 0; p < ctx; ++p) {
        sc[p] = expf(sc[p] - mx);
        sum += sc[p];
      }
      float* out = att + (size_t)i * d + h * hd;
      for (int e = 0; e < hd; ++e) out[e] = 0.f;
      for (int p = 0; p < ctx; ++p) {
        const float w = (float)(sc[p] / sum);
        const float* vp = vc + (size_t)p * d + h * hd;
        for (int e = 0; e < hd; ++e) out[e] += w * vp[e];
      }
      free(sc);
    }
    matmul_nt(att, L->wo, o, n, d, d);
    for (size_t i = 0; i < (size_t)n * d; ++i) x[i] += o[i];
  }
  memcpy(x_out, x, (size_t)n * d * 4);
  free(x); free(xn); free(q); free(k); free(v); free(att); free(o); free(g); free(u);
  return 0;
}

/* signature_similarity (proj/core/src/zoo.cpp:78-88): dot / (sqrt(na) * sqrt(nb)) in double.
 * *err = 1 on length mismatch is not representable here (same n); *err = 2 on a zero norm
 * (the reference throws std::invalid_argument). */
double or_cosine(const double* a, const double* b, int n, int* err) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int i = 0; i < n; ++i) {
    dot += a[i] * b[i];
    na += a[i] * a[i];
    nb += b[i] * b[i];
  }
  if (err) *err = 0;
  if (na == 0.0 || nb == 0.0) {
    if (err) *err = 2;
    return 0.0;
  }
  return dot / (sqrt(na) * sqrt(nb));
}

/* K7 per-row restatement over [rows][d] fp32 inputs (the values of the bf16 rows). */
void or_cosine_rows(const float* a, const float* b, int rows, int d, float thr, float* cos_out,
                    int* accept) {
  for (int r = 0; r < rows; ++r) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (int i = 0; i < d; ++i) {
      const double x = a[(size_t)r * d + i], y = b[(size_t)r * d + i];
      dot += x * y;
      na += x * x;
      nb += y * y;
    }
    const float c = (na > 0.0 && nb > 0.0) ? (float)(dot / (sqrt(na) * sqrt(nb))) : NAN;
    cos_out[r] = c;
    if (accept) accept[r] = c >= thr ? 1 : 0;
  }
}

/* element i of a synthetic stream (same bits as the device generator) */
float or_synth(uint64_t seed, const char* stream_id, uint64_t i, float scale) {
  return or_synth_value(or_stream_key(seed, stream_id), i, scale);
}
void or_synth_fill(float* dst, uint64_t n, uint64_t seed, const char* stream_id, float scale,
                   int round_bf16) {
  const uint64_t key = or_stream_key(seed, stream_id);
  for (uint64_t i = 0; i < n; ++i) {
    const float v = or_synth_value(key, i, scale);
    dst[i] = round_bf16 ? or_bf16_round(v) : v;
  }
}
