// C-ABI implementation of include/blockexec.h: contexts, synthetic block weights, paged KV
// pools, workspaces and the per-block batched execution (gather -> L x decoder layer -> scatter).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "../../include/blockexec.h"
#include "gemm_tc.cuh"

namespace bx {
// rowops.cu
cudaError_t launch_gather(const __nv_bfloat16*, const int*, int, int, int, __nv_bfloat16*, float*, float*, cudaStream_t,
                          unsigned long long*, int);
cudaError_t launch_scatter(const __nv_bfloat16*, const int*, int, int, int, __nv_bfloat16*, cudaStream_t,
                           unsigned long long*, int);
cudaError_t launch_cosine(const __nv_bfloat16*, const __nv_bfloat16*, int, int, float, float*, int*, cudaStream_t);
cudaError_t launch_synth_weight(__nv_bfloat16*, int, int, uint64_t, uint64_t, float, int, int, const float*, cudaStream_t,
                                int src_cols = 0);
cudaError_t launch_synth_rows(__nv_bfloat16*, long long, uint64_t, float, cudaStream_t);
cudaError_t launch_pack_weight(const __nv_bfloat16*, __nv_bfloat16*, int, int, cudaStream_t);
cudaError_t launch_rope_table(float2*, int, int, double, cudaStream_t);
cudaError_t launch_synth_plain(__nv_bfloat16*, int, int, uint64_t, float, int, int, cudaStream_t);
cudaError_t launch_lora_shrink(const __nv_bfloat16*, int, int, const float*, int, float,
                               const LoraTable&, int, const int*, float*, int, cudaStream_t);
// attention.cu
struct AttnParams {
  const __nv_bfloat16* q;
  const __nv_bfloat16* pool;
  long long page_elems;
  long long layer_elems;
  int layer;
  const int* page_table;
  int pt_stride;
  const int* row_pt;
  const int* row_ctx;
  int meta_stride;
  int ctx_add;
  int H;
  float scale_log2;
  __nv_bfloat16* out;
  float* part;
  int splits;
  int n_grp;
  int grp_rows;
  const __nv_bfloat16* pools[8];
  unsigned long long* tl;
  int tl_cap;
};
cudaError_t launch_attention(const AttnParams&, int rows, int head_dim, cudaStream_t);
// attention_prefill.cu
struct PrefillAttnParams {
  const __nv_bfloat16* q;
  const __nv_bfloat16* pool;
  long long page_elems;
  long long layer_elems;
  int layer;
  const int* page_table;
  int pt_stride;
  const int* tok;
  int rows;
  int H;
  float scale_log2;
  __nv_bfloat16* out;
  int* tiles;
};
struct PrefillTcParams {
  const int* page_table;
  int pt_stride;
  const int* tok;
  int rows;
  int H;
  int layer, n_layers;
  float scale_log2;
  __nv_bfloat16* out;
  const int* tiles;
};
cudaError_t launch_attention_prefill_pipe(const PrefillTcParams& P, const CUtensorMap& map_q,
                                          const CUtensorMap& map_kv, int num_sms,
                                          cudaStream_t stream);
cudaError_t launch_attention_prefill_tc(const PrefillTcParams& P, const CUtensorMap& map_q,
                                        const CUtensorMap& map_kv, int num_sms,
                                        cudaStream_t stream);
cudaError_t launch_attention_prefill(const PrefillAttnParams&, int head_dim, int num_sms,
                                     cudaStream_t);
}  // namespace bx

using bx::EpiParams;
using bf16 = __nv_bfloat16;

// ------------------------------------------------------------------------------ objects
struct be_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  // scratch for the standalone GEMM entry point
  float* gemm_ws = nullptr;
  size_t gemm_ws_elems = 0;
  int* gemm_counters = nullptr;
  int gemm_grid_cap = 0;  // 0 = one persistent CTA per SM (BE_GEMM_GRID overrides)
  int use_pdl = 1;        // programmatic dependent launch of GEMMs (BE_PDL=0 disables)
  int prefill_tc = 1;     // prefill attention (BE_PREFILL_TC): 1 tcgen05, two CTAs per SM (hd
                          // 128; mma.sync for hd 64), 4 tcgen05 warp-specialised one CTA per SM
                          // (experiment: slower), 2 mma.sync, 0 the per-row decode kernel
  int attn_splits_force = 0;  // decode attention split-K count (BE_ATTN_SPLITS=1..16; 0 = auto)
  // per-launch event timing of exec_batch kernels (be_prof_enable); off on the hot path
  struct ProfRec {
    be_prof_rec r;
    cudaEvent_t a, b;
  };
  // kernel timeline (be_timeline_*): [4][tl_cap] u64 on the device, slots in launch order
  unsigned long long* tl = nullptr;
  int tl_cap = 0;
  int tl_next = 0;
  std::vector<int> tl_cls;
  // speculation (be_exec_speculative): the draft lane's stream, fork/join events, verdict scratch
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_copy = nullptr;  // be_kv_copy_pages: reads of this context's pools wait on it
  float* attn_part = nullptr;     // be_attention's split-K partials
  size_t attn_part_elems = 0;
  float* spec_cos = nullptr;
  int* spec_accept = nullptr;
  int spec_cap = 0;
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;
  size_t prof_ev_used = 0;
  std::vector<ProfRec> prof_recs;
};

struct be_block {
  be_ctx* ctx = nullptr;
  be_block_desc desc{};
  std::string name;
  bf16* slab = nullptr;
  size_t slab_elems = 0;
  float2* rope = nullptr;
  struct Layer {
    bf16 *wqkv, *wo, *wgu, *wd;  // packed tile layout (ptx.cuh packed_index); null if absent
  };
  std::vector<Layer> layers;  // l-th attention component uses wqkv/wo, l-th ffn wgu/wd
  std::string comps;          // component sequence, 'a' attention / 'f' ffn
  int n_att = 0, n_ffn = 0;
};

struct be_kv_pool {
  be_ctx* ctx = nullptr;
  bf16* base = nullptr;
  int n_pages = 0;
  long long page_elems = 0;
  long long layer_elems = 0;
  int n_layers = 0, n_heads = 0, head_dim = 0;
  // 5-D TMA map [page*layers + layer][K|V][head][16 tokens][hd], box {64, 16, 1, 1, 1}: the
  // tcgen05 prefill attention's K / V page loads (encoded on first use)
  CUtensorMap m_kv{};
  bool has_m_kv = false;
};

// LoRA adapter of a block's attention components: per attention layer
// A_qkv [3r][d] (q, k, v stacked), B_qkv [3d][r] (rows in the fused QKV GEMM's physical order),
// A_o [r][d], B_o [d][r]; plain row-major bf16, r = kLoraRank
struct be_lora {
  be_ctx* ctx = nullptr;
  int d = 0, n_att = 0;
  bf16* slab = nullptr;
  struct Layer {
    bf16 *aqkv, *bqkv, *ao, *bo;
  };
  std::vector<Layer> layers;
};

struct be_workspace {
  be_ctx* ctx = nullptr;
  int d = 0, dff = 0, H = 0, max_tok = 0, max_rows = 0, max_pages = 0;
  float* X = nullptr;
  bf16* Xb = nullptr;
  bf16* q = nullptr;
  bf16* attn = nullptr;
  bf16* h = nullptr;
  float* ss = nullptr;  // [max_tok][d / 32] sums of squares of the residual stream (fused RMSNorm)
  float* rstd = nullptr;  // [max_tok] its per-token rstd, reduced once for round-robin GEMMs
  float* lora_u = nullptr;  // [max_tok][3 * kLoraRank] LoRA shrink outputs
  int32_t* d_lora_idx = nullptr;  // [max_tok] adapter per token (be_exec_lora_batch staging)
  float* splitws = nullptr;
  size_t splitws_elems = 0;
  int* counters = nullptr;
  int n_counters = 0;
  int* prefill_tiles = nullptr;  // [max_tok + 2] query tiles of the tensor-core prefill attention
  float* attn_part = nullptr;
  size_t attn_part_elems = 0;
  be_token* d_tokens = nullptr;
  int32_t* d_pt = nullptr;
  size_t pt_capacity = 0;
  // TMA maps of the B operands by BN (16..256)
  std::map<int, CUtensorMap> m_xb, m_attn, m_h;
  CUtensorMap m_q{};        // q rows, box {64, 128}: the tcgen05 prefill attention's Q tiles
  bool has_m_q = false;
};

// ------------------------------------------------------------------------------ helpers
namespace {

int fail(be_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx != nullptr) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return code;
}

#define BE_CUDA(ctx, call)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail((ctx), BE_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                  __FILE__, __LINE__);                                                     \
  } while (0)

uint64_t fnv1a64(const std::string& s) {
  uint64_t h = 14695981039346656037ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

// Key of a synthetic stream: the splitmix64 seeding state of blocksim's RngStream
// (proj/core/include/blocksim/rng.hpp:17-19): seed ^ fnv1a64(stream_id).
uint64_t stream_key(uint64_t seed, const std::string& id) { return seed ^ fnv1a64(id); }

std::string weight_stream(const std::string& block, int layer, const char* tensor) {
  return "weights:" + block + ":" + std::to_string(layer) + ":" + tensor;
}

// 2D bf16 row-major [rows][cols] tensor map, box {64 cols, box_rows rows}, 128B swizzle.
int make_map(be_ctx* ctx, CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
             uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * sizeof(bf16)};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ctx, BE_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu box=%u",
                (int)r, (unsigned long long)rows, (unsigned long long)cols, box_rows);
  return BE_OK;
}

cudaStream_t pick_stream(be_ctx* ctx, void* s) {
  return s != nullptr ? static_cast<cudaStream_t>(s) : ctx->stream;
}

const int kBNs[5] = {16, 32, 64, 128, 256};

int attn_splits(const be_ctx* ctx, int rows, int H, int max_pages) {
  if (ctx->attn_splits_force > 0) return ctx->attn_splits_force;  // tests: the split-K path
  const long long ctas = (long long)rows * H;
  const long long want = 4LL * ctx->num_sms;
  if (ctas >= want) return 1;
  int s = (int)((want + ctas - 1) / ctas);
  if (s > 16) s = 16;
  const int cap = max_pages / 4 > 1 ? max_pages / 4 : 1;  // keep >= 4 pages per split
  if (s > cap) s = cap;
  return s < 1 ? 1 : s;
}

}  // namespace

// ------------------------------------------------------------------------------ context
extern "C" int be_ctx_create(int device, be_ctx** out) {
  if (out == nullptr) return BE_ERR_INVALID;
  *out = nullptr;
  auto* ctx = new be_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return BE_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10) {
    delete ctx;
    return BE_ERR_RUNTIME;  // sm_100a only
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return BE_ERR_CUDA;
  }
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
          cudaSuccess ||
      fn == nullptr) {
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return BE_ERR_CUDA;
  }
  ctx->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  if (const char* g = getenv("BE_GEMM_GRID")) ctx->gemm_grid_cap = atoi(g);
  if (const char* p = getenv("BE_PDL")) ctx->use_pdl = atoi(p) != 0;
  if (const char* p = getenv("BE_PREFILL_TC")) ctx->prefill_tc = atoi(p);
  if (const char* p = getenv("BE_ATTN_SPLITS")) {
    const int v = atoi(p);
    ctx->attn_splits_force = v < 0 ? 0 : v > 16 ? 16 : v;
  }
  *out = ctx;
  return BE_OK;
}

extern "C" int be_ctx_destroy(be_ctx* ctx) {
  if (ctx == nullptr) return BE_ERR_INVALID;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (cudaEvent_t ev : ctx->prof_ev) cudaEventDestroy(ev);
  if (ctx->tl) cudaFree(ctx->tl);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
  if (ctx->attn_part) cudaFree(ctx->attn_part);
  if (ctx->spec_cos) cudaFree(ctx->spec_cos);
  if (ctx->spec_accept) cudaFree(ctx->spec_accept);
  if (ctx->gemm_ws) cudaFree(ctx->gemm_ws);
  if (ctx->gemm_counters) cudaFree(ctx->gemm_counters);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return BE_OK;
}

extern "C" const char* be_last_error(const be_ctx* ctx) {
  return ctx == nullptr ? "null context" : ctx->err.c_str();
}
extern "C" int be_ctx_num_sms(const be_ctx* ctx) { return ctx ? ctx->num_sms : 0; }
extern "C" void* be_ctx_stream(be_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
extern "C" int be_synchronize(be_ctx* ctx) {
  if (ctx == nullptr) return BE_ERR_INVALID;
  BE_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  BE_CUDA(ctx, cudaGetLastError());
  return BE_OK;
}

// ------------------------------------------------------------------------------ blocks
extern "C" int be_block_load(be_ctx* ctx, const be_block_desc* d, be_block** out) {
  if (ctx == nullptr || d == nullptr || out == nullptr) return BE_ERR_INVALID;
  *out = nullptr;
  // component sequence: explicit ("a" attention, "f" ffn, zoo.hpp:12), else n_layers x "af"
  std::string comps;
  if (d->components != nullptr) {
    comps = d->components;
    for (char c : comps)
      if (c != 'a' && c != 'f') return fail(ctx, BE_ERR_INVALID, "block: component kinds are 'a'/'f'");
  } else {
    for (int l = 0; l < d->n_layers; ++l) comps += "af";
  }
  if (comps.empty() || d->d_model <= 0 || d->n_heads <= 0 || d->head_dim <= 0 ||
      d->d_ff <= 0 || d->n_heads * d->head_dim != d->d_model)
    return fail(ctx, BE_ERR_INVALID, "block: inconsistent shape");
  if (d->d_model % 128 != 0 || d->d_ff % 64 != 0 || (2 * d->d_ff) % 128 != 0)
    return fail(ctx, BE_ERR_INVALID, "block: d_model %% 128 and d_ff %% 64 required");
  if (d->d_model > 8192) return fail(ctx, BE_ERR_INVALID, "block: d_model <= 8192 required");
  if (d->head_dim != 64 && d->head_dim != 128)
    return fail(ctx, BE_ERR_INVALID, "block: head_dim must be 64 or 128");
  if (d->max_pos <= 0) return fail(ctx, BE_ERR_INVALID, "block: max_pos must be positive");
  if (d->ffn_src != 0 && d->ffn_src < d->d_ff)
    return fail(ctx, BE_ERR_INVALID, "block: ffn_src must be 0 or >= d_ff");
  const int F_src = d->ffn_src > 0 ? d->ffn_src : d->d_ff;
  cudaSetDevice(ctx->device);
  auto* b = new be_block();
  b->ctx = ctx;
  b->desc = *d;
  b->name = d->name ? d->name : "block";
  b->desc.name = nullptr;
  b->desc.components = nullptr;
  b->comps = comps;
  b->n_att = (int)std::count(comps.begin(), comps.end(), 'a');
  b->n_ffn = (int)comps.size() - b->n_att;
  b->desc.n_layers = std::max(b->n_att, b->n_ffn);
  const size_t D = d->d_model, F = d->d_ff;
  const size_t att_elems = 3 * D * D + D * D, ffn_elems = 2 * F * D + D * F;
  b->slab_elems = att_elems * b->n_att + ffn_elems * b->n_ffn;
  if (cudaMalloc(&b->slab, b->slab_elems * sizeof(bf16)) != cudaSuccess) {
    delete b;
    return fail(ctx, BE_ERR_NOMEM, "block: weight slab (%zu B) allocation failed",
                b->slab_elems * sizeof(bf16));
  }
  if (cudaMalloc(&b->rope, (size_t)d->max_pos * d->head_dim / 2 * sizeof(float2)) != cudaSuccess) {
    cudaFree(b->slab);
    delete b;
    return fail(ctx, BE_ERR_NOMEM, "block: rope table allocation failed");
  }
  cudaStream_t st = ctx->stream;
  bx::launch_rope_table(b->rope, d->max_pos, d->head_dim, (double)d->rope_theta, st);
  const float s = d->init_scale;
  // weights in component order; the l-th attention (ffn) component is "layer" l of its kind
  b->layers.assign(b->desc.n_layers, be_block::Layer{nullptr, nullptr, nullptr, nullptr});
  bf16* cur = b->slab;
  int ia = 0, jf = 0;
  for (char c : comps) {
    if (c == 'a') {
      auto& L = b->layers[ia];
      auto key = [&](const char* t) { return stream_key(d->seed, weight_stream(b->name, ia, t)); };
      L.wqkv = cur;
      L.wo = cur + 3 * D * D;
      cur += att_elems;
      bx::launch_synth_weight(L.wqkv, (int)D, (int)D, key("wq"), 0, s, 1, d->head_dim, nullptr, st);
      bx::launch_synth_weight(L.wqkv + D * D, (int)D, (int)D, key("wk"), 0, s, 1, d->head_dim, nullptr, st);
      bx::launch_synth_weight(L.wqkv + 2 * D * D, (int)D, (int)D, key("wv"), 0, s, 0, d->head_dim, nullptr, st);
      bx::launch_synth_weight(L.wo, (int)D, (int)D, key("wo"), 0, s, 0, d->head_dim, nullptr, st);
      ++ia;
    } else {
      auto& L = b->layers[jf];
      auto key = [&](const char* t) { return stream_key(d->seed, weight_stream(b->name, jf, t)); };
      L.wgu = cur;
      L.wd = cur + 2 * F * D;
      cur += ffn_elems;
      bx::launch_synth_weight(L.wgu, (int)(2 * F), (int)D, key("wg"), key("wu"), s, 2, d->head_dim, nullptr, st);
      bx::launch_synth_weight(L.wd, (int)D, (int)F, key("wd"), 0, s, 0, d->head_dim, nullptr, st,
                              F_src);
      ++jf;
    }
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    be_block_free(b);
    return fail(ctx, BE_ERR_CUDA, "block init: %s", cudaGetErrorString(e));
  }
  *out = b;
  return BE_OK;
}

extern "C" int be_block_free(be_block* b) {
  if (b == nullptr) return BE_ERR_INVALID;
  cudaSetDevice(b->ctx->device);
  if (b->slab) cudaFree(b->slab);
  if (b->rope) cudaFree(b->rope);
  delete b;
  return BE_OK;
}

extern "C" int64_t be_block_param_bytes(const be_block* b) {
  return b ? (int64_t)(b->slab_elems * sizeof(bf16)) : 0;
}

extern "C" int64_t be_block_kv_bytes_per_token(const be_block* b) {
  return b ? 4LL * b->desc.d_model * b->n_att : 0;
}

extern "C" int be_block_read_weight(be_block* b, int layer, const char* tensor, float* host_out) {
  if (b == nullptr || tensor == nullptr || host_out == nullptr) return BE_ERR_INVALID;
  be_ctx* ctx = b->ctx;
  if (layer < 0 || layer >= b->desc.n_layers) return fail(ctx, BE_ERR_INVALID, "bad layer");
  const int D = b->desc.d_model, F = b->desc.d_ff, hd = b->desc.head_dim;
  const auto& L = b->layers[layer];
  const std::string t = tensor;
  const bool att_t = t == "wq" || t == "wk" || t == "wv" || t == "wo";
  if ((att_t && L.wqkv == nullptr) || (!att_t && L.wgu == nullptr))
    return fail(ctx, BE_ERR_INVALID, "block has no %s of component %d", tensor, layer);
  const bf16* src = nullptr;
  int rows = 0, cols = 0, perm = 0, parity = 0;
  if (t == "wq") { src = L.wqkv; rows = D; cols = D; perm = 1; }
  else if (t == "wk") { src = L.wqkv + (size_t)D * D; rows = D; cols = D; perm = 1; }
  else if (t == "wv") { src = L.wqkv + 2 * (size_t)D * D; rows = D; cols = D; }
  else if (t == "wo") { src = L.wo; rows = D; cols = D; }
  else if (t == "wg") { src = L.wgu; rows = F; cols = D; perm = 2; parity = 0; }
  else if (t == "wu") { src = L.wgu; rows = F; cols = D; perm = 2; parity = 1; }
  else if (t == "wd") { src = L.wd; rows = D; cols = F; }
  else return fail(ctx, BE_ERR_INVALID, "unknown tensor %s", tensor);
  const int prow = perm == 2 ? 2 * rows : rows;
  std::vector<bf16> tmp((size_t)prow * cols);
  BE_CUDA(ctx, cudaMemcpy(tmp.data(), src, tmp.size() * sizeof(bf16), cudaMemcpyDeviceToHost));
  for (int pr = 0; pr < prow; ++pr) {
    int lr = pr;
    if (perm == 1) {
      const int h = pr / hd, e = pr % hd;
      lr = h * hd + ((e & 1) ? (e >> 1) + hd / 2 : (e >> 1));
    } else if (perm == 2) {
      if ((pr & 1) != parity) continue;
      lr = pr >> 1;
    }
    for (int c = 0; c < cols; ++c)
      host_out[(size_t)lr * cols + c] = __bfloat162float(tmp[bx::packed_index(pr, c, cols)]);
  }
  return BE_OK;
}

// ------------------------------------------------------------------------------ KV pool
extern "C" int be_kv_pool_create(be_ctx* ctx, const be_block* b, int n_pages, be_kv_pool** out) {
  if (ctx == nullptr || b == nullptr || out == nullptr || n_pages <= 0) return BE_ERR_INVALID;
  *out = nullptr;
  cudaSetDevice(ctx->device);
  auto* p = new be_kv_pool();
  p->ctx = ctx;
  p->n_pages = n_pages;
  p->n_layers = b->n_att;  // one K/V plane pair per attention component of the block
  p->n_heads = b->desc.n_heads;
  p->head_dim = b->desc.head_dim;
  p->layer_elems = 2LL * p->n_heads * 16 * p->head_dim;
  p->page_elems = p->layer_elems * p->n_layers;
  const size_t bytes = (size_t)p->page_elems * n_pages * sizeof(bf16);
  if (bytes > 0) {  // ffn-only blocks keep no KV
    if (cudaMalloc(&p->base, bytes) != cudaSuccess) {
      delete p;
      return fail(ctx, BE_ERR_NOMEM, "kv pool: %zu B allocation failed", bytes);
    }
    cudaMemsetAsync(p->base, 0, bytes, ctx->stream);
  }
  *out = p;
  return BE_OK;
}

extern "C" int be_kv_pool_free(be_kv_pool* p) {
  if (p == nullptr) return BE_ERR_INVALID;
  cudaSetDevice(p->ctx->device);
  if (p->base) cudaFree(p->base);
  delete p;
  return BE_OK;
}

extern "C" void* be_kv_pool_data(be_kv_pool* p) { return p ? p->base : nullptr; }
extern "C" int64_t be_kv_pool_page_bytes(const be_kv_pool* p) {
  return p ? p->page_elems * (int64_t)sizeof(bf16) : 0;
}

extern "C" int be_kv_pool_read(be_kv_pool* p, int64_t offset, int64_t bytes, void* host_dst) {
  if (p == nullptr || host_dst == nullptr || offset < 0 || bytes < 0 ||
      offset + bytes > p->page_elems * (int64_t)sizeof(bf16) * p->n_pages)
    return BE_ERR_INVALID;
  cudaSetDevice(p->ctx->device);
  BE_CUDA(p->ctx, cudaStreamSynchronize(p->ctx->stream));
  BE_CUDA(p->ctx, cudaMemcpy(host_dst, reinterpret_cast<const char*>(p->base) + offset, bytes,
                             cudaMemcpyDeviceToHost));
  return BE_OK;
}

// ------------------------------------------------------------------------------ workspace
extern "C" int be_workspace_create(be_ctx* ctx, int d, int dff, int H, int max_tok, int max_rows,
                                   int max_pages, be_workspace** out) {
  if (ctx == nullptr || out == nullptr || d <= 0 || dff <= 0 || H <= 0 || max_tok <= 0 ||
      max_rows <= 0 || max_pages <= 0)
    return BE_ERR_INVALID;
  *out = nullptr;
  cudaSetDevice(ctx->device);
  auto* w = new be_workspace();
  w->ctx = ctx;
  w->d = d;
  w->dff = dff;
  w->H = H;
  w->max_tok = max_tok;
  w->max_rows = max_rows;
  w->max_pages = max_pages;
  const size_t T = max_tok;
  bool ok = true;
  ok &= cudaMalloc(&w->X, T * d * sizeof(float)) == cudaSuccess;
  ok &= cudaMalloc(&w->Xb, T * d * sizeof(bf16)) == cudaSuccess;
  ok &= cudaMalloc(&w->q, T * d * sizeof(bf16)) == cudaSuccess;
  ok &= cudaMalloc(&w->attn, T * d * sizeof(bf16)) == cudaSuccess;
  ok &= cudaMalloc(&w->h, T * dff * sizeof(bf16)) == cudaSuccess;
  ok &= cudaMalloc(&w->ss, T * (d / 32) * sizeof(float)) == cudaSuccess;
  ok &= cudaMalloc(&w->rstd, T * sizeof(float)) == cudaSuccess;
  ok &= cudaMalloc(&w->lora_u, T * 3 * bx::kLoraRank * sizeof(float)) == cudaSuccess;
  ok &= cudaMalloc(&w->d_lora_idx, T * sizeof(int32_t)) == cudaSuccess;
  w->splitws_elems = (size_t)16 << 20;  // 64 MB of fp32 split-K partials (L2 sized)
  ok &= cudaMalloc(&w->splitws, w->splitws_elems * sizeof(float)) == cudaSuccess;
  w->n_counters = 1 << 16;
  ok &= cudaMalloc(&w->counters, w->n_counters * sizeof(int)) == cudaSuccess;
  ok &= cudaMalloc(&w->prefill_tiles, (T + 2) * sizeof(int)) == cudaSuccess;
  const size_t part_rows = T < 1024 ? T : 1024;
  w->attn_part_elems = part_rows * H * 16 * (128 + 2);
  ok &= cudaMalloc(&w->attn_part, w->attn_part_elems * sizeof(float)) == cudaSuccess;
  ok &= cudaMalloc(&w->d_tokens, T * sizeof(be_token)) == cudaSuccess;
  w->pt_capacity = (size_t)max_rows * max_pages;
  ok &= cudaMalloc(&w->d_pt, w->pt_capacity * sizeof(int32_t)) == cudaSuccess;
  if (!ok) {
    be_workspace_free(w);
    return fail(ctx, BE_ERR_NOMEM, "workspace allocation failed (max_tok=%d)", max_tok);
  }
  cudaMemsetAsync(w->counters, 0, w->n_counters * sizeof(int), ctx->stream);
  cudaMemsetAsync(w->X, 0, T * d * sizeof(float), ctx->stream);
  cudaMemsetAsync(w->Xb, 0, T * d * sizeof(bf16), ctx->stream);
  cudaMemsetAsync(w->attn, 0, T * d * sizeof(bf16), ctx->stream);
  cudaMemsetAsync(w->h, 0, T * dff * sizeof(bf16), ctx->stream);
  for (int bn : kBNs) {
    CUtensorMap a, b2, c;
    int rc;
    if ((rc = make_map(ctx, &a, w->Xb, T, d, bn)) != BE_OK ||
        (rc = make_map(ctx, &b2, w->attn, T, d, bn)) != BE_OK ||
        (rc = make_map(ctx, &c, w->h, T, dff, bn)) != BE_OK) {
      be_workspace_free(w);
      return rc;
    }
    w->m_xb[bn] = a;
    w->m_attn[bn] = b2;
    w->m_h[bn] = c;
  }
  *out = w;
  return BE_OK;
}

extern "C" int be_workspace_free(be_workspace* w) {
  if (w == nullptr) return BE_ERR_INVALID;
  cudaSetDevice(w->ctx->device);
  void* ptrs[] = {w->X, w->Xb, w->q, w->attn, w->h, w->ss, w->rstd, w->splitws, w->counters, w->prefill_tiles,
                  w->attn_part, w->d_tokens, w->d_pt, w->lora_u, w->d_lora_idx};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete w;
  return BE_OK;
}

// ------------------------------------------------------------------------------ profiling
namespace {

cudaEvent_t prof_event(be_ctx* ctx) {
  if (ctx->prof_ev_used == ctx->prof_ev.size()) {
    cudaEvent_t ev;
    if (cudaEventCreate(&ev) != cudaSuccess) return nullptr;
    ctx->prof_ev.push_back(ev);
  }
  return ctx->prof_ev[ctx->prof_ev_used++];
}

// Brackets one launch with events on its stream when profiling is on.
struct ProfScope {
  be_ctx* ctx;
  cudaStream_t st;
  int idx = -1;
  ProfScope(be_ctx* c, cudaStream_t s, int cls, int ntok, int N, int K, double bytes,
            double flops)
      : ctx(c), st(s) {
    if (!ctx->prof) return;
    cudaEvent_t a = prof_event(ctx), b = prof_event(ctx);
    if (a == nullptr || b == nullptr) return;
    be_ctx::ProfRec rec{};
    rec.r.cls = cls;
    rec.r.ntok = ntok;
    rec.r.n = N;
    rec.r.k = K;
    rec.r.bytes = bytes;
    rec.r.flops = flops;
    rec.a = a;
    rec.b = b;
    cudaEventRecord(a, st);
    idx = (int)ctx->prof_recs.size();
    ctx->prof_recs.push_back(rec);
  }
  ~ProfScope() {
    if (idx >= 0) cudaEventRecord(ctx->prof_recs[idx].b, st);
  }
};



// next timeline slot for a launch of class cls (nullptr when the timeline is off or full)
unsigned long long* tl_slot(be_ctx* ctx, int cls) {
  if (ctx->tl == nullptr || ctx->tl_next >= ctx->tl_cap) return nullptr;
  const int s = ctx->tl_next++;
  if ((int)ctx->tl_cls.size() <= s) ctx->tl_cls.resize(s + 1);
  ctx->tl_cls[s] = cls;
  return ctx->tl + s;
}

}  // namespace

extern "C" int be_timeline_enable(be_ctx* ctx, int cap) {
  if (ctx == nullptr || cap < 0) return BE_ERR_INVALID;
  cudaSetDevice(ctx->device);
  BE_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->tl) cudaFree(ctx->tl);
  ctx->tl = nullptr;
  ctx->tl_cap = 0;
  ctx->tl_next = 0;
  ctx->tl_cls.clear();
  if (cap == 0) return BE_OK;
  BE_CUDA(ctx, cudaMalloc(&ctx->tl, (size_t)4 * cap * sizeof(unsigned long long)));
  ctx->tl_cap = cap;
  return BE_OK;
}

extern "C" int be_timeline_begin(be_ctx* ctx) {
  if (ctx == nullptr || ctx->tl == nullptr) return BE_ERR_INVALID;
  ctx->tl_next = 0;
  const size_t n = (size_t)ctx->tl_cap * sizeof(unsigned long long);
  BE_CUDA(ctx, cudaMemsetAsync(ctx->tl, 0xff, n, ctx->stream));                    // min start
  BE_CUDA(ctx, cudaMemsetAsync(ctx->tl + ctx->tl_cap, 0, n, ctx->stream));         // max start
  BE_CUDA(ctx, cudaMemsetAsync(ctx->tl + 2 * ctx->tl_cap, 0xff, n, ctx->stream));  // min go
  BE_CUDA(ctx, cudaMemsetAsync(ctx->tl + 3 * ctx->tl_cap, 0, n, ctx->stream));     // max end
  return BE_OK;
}

extern "C" int be_timeline_read(be_ctx* ctx, be_timeline_rec* out, int cap, int* n_out) {
  if (ctx == nullptr || n_out == nullptr || ctx->tl == nullptr) return BE_ERR_INVALID;
  BE_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<unsigned long long> h((size_t)4 * ctx->tl_cap);
  BE_CUDA(ctx, cudaMemcpy(h.data(), ctx->tl, h.size() * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost));
  int n = 0;
  for (int s = 0; s < ctx->tl_cap && s < (int)ctx->tl_cls.size(); ++s) {
    if (h[3 * ctx->tl_cap + s] == 0) continue;  // slot not written in this window
    if (out != nullptr && n < cap) {
      out[n].slot = s;
      out[n].cls = ctx->tl_cls[s];
      out[n].start_first = h[s];
      out[n].start_last = h[ctx->tl_cap + s];
      out[n].go_first = h[2 * ctx->tl_cap + s];
      out[n].end_last = h[3 * ctx->tl_cap + s];
    }
    ++n;
  }
  *n_out = n;
  return BE_OK;
}

extern "C" int be_prof_enable(be_ctx* ctx, int on) {
  if (ctx == nullptr) return BE_ERR_INVALID;
  ctx->prof = on != 0;
  ctx->prof_recs.clear();
  ctx->prof_ev_used = 0;
  return BE_OK;
}

extern "C" int be_prof_active(const be_ctx* ctx) { return ctx != nullptr && ctx->prof ? 1 : 0; }

extern "C" int be_prof_read(be_ctx* ctx, be_prof_rec* out, int cap, int* n_out) {
  if (ctx == nullptr || n_out == nullptr || (cap > 0 && out == nullptr)) return BE_ERR_INVALID;
  BE_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  const int n = (int)ctx->prof_recs.size();
  *n_out = n;
  if (cap < n) return BE_OK;  // size query
  for (int i = 0; i < n; ++i) {
    auto& rec = ctx->prof_recs[i];
    float ms = 0.f;
    BE_CUDA(ctx, cudaEventElapsedTime(&ms, rec.a, rec.b));
    out[i] = rec.r;
    out[i].ms = ms;
  }
  ctx->prof_recs.clear();
  ctx->prof_ev_used = 0;
  return BE_OK;
}

// ------------------------------------------------------------------------------ execution
namespace {

// algorithmic bytes of one GEMM: weights + activations in + outputs
double gemm_bytes(int N, int K, int ntok) {
  return 2.0 * ((double)N * K + (double)ntok * K + (double)ntok * N);
}

int run_gemm(be_ctx* ctx, be_workspace* ws, const bf16* w_packed, const CUtensorMap* mx, int N,
             int K, int ntok, int bn, EpiParams epi, cudaStream_t st) {
  bx::GemmLaunch L{};
  L.w_packed = w_packed;
  L.map_x = mx;
  L.N = N;
  L.K = K;
  L.bn = bn;
  const bx::GemmPlan p = bx::gemm_plan(N, K, ntok, bn, ctx->num_sms, ws->splitws_elems,
                                       ws->n_counters, ctx->gemm_grid_cap);
  if (p.ws_needed > ws->splitws_elems || p.tiles > ws->n_counters)
    return fail(ctx, BE_ERR_INVALID, "gemm N=%d K=%d ntok=%d: stream-K workspace too small", N, K, ntok);
  L.grid = p.grid;
  L.rr = p.rr;
  L.pdl = ctx->use_pdl;
  epi.ws = ws->splitws;
  epi.counters = ws->counters;
  cudaError_t e = cudaSuccess;
  if (p.rr && epi.ss_in != nullptr && epi.n_grp <= 1) {
    // prefill: every weight tile of a token tile needs the same per-token rstd - reduce once
    e = bx::launch_rstd(epi.ss_in, epi.ss_groups, ntok, epi.norm_eps, ws->rstd, st);
    if (e != cudaSuccess) return fail(ctx, BE_ERR_CUDA, "rstd: %s", cudaGetErrorString(e));
    epi.rs_in = ws->rstd;
  }
  L.epi = epi;
  e = bx::launch_gemm(L, st);
  if (e != cudaSuccess)
    return fail(ctx, BE_ERR_CUDA, "gemm N=%d K=%d ntok=%d: %s", N, K, ntok, cudaGetErrorString(e));
  return BE_OK;
}

// One batch of one block, or a grouped batch of n_grp independent blocks of one shape whose
// token rows sit side by side in groups of grp_rows = ntok / n_grp (one GEMM n-tile each).
int check_loras(be_ctx* ctx, const be_block* blk, int n_lora, const be_lora* const* loras);
// Adapters of one launch: token t uses loras[idx[t]] (idx on the device, -1 = base block only)
struct LoraSet {
  int n = 0;
  const be_lora* const* loras = nullptr;
  const int32_t* idx = nullptr;
};

int exec_dev(be_ctx* ctx, int n_grp, be_block* const* blks, be_kv_pool* const* pools,
             be_workspace* ws, int phase, int ntok, const be_token* d_tok, int pt_stride,
             const int32_t* d_pt, const void* arena_in, void* arena_out, cudaStream_t st,
             const LoraSet* lora = nullptr) {
  be_block* blk = blks[0];
  be_kv_pool* pool = pools[0];
  cudaSetDevice(ctx->device);  // several contexts (GPUs) may share one host thread
  const auto& D = blk->desc;
  const int d = D.d_model, F = D.d_ff, H = D.n_heads, hd = D.head_dim;
  // a workspace serves any block of its d_model / heads with d_ff <= its own (pruned surrogates)
  if (ws->d != d || ws->dff < F || ws->H != H)
    return fail(ctx, BE_ERR_INVALID, "workspace shape does not match block");
  if (ntok > ws->max_tok) return fail(ctx, BE_ERR_INVALID, "batch of %d tokens > workspace %d", ntok, ws->max_tok);
  if (pool->n_layers != blk->n_att || pool->n_heads != H || pool->head_dim != hd)
    return fail(ctx, BE_ERR_INVALID, "kv pool shape does not match block");
  if (ntok == 0) return BE_OK;
  const int* tok = reinterpret_cast<const int*>(d_tok);
  const int grp_rows = n_grp > 1 ? ntok / n_grp : ntok;
  // grouped blocks stream their own weights per n-tile (BN = rows per block); LoRA variants of one
  // base share its weights, so their rows form one matrix streamed once
  const int bn = n_grp > 1 && lora == nullptr ? grp_rows : bx::gemm_pick_bn(ntok);
  // narrow GEMMs (O, down: N = d, <= 40 weight tiles) at 129-256 rows: 128-token tiles halve the
  // split-tile partials (128 KB at 256 tokens) the stream-K owners must read; wide GEMMs keep
  // 256-token tiles (one weight stream). Prefill widths (round-robin) are unaffected.
  static const bool kNarrowBn128 = [] {
    const char* e = getenv("BE_GEMM_NARROW_BN128");
    return e ? atoi(e) != 0 : true;
  }();
  auto bn_narrow = [&](int N) {
    return kNarrowBn128 && n_grp == 1 && lora == nullptr && bn == 256 && ntok <= 256 &&
                   N / bx::kBM <= 40
               ? 128
               : bn;
  };
  const int wcopies = lora != nullptr ? 1 : n_grp;  // weight streams per GEMM (byte accounting)
  if (n_grp > 1) {
    if (n_grp > bx::kMaxGroup || ntok % n_grp != 0 || (grp_rows != 16 && grp_rows != 32 && grp_rows != 64))
      return fail(ctx, BE_ERR_INVALID, "grouped batch: %d blocks x %d rows unsupported", n_grp, grp_rows);
    for (int g = 1; g < n_grp; ++g) {
      const be_block* b = blks[g];
      if (b->comps != blk->comps || b->desc.d_model != d || b->desc.d_ff != F ||
          b->desc.n_heads != H || pools[g]->page_elems != pool->page_elems ||
          pools[g]->n_layers != blk->n_att)
        return fail(ctx, BE_ERR_INVALID, "grouped batch: blocks differ in shape");
    }
  }
  // per-GEMM group tables: the weights of block g for n-tile g
  auto group = [&](EpiParams& E, bf16* const be_block::Layer::*w, int li) {
    E.n_grp = n_grp;
    E.grp_rows = grp_rows;
    for (int g = 0; g < n_grp; ++g) {
      E.wgrp[g] = blks[g]->layers[li].*w;
      E.kvgrp[g] = pools[g]->base;
    }
  };
  cudaError_t e;

  // K1: gather the members' input rows into the batch (fp32 residual + bf16 shadow)
  {
    ProfScope ps(ctx, st, BE_K_GATHER, ntok, d, 0, 8.0 * ntok * d, 0);
    e = bx::launch_gather(static_cast<const bf16*>(arena_in), tok + 0, 5, ntok, d, ws->Xb, ws->X,
                          ws->ss, st, tl_slot(ctx, BE_K_GATHER), ctx->tl_cap);
  }
  if (e != cudaSuccess) return fail(ctx, BE_ERR_CUDA, "gather: %s", cudaGetErrorString(e));

  const int max_pages = pt_stride;
  int splits = attn_splits(ctx, ntok, H, max_pages);
  // a forced split count (tests / experiments) applies where its partials fit (decode sizes)
  if (ctx->attn_splits_force > 0 && (size_t)ntok * H * splits * (hd + 2) > ws->attn_part_elems)
    splits = 1;
  if ((size_t)ntok * H * splits * (hd + 2) > ws->attn_part_elems && splits > 1)
    return fail(ctx, BE_ERR_INVALID, "attention partial buffer too small");

  int ia = 0, jf = 0;
  const int n_comp = (int)blk->comps.size();
  int ci = -1;
  // the block's last GEMM writes the next-hop rows itself (kResidOut: K2 fused in its epilogue)
  auto finish = [&](EpiParams& e) {
    if (ci != n_comp - 1) return;
    e.mode = bx::kResidOut;
    e.out = static_cast<bf16*>(arena_out);
    e.ldo = d;
    e.tok = tok;
    e.ss_out = nullptr;
  };
  for (char kind : blk->comps) {
    int rc;
    ++ci;
    if (kind == 'f') {
      // ---- ffn component: RMSNorm (fused) -> gate/up + SwiGLU -> down + residual
      const int li = jf;
      const auto& L = blk->layers[jf++];
      EpiParams eg{};
      group(eg, &be_block::Layer::wgu, li);
      eg.mode = bx::kSwiGLU;
      eg.ntok = ntok;
      eg.ss_in = ws->ss;
      eg.ss_groups = d / 32;
      eg.norm_eps = D.norm_eps;
      eg.out = ws->h;
      eg.ldo = ws->dff;  // row stride of h (its TMA map); the down GEMM reads the first F columns
      {
        eg.tl = tl_slot(ctx, BE_K_GEMM_GATE_UP);
        eg.tl_cap = ctx->tl_cap;
        ProfScope ps(ctx, st, BE_K_GEMM_GATE_UP, ntok, 2 * F, d, gemm_bytes(2 * F, d, ntok) + 2.0 * (wcopies - 1) * (2 * F) * (d),
                     2.0 * (2 * F) * (d) * ntok);
        rc = run_gemm(ctx, ws, L.wgu, &ws->m_xb[bn], 2 * F, d, ntok, bn, eg, st);
      }
      if (rc != BE_OK) return rc;
      EpiParams ed{};
      group(ed, &be_block::Layer::wd, li);
      ed.mode = bx::kResid;
      ed.ntok = ntok;
      ed.xres = ws->X;
      ed.xres_b = ws->Xb;
      ed.ldr = d;
      ed.ss_out = ws->ss;  // the next component's RMSNorm statistics
      ed.ss_groups = d / 32;
      finish(ed);
      {
        ed.tl = tl_slot(ctx, BE_K_GEMM_DOWN);
        ed.tl_cap = ctx->tl_cap;
        ProfScope ps(ctx, st, BE_K_GEMM_DOWN, ntok, d, F, gemm_bytes(d, F, ntok) + 2.0 * (wcopies - 1) * (d) * (F),
                     2.0 * (d) * (F) * ntok);
        rc = run_gemm(ctx, ws, L.wd, &ws->m_h[bn_narrow(d)], d, F, ntok, bn_narrow(d), ed, st);
      }
      if (rc != BE_OK) return rc;
      continue;
    }
    const int l = ia++;
    const auto& L = blk->layers[l];
    // ---- attention component: RMSNorm (fused) -> QKV + RoPE + KV append -> paged attn -> O + residual
    EpiParams eq{};
    group(eq, &be_block::Layer::wqkv, l);
    eq.mode = bx::kQKV;
    eq.ntok = ntok;
    eq.ss_in = ws->ss;
    eq.ss_groups = d / 32;
    eq.norm_eps = D.norm_eps;
    eq.out = ws->q;
    eq.ldo = d;
    eq.tok = tok;
    eq.kv_pool = pool->base;
    eq.page_elems = pool->page_elems;
    eq.layer_elems = pool->layer_elems;
    eq.layer = l;
    eq.d_model = d;
    eq.head_dim = hd;
    eq.rope = blk->rope;
    if (lora != nullptr) {
      // segmented LoRA: u = rstd * A_qkv x per token (its adapter), delta added in the epilogue
      bx::LoraTable ta{}, tb{};
      for (int a = 0; a < lora->n; ++a) {
        ta.p[a] = lora->loras[a]->layers[l].aqkv;
        tb.p[a] = lora->loras[a]->layers[l].bqkv;
      }
      e = bx::launch_lora_shrink(ws->Xb, d, d, ws->ss, d / 32, D.norm_eps, ta, 3 * bx::kLoraRank,
                                 lora->idx, ws->lora_u, ntok, st);
      if (e != cudaSuccess) return fail(ctx, BE_ERR_CUDA, "lora shrink: %s", cudaGetErrorString(e));
      eq.mode = bx::kQKVLora;
      eq.lora_u = ws->lora_u;
      eq.lora_ustride = 3 * bx::kLoraRank;
      eq.lora_seg = d;
      eq.lora_idx = lora->idx;
      eq.lora_b = tb;
    }
    {
      eq.tl = tl_slot(ctx, BE_K_GEMM_QKV);
        eq.tl_cap = ctx->tl_cap;
        ProfScope ps(ctx, st, BE_K_GEMM_QKV, ntok, 3 * d, d, gemm_bytes(3 * d, d, ntok) + 2.0 * (wcopies - 1) * (3 * d) * (d),
                     2.0 * (3 * d) * (d) * ntok);
      rc = run_gemm(ctx, ws, L.wqkv, &ws->m_xb[bn], 3 * d, d, ntok, bn, eq, st);
    }
    if (rc != BE_OK) return rc;

    bx::AttnParams ap{};
    ap.q = ws->q;
    ap.pool = pool->base;
    ap.page_elems = pool->page_elems;
    ap.layer_elems = pool->layer_elems;
    ap.layer = l;
    ap.page_table = d_pt;
    ap.pt_stride = pt_stride;
    ap.row_pt = tok + 4;
    ap.row_ctx = tok + 3;
    ap.meta_stride = 5;
    ap.ctx_add = 1;  // a token sees positions [0, pos]
    ap.H = H;
    ap.scale_log2 = (1.0f / sqrtf((float)hd)) * 1.4426950408889634f;
    ap.out = ws->attn;
    ap.part = ws->attn_part;
    ap.splits = splits;
    ap.n_grp = n_grp;
    ap.grp_rows = grp_rows;
    for (int g = 0; g < n_grp; ++g) ap.pools[g] = pools[g]->base;
    ap.tl = tl_slot(ctx, BE_K_ATTENTION);
    ap.tl_cap = ctx->tl_cap;
    if (ap.tl != nullptr && splits > 1) tl_slot(ctx, BE_K_ATTENTION);  // combine's slot = tl + 1
    {
      ProfScope ps(ctx, st, BE_K_ATTENTION, ntok, H, hd, 0, 0);
      if (phase == BE_PHASE_PREFILL && n_grp == 1 && (ctx->prefill_tc == 1 || ctx->prefill_tc == 4) &&
          hd == 128) {
        // prompt rows on tcgen05: S and O in TMEM, Q / K / V tiles by TMA
        if (!ws->has_m_q) {
          if (make_map(ctx, &ws->m_q, ws->q, ws->max_tok, (uint64_t)H * hd, 128) != BE_OK)
            return BE_ERR_CUDA;
          ws->has_m_q = true;
        }
        if (!pool->has_m_kv) {
          cuuint64_t dims[5] = {(cuuint64_t)hd, 16, (cuuint64_t)H, 2,
                                (cuuint64_t)pool->n_pages * pool->n_layers};
          cuuint64_t strides[4] = {(cuuint64_t)hd * 2, (cuuint64_t)16 * hd * 2,
                                   (cuuint64_t)H * 16 * hd * 2, (cuuint64_t)pool->layer_elems * 2};
          cuuint32_t box[5] = {64, 16, 1, 1, 1};
          cuuint32_t estr[5] = {1, 1, 1, 1, 1};
          const CUresult r = ctx->encode(&pool->m_kv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                                         pool->base, dims, strides, box, estr,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) return fail(ctx, BE_ERR_CUDA, "kv pool tensor map (%d)", (int)r);
          pool->has_m_kv = true;
        }
        bx::PrefillTcParams pt{};
        pt.page_table = d_pt;
        pt.pt_stride = pt_stride;
        pt.tok = tok;
        pt.rows = ntok;
        pt.H = H;
        pt.layer = l;
        pt.n_layers = pool->n_layers;
        pt.scale_log2 = ap.scale_log2;
        pt.out = ws->attn;
        pt.tiles = ws->prefill_tiles;
        e = ctx->prefill_tc == 4
                ? bx::launch_attention_prefill_pipe(pt, ws->m_q, pool->m_kv, ctx->num_sms, st)
                : bx::launch_attention_prefill_tc(pt, ws->m_q, pool->m_kv, ctx->num_sms, st);
      } else if (phase == BE_PHASE_PREFILL && n_grp == 1 && ctx->prefill_tc) {
        // prompt rows: query tiles share K/V tiles on tensor cores
        bx::PrefillAttnParams pp{};
        pp.q = ws->q;
        pp.pool = pool->base;
        pp.page_elems = pool->page_elems;
        pp.layer_elems = pool->layer_elems;
        pp.layer = l;
        pp.page_table = d_pt;
        pp.pt_stride = pt_stride;
        pp.tok = tok;
        pp.rows = ntok;
        pp.H = H;
        pp.scale_log2 = ap.scale_log2;
        pp.out = ws->attn;
        pp.tiles = ws->prefill_tiles;
        e = bx::launch_attention_prefill(pp, hd, ctx->num_sms, st);
      } else {
        e = bx::launch_attention(ap, ntok, hd, st);
      }
    }
    if (e != cudaSuccess) return fail(ctx, BE_ERR_CUDA, "attention: %s", cudaGetErrorString(e));

    EpiParams eo{};
    group(eo, &be_block::Layer::wo, l);
    eo.mode = bx::kResid;
    eo.ntok = ntok;
    eo.xres = ws->X;
    eo.xres_b = ws->Xb;
    eo.ldr = d;
    eo.ss_out = ws->ss;
    eo.ss_groups = d / 32;
    finish(eo);
    if (lora != nullptr) {
      bx::LoraTable ta{}, tb{};
      for (int a = 0; a < lora->n; ++a) {
        ta.p[a] = lora->loras[a]->layers[l].ao;
        tb.p[a] = lora->loras[a]->layers[l].bo;
      }
      e = bx::launch_lora_shrink(ws->attn, d, d, nullptr, d / 32, 0.f, ta, bx::kLoraRank,
                                 lora->idx, ws->lora_u, ntok, st);
      if (e != cudaSuccess) return fail(ctx, BE_ERR_CUDA, "lora shrink: %s", cudaGetErrorString(e));
      eo.mode = eo.mode == bx::kResidOut ? bx::kResidOutLora : bx::kResidLora;
      eo.lora_u = ws->lora_u;
      eo.lora_ustride = bx::kLoraRank;
      eo.lora_seg = d;
      eo.lora_idx = lora->idx;
      eo.lora_b = tb;
    }
    {
      eo.tl = tl_slot(ctx, BE_K_GEMM_O);
        eo.tl_cap = ctx->tl_cap;
        ProfScope ps(ctx, st, BE_K_GEMM_O, ntok, d, d, gemm_bytes(d, d, ntok) + 2.0 * (wcopies - 1) * (d) * (d),
                     2.0 * (d) * (d) * ntok);
      rc = run_gemm(ctx, ws, L.wo, &ws->m_attn[bn_narrow(d)], d, d, ntok, bn_narrow(d), eo, st);
    }
    if (rc != BE_OK) return rc;
  }
  // K2 (the scatter to the next-hop rows) ran inside the last GEMM's epilogue (kResidOut)
  return BE_OK;
}

}  // namespace

extern "C" int be_exec_batch_dev(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws,
                                 int phase, int n_tokens, const be_token* d_tokens, int pt_stride,
                                 const int32_t* d_page_table, const void* d_arena_in,
                                 void* d_arena_out, void* stream) {
  if (ctx == nullptr || blk == nullptr || pool == nullptr || ws == nullptr || n_tokens < 0 ||
      (n_tokens > 0 && (d_tokens == nullptr || d_page_table == nullptr || d_arena_in == nullptr ||
                        d_arena_out == nullptr)) ||
      pt_stride <= 0)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_exec_batch_dev: bad arguments") : BE_ERR_INVALID;
  if (phase != BE_PHASE_PREFILL && phase != BE_PHASE_DECODE)
    return fail(ctx, BE_ERR_INVALID, "unknown phase %d", phase);
  return exec_dev(ctx, 1, &blk, &pool, ws, phase, n_tokens, d_tokens, pt_stride, d_page_table,
                  d_arena_in, d_arena_out, pick_stream(ctx, stream));
}

extern "C" int be_exec_group_dev(be_ctx* ctx, int n_blocks, be_block* const* blks,
                                 be_kv_pool* const* pools, be_workspace* ws, int phase,
                                 int n_tokens, const be_token* d_tokens, int pt_stride,
                                 const int32_t* d_page_table, const void* d_arena_in,
                                 void* d_arena_out, void* stream) {
  if (ctx == nullptr || n_blocks < 1 || blks == nullptr || pools == nullptr || ws == nullptr ||
      n_tokens <= 0 || d_tokens == nullptr || d_page_table == nullptr || d_arena_in == nullptr ||
      d_arena_out == nullptr || pt_stride <= 0)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_exec_group_dev: bad arguments") : BE_ERR_INVALID;
  for (int g = 0; g < n_blocks; ++g)
    if (blks[g] == nullptr || pools[g] == nullptr)
      return fail(ctx, BE_ERR_INVALID, "be_exec_group_dev: null block or pool");
  if (phase != BE_PHASE_PREFILL && phase != BE_PHASE_DECODE)
    return fail(ctx, BE_ERR_INVALID, "unknown phase %d", phase);
  return exec_dev(ctx, n_blocks, blks, pools, ws, phase, n_tokens, d_tokens, pt_stride,
                  d_page_table, d_arena_in, d_arena_out, pick_stream(ctx, stream));
}

extern "C" int be_exec_lora_group_dev(be_ctx* ctx, int n_blocks, be_block* const* blks,
                                      be_kv_pool* const* pools, be_workspace* ws, int phase,
                                      int n_tokens, const be_token* d_tokens, int pt_stride,
                                      const int32_t* d_page_table, int n_lora,
                                      const be_lora* const* loras, const int32_t* d_lora_idx,
                                      const void* d_arena_in, void* d_arena_out, void* stream) {
  if (ctx == nullptr || n_blocks < 1 || blks == nullptr || pools == nullptr || ws == nullptr ||
      n_tokens <= 0 || d_tokens == nullptr || d_page_table == nullptr || d_lora_idx == nullptr ||
      d_arena_in == nullptr || d_arena_out == nullptr || pt_stride <= 0)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_exec_lora_group_dev: bad arguments") : BE_ERR_INVALID;
  for (int g = 0; g < n_blocks; ++g)
    if (blks[g] == nullptr || pools[g] == nullptr || blks[g] != blks[0])
      return fail(ctx, BE_ERR_INVALID, "be_exec_lora_group_dev: the groups must share one base block");
  int rc = check_loras(ctx, blks[0], n_lora, loras);
  if (rc != BE_OK) return rc;
  if (phase != BE_PHASE_PREFILL && phase != BE_PHASE_DECODE)
    return fail(ctx, BE_ERR_INVALID, "unknown phase %d", phase);
  LoraSet set{n_lora, loras, d_lora_idx};
  return exec_dev(ctx, n_blocks, blks, pools, ws, phase, n_tokens, d_tokens, pt_stride,
                  d_page_table, d_arena_in, d_arena_out, pick_stream(ctx, stream), &set);
}

namespace {
int exec_batch_host(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws, int phase,
                    int n_tokens, const be_token* tokens, int n_pt_rows, int pt_stride,
                    const int32_t* page_table, const void* d_arena_in, void* d_arena_out,
                    cudaStream_t stream, const LoraSet* lora);
}  // namespace

extern "C" int be_exec_batch(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws,
                             int phase, int n_tokens, const be_token* tokens, int n_pt_rows,
                             int pt_stride, const int32_t* page_table, const void* d_arena_in,
                             void* d_arena_out, void* stream) {
  return exec_batch_host(ctx, blk, pool, ws, phase, n_tokens, tokens, n_pt_rows, pt_stride,
                         page_table, d_arena_in, d_arena_out,
                         ctx ? pick_stream(ctx, stream) : nullptr, nullptr);
}

namespace {
int exec_batch_host(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws, int phase,
                    int n_tokens, const be_token* tokens, int n_pt_rows, int pt_stride,
                    const int32_t* page_table, const void* d_arena_in, void* d_arena_out,
                    cudaStream_t stream, const LoraSet* lora) {
  if (ctx == nullptr || blk == nullptr || pool == nullptr || ws == nullptr || n_tokens < 0 ||
      (n_tokens > 0 && tokens == nullptr) || pt_stride <= 0 || n_pt_rows < 0)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_exec_batch: bad arguments") : BE_ERR_INVALID;
  if (n_tokens > ws->max_tok)
    return fail(ctx, BE_ERR_INVALID, "batch of %d tokens > workspace %d", n_tokens, ws->max_tok);
  if ((size_t)n_pt_rows * pt_stride > ws->pt_capacity)
    return fail(ctx, BE_ERR_INVALID, "page table %dx%d exceeds workspace", n_pt_rows, pt_stride);
  // host-side validation of the routing metadata (the kernels trust it)
  const int64_t kv_slots = (int64_t)pool->n_pages * 16;
  for (int t = 0; t < n_tokens; ++t) {
    const be_token& k = tokens[t];
    if (k.pt_row < 0 || k.pt_row >= n_pt_rows || k.pos < 0 || k.kv_slot < 0 ||
        k.kv_slot >= kv_slots || (k.kv_slot & 15) != (k.pos & 15) || k.src_row < 0 ||
        (k.pos >> 4) >= pt_stride || k.pos >= blk->desc.max_pos)
      return fail(ctx, BE_ERR_INVALID, "token %d: inconsistent routing metadata", t);
  }
  for (int64_t i = 0; i < (int64_t)n_pt_rows * pt_stride; ++i)
    if (page_table[i] < -1 || page_table[i] >= pool->n_pages)
      return fail(ctx, BE_ERR_INVALID, "page table entry %lld out of range", (long long)i);
  // attention reads pages 0..pos>>4 of the token's row without a guard, and the QKV epilogue
  // appends K/V at kv_slot: every page up to the token's must be mapped, the last one to the
  // page holding kv_slot (blocks without attention components touch no KV page)
  for (int t = 0; t < n_tokens && blk->n_att > 0; ++t) {
    const be_token& k = tokens[t];
    const int32_t* row = page_table + (size_t)k.pt_row * pt_stride;
    for (int p = 0; p <= (k.pos >> 4); ++p)
      if (row[p] < 0)
        return fail(ctx, BE_ERR_INVALID, "token %d: page %d of its page-table row is unmapped", t, p);
    if (row[k.pos >> 4] != (k.kv_slot >> 4))
      return fail(ctx, BE_ERR_INVALID, "token %d: kv_slot %d is not on page-table page %d", t,
                  k.kv_slot, row[k.pos >> 4]);
  }
  cudaSetDevice(ctx->device);
  cudaStream_t st = stream;
  if (n_tokens > 0)
    BE_CUDA(ctx, cudaMemcpyAsync(ws->d_tokens, tokens, n_tokens * sizeof(be_token),
                                 cudaMemcpyHostToDevice, st));
  if (n_pt_rows > 0)
    BE_CUDA(ctx, cudaMemcpyAsync(ws->d_pt, page_table, (size_t)n_pt_rows * pt_stride * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, st));
  return exec_dev(ctx, 1, &blk, &pool, ws, phase, n_tokens, ws->d_tokens, pt_stride, ws->d_pt,
                  d_arena_in, d_arena_out, st, lora);
}
}  // namespace

// ------------------------------------------------------------------------------ LoRA adapters
extern "C" int be_lora_load(be_ctx* ctx, const be_block* base, const char* name, uint64_t seed,
                            float scale_a, float scale_b, be_lora** out) {
  if (ctx == nullptr || base == nullptr || name == nullptr || out == nullptr)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_lora_load: bad arguments") : BE_ERR_INVALID;
  if (base->n_att == 0) return fail(ctx, BE_ERR_INVALID, "be_lora_load: block has no attention");
  cudaSetDevice(ctx->device);
  constexpr int r = bx::kLoraRank;
  const size_t D = base->desc.d_model;
  const size_t per_layer = 3 * r * D + 3 * D * r + r * D + D * r;
  auto* L = new be_lora();
  L->ctx = ctx;
  L->d = (int)D;
  L->n_att = base->n_att;
  if (cudaMalloc(&L->slab, per_layer * L->n_att * sizeof(bf16)) != cudaSuccess) {
    delete L;
    return fail(ctx, BE_ERR_NOMEM, "be_lora_load: allocation failed");
  }
  cudaStream_t st = ctx->stream;
  const int hd = base->desc.head_dim;
  bf16* cur = L->slab;
  for (int l = 0; l < L->n_att; ++l) {
    be_lora::Layer Y{cur, cur + 3 * r * D, cur + 6 * r * D, cur + 7 * r * D};
    cur += per_layer;
    auto key = [&](const char* t) {
      return stream_key(seed, std::string("lora:") + name + ":" + std::to_string(l) + ":" + t);
    };
    // A rows: logical order; B rows: the GEMM's physical row order (q/k pair interleave)
    bx::launch_synth_plain(Y.aqkv, r, (int)D, key("aq"), scale_a, 0, hd, st);
    bx::launch_synth_plain(Y.aqkv + r * D, r, (int)D, key("ak"), scale_a, 0, hd, st);
    bx::launch_synth_plain(Y.aqkv + 2 * r * D, r, (int)D, key("av"), scale_a, 0, hd, st);
    bx::launch_synth_plain(Y.bqkv, (int)D, r, key("bq"), scale_b, 1, hd, st);
    bx::launch_synth_plain(Y.bqkv + D * r, (int)D, r, key("bk"), scale_b, 1, hd, st);
    bx::launch_synth_plain(Y.bqkv + 2 * D * r, (int)D, r, key("bv"), scale_b, 0, hd, st);
    bx::launch_synth_plain(Y.ao, r, (int)D, key("ao"), scale_a, 0, hd, st);
    bx::launch_synth_plain(Y.bo, (int)D, r, key("bo"), scale_b, 0, hd, st);
    L->layers.push_back(Y);
  }
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    cudaFree(L->slab);
    delete L;
    return fail(ctx, BE_ERR_CUDA, "be_lora_load: %s", cudaGetErrorString(e));
  }
  *out = L;
  return BE_OK;
}

extern "C" int be_lora_free(be_lora* l) {
  if (l == nullptr) return BE_ERR_INVALID;
  cudaSetDevice(l->ctx->device);
  if (l->slab) cudaFree(l->slab);
  delete l;
  return BE_OK;
}

namespace {
int check_loras(be_ctx* ctx, const be_block* blk, int n_lora, const be_lora* const* loras) {
  if (n_lora < 1 || n_lora > bx::kMaxLora || loras == nullptr)
    return fail(ctx, BE_ERR_INVALID, "lora batch: 1..%d adapters", bx::kMaxLora);
  for (int a = 0; a < n_lora; ++a)
    if (loras[a] == nullptr || loras[a]->d != blk->desc.d_model || loras[a]->n_att != blk->n_att)
      return fail(ctx, BE_ERR_INVALID, "lora batch: adapter %d does not fit the block", a);
  return BE_OK;
}
}  // namespace

extern "C" int be_exec_lora_batch_dev(be_ctx* ctx, be_block* blk, be_kv_pool* pool,
                                      be_workspace* ws, int phase, int n_tokens,
                                      const be_token* d_tokens, int pt_stride,
                                      const int32_t* d_page_table, int n_lora,
                                      const be_lora* const* loras, const int32_t* d_lora_idx,
                                      const void* d_arena_in, void* d_arena_out, void* stream) {
  if (ctx == nullptr || blk == nullptr || pool == nullptr || ws == nullptr || n_tokens <= 0 ||
      d_tokens == nullptr || d_page_table == nullptr || d_lora_idx == nullptr ||
      d_arena_in == nullptr || pt_stride <= 0 || n_tokens > ws->max_tok)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_exec_lora_batch_dev: bad arguments") : BE_ERR_INVALID;
  int rc = check_loras(ctx, blk, n_lora, loras);
  if (rc != BE_OK) return rc;
  LoraSet set{n_lora, loras, d_lora_idx};
  return exec_dev(ctx, 1, &blk, &pool, ws, phase, n_tokens, d_tokens, pt_stride, d_page_table,
                  d_arena_in, d_arena_out, pick_stream(ctx, stream), &set);
}

extern "C" int be_exec_lora_batch(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws,
                                  int phase, int n_tokens, const be_token* tokens, int n_pt_rows,
                                  int pt_stride, const int32_t* page_table, int n_lora,
                                  const be_lora* const* loras, const int32_t* lora_idx,
                                  const void* d_arena_in, void* d_arena_out, void* stream) {
  if (ctx == nullptr || blk == nullptr || n_tokens <= 0 || lora_idx == nullptr)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_exec_lora_batch: bad arguments") : BE_ERR_INVALID;
  int rc = check_loras(ctx, blk, n_lora, loras);
  if (rc != BE_OK) return rc;
  for (int t = 0; t < n_tokens; ++t)
    if (lora_idx[t] < -1 || lora_idx[t] >= n_lora)
      return fail(ctx, BE_ERR_INVALID, "token %d: adapter index %d out of range", t, lora_idx[t]);
  if (n_tokens > ws->max_tok)
    return fail(ctx, BE_ERR_INVALID, "batch of %d tokens > workspace %d", n_tokens, ws->max_tok);
  cudaSetDevice(ctx->device);
  cudaStream_t st = pick_stream(ctx, stream);
  BE_CUDA(ctx, cudaMemcpyAsync(ws->d_lora_idx, lora_idx, n_tokens * sizeof(int32_t),
                               cudaMemcpyHostToDevice, st));
  // the token / page-table validation and staging of be_exec_batch, then the adapter launch
  LoraSet set{n_lora, loras, ws->d_lora_idx};
  return exec_batch_host(ctx, blk, pool, ws, phase, n_tokens, tokens, n_pt_rows, pt_stride,
                         page_table, d_arena_in, d_arena_out, st, &set);
}

extern "C" int be_exec_speculative(be_ctx* ctx, const be_spec_stage* verify,
                                   const be_spec_stage* draft, const be_spec_stage* next,
                                   int n_tokens, const void* d_x_in, void* d_y_draft,
                                   void* d_y_true, void* d_z_out, float threshold, float* cos_out,
                                   int32_t* accept_out, int* n_accepted) {
  if (ctx == nullptr || verify == nullptr || draft == nullptr || next == nullptr ||
      n_tokens <= 0 || d_x_in == nullptr || d_y_draft == nullptr || d_y_true == nullptr ||
      d_z_out == nullptr || cos_out == nullptr || accept_out == nullptr || n_accepted == nullptr)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_exec_speculative: bad arguments") : BE_ERR_INVALID;
  const be_spec_stage* st3[3] = {verify, draft, next};
  for (const be_spec_stage* g : st3)
    if (g->blk == nullptr || g->pool == nullptr || g->ws == nullptr || g->tokens == nullptr)
      return fail(ctx, BE_ERR_INVALID, "be_exec_speculative: incomplete stage");
  if (verify->ws == draft->ws || verify->ws == next->ws)
    return fail(ctx, BE_ERR_INVALID, "be_exec_speculative: the verify lane needs its own workspace");
  const int d = verify->blk->desc.d_model;
  if (draft->blk->desc.d_model != d || next->blk->desc.d_model != d)
    return fail(ctx, BE_ERR_INVALID, "be_exec_speculative: blocks differ in d_model");
  cudaSetDevice(ctx->device);
  if (ctx->side == nullptr) {
    BE_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    BE_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    BE_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  }
  if (n_tokens > ctx->spec_cap) {
    if (ctx->spec_cos) cudaFree(ctx->spec_cos);
    if (ctx->spec_accept) cudaFree(ctx->spec_accept);
    ctx->spec_cos = nullptr;
    ctx->spec_accept = nullptr;
    BE_CUDA(ctx, cudaMalloc(&ctx->spec_cos, n_tokens * sizeof(float)));
    BE_CUDA(ctx, cudaMalloc(&ctx->spec_accept, n_tokens * sizeof(int)));
    ctx->spec_cap = n_tokens;
  }
  cudaStream_t lane = ctx->stream, side = ctx->side;
  auto run = [&](const be_spec_stage* g, const be_token* toks, int n, const void* in, void* out,
                 cudaStream_t s) {
    return be_exec_batch(ctx, g->blk, g->pool, g->ws, BE_PHASE_DECODE, n, toks, g->n_pt_rows,
                         g->pt_stride, g->page_table, in, out, s);
  };
  int rc;
  // Two lanes run stream-K GEMMs at once. A stream-K tile owner spin-waits for its contributor
  // CTAs, which is safe only while every CTA of the grid can become resident: each lane's GEMMs
  // get their own share of the SMs (one CTA per SM each, shares summing to the SM count) and no
  // programmatic dependent launch (at most one GEMM grid per lane in flight). Restored on exit.
  struct LaneCaps {
    be_ctx* c;
    int cap, pdl;
    explicit LaneCaps(be_ctx* x) : c(x), cap(x->gemm_grid_cap), pdl(x->use_pdl) { c->use_pdl = 0; }
    void set(int sms) { c->gemm_grid_cap = cap > 0 && cap < sms ? cap : sms; }
    ~LaneCaps() {
      c->gemm_grid_cap = cap;
      c->use_pdl = pdl;
    }
  } caps(ctx);
  const int side_sms = ctx->num_sms / 2, lane_sms = ctx->num_sms - side_sms;
  // K6: the draft lane (scenario.cpp:521-537) - surrogate, then the next block fed by its output
  BE_CUDA(ctx, cudaEventRecord(ctx->ev_fork, lane));
  BE_CUDA(ctx, cudaStreamWaitEvent(side, ctx->ev_fork, 0));
  caps.set(side_sms);
  if ((rc = run(draft, draft->tokens, n_tokens, d_x_in, d_y_draft, side)) != BE_OK) return rc;
  if ((rc = run(next, next->tokens, n_tokens, d_y_draft, d_z_out, side)) != BE_OK) return rc;
  // the verifying block on the main lane, concurrently
  caps.set(lane_sms);
  if ((rc = run(verify, verify->tokens, n_tokens, d_x_in, d_y_true, lane)) != BE_OK) return rc;
  caps.set(ctx->num_sms);
  BE_CUDA(ctx, cudaEventRecord(ctx->ev_join, side));
  BE_CUDA(ctx, cudaStreamWaitEvent(lane, ctx->ev_join, 0));
  // K7 verdict: per-row cosine(draft, true) >= threshold
  cudaError_t e = bx::launch_cosine(static_cast<const bf16*>(d_y_draft),
                                    static_cast<const bf16*>(d_y_true), n_tokens, d, threshold,
                                    ctx->spec_cos, ctx->spec_accept, lane);
  if (e != cudaSuccess) return fail(ctx, BE_ERR_CUDA, "cosine: %s", cudaGetErrorString(e));
  BE_CUDA(ctx, cudaMemcpyAsync(cos_out, ctx->spec_cos, n_tokens * sizeof(float),
                               cudaMemcpyDeviceToHost, lane));
  BE_CUDA(ctx, cudaMemcpyAsync(accept_out, ctx->spec_accept, n_tokens * sizeof(int),
                               cudaMemcpyDeviceToHost, lane));
  BE_CUDA(ctx, cudaStreamSynchronize(lane));
  // rejected rows: everything computed from their draft is redone from the true rows
  // (finish_verified, scenario.cpp:740-807); their KV slots in `next` are overwritten
  std::vector<be_token> redo;
  for (int i = 0; i < n_tokens; ++i)
    if (!accept_out[i]) redo.push_back(next->tokens[i]);
  *n_accepted = n_tokens - (int)redo.size();
  if (!redo.empty()) {
    if ((rc = run(next, redo.data(), (int)redo.size(), d_y_true, d_z_out, lane)) != BE_OK)
      return rc;
    BE_CUDA(ctx, cudaStreamSynchronize(lane));
  }
  return BE_OK;
}

extern "C" int be_exec_batch_launches(be_ctx* ctx, const be_block* blk, int n_tokens,
                                      int pt_stride) {
  if (ctx == nullptr || blk == nullptr || n_tokens <= 0) return 0;
  const int splits = attn_splits(ctx, n_tokens, blk->desc.n_heads, pt_stride);
  // gather; attention: qkv, attention (+combine), o; ffn: gate/up, down (the RMSNorms are fused:
  // statistics from the residual producer, scale in the consumer's epilogue; the scatter is fused
  // into the last GEMM's epilogue)
  return 1 + blk->n_att * (3 + (splits > 1 ? 1 : 0)) + blk->n_ffn * 2;
}

// ------------------------------------------------------------------------------ KV migration
extern "C" int be_kv_copy_pages(be_ctx* dst_ctx, const be_kv_pool* src_pool, be_kv_pool* dst_pool,
                                const int32_t* src_slots, const int32_t* dst_slots, int n,
                                void* stream) {
  if (dst_ctx == nullptr || src_pool == nullptr || dst_pool == nullptr || n < 0 ||
      (n > 0 && (src_slots == nullptr || dst_slots == nullptr)))
    return dst_ctx ? fail(dst_ctx, BE_ERR_INVALID, "be_kv_copy_pages: bad arguments") : BE_ERR_INVALID;
  if (src_pool->page_elems != dst_pool->page_elems)
    return fail(dst_ctx, BE_ERR_INVALID, "be_kv_copy_pages: pools differ in page layout");
  for (int i = 0; i < n; ++i)
    if (src_slots[i] < 0 || src_slots[i] >= src_pool->n_pages || dst_slots[i] < 0 ||
        dst_slots[i] >= dst_pool->n_pages)
      return fail(dst_ctx, BE_ERR_INVALID, "be_kv_copy_pages: slot %d out of range", i);
  const int src_dev = src_pool->ctx->device, dst_dev = dst_ctx->device;
  cudaSetDevice(dst_dev);
  if (src_dev != dst_dev) {
    int can = 0;
    BE_CUDA(dst_ctx, cudaDeviceCanAccessPeer(&can, dst_dev, src_dev));
    if (can) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(src_dev, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(dst_ctx, BE_ERR_CUDA, "peer access %d->%d: %s", dst_dev, src_dev, cudaGetErrorString(e));
      cudaGetLastError();
    }
  }
  cudaStream_t st = pick_stream(dst_ctx, stream);
  if (src_pool->ctx != dst_ctx || st != src_pool->ctx->stream) {
    // the copy reads pages the source context's stream may still be writing (KV appends of
    // kernels in flight): order it after everything queued there so far
    be_ctx* sc = src_pool->ctx;
    cudaSetDevice(src_dev);
    if (sc->ev_copy == nullptr)
      BE_CUDA(dst_ctx, cudaEventCreateWithFlags(&sc->ev_copy, cudaEventDisableTiming));
    BE_CUDA(dst_ctx, cudaEventRecord(sc->ev_copy, sc->stream));
    cudaSetDevice(dst_dev);
    BE_CUDA(dst_ctx, cudaStreamWaitEvent(st, sc->ev_copy, 0));
  }
  const size_t page_bytes = (size_t)src_pool->page_elems * sizeof(bf16);
  int i = 0;
  while (i < n) {
    int j = i + 1;  // coalesce runs contiguous on both sides
    while (j < n && src_slots[j] == src_slots[j - 1] + 1 && dst_slots[j] == dst_slots[j - 1] + 1) ++j;
    const char* s = reinterpret_cast<const char*>(src_pool->base) + (size_t)src_slots[i] * page_bytes;
    char* d = reinterpret_cast<char*>(dst_pool->base) + (size_t)dst_slots[i] * page_bytes;
    const size_t bytes = (size_t)(j - i) * page_bytes;
    if (src_dev == dst_dev) {
      BE_CUDA(dst_ctx, cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, st));
    } else {
      BE_CUDA(dst_ctx, cudaMemcpyPeerAsync(d, dst_dev, s, src_dev, bytes, st));
    }
    i = j;
  }
  return BE_OK;
}

extern "C" int be_kv_migrate(be_ctx* ctx, be_block* blk, const be_kv_pool* src_pool,
                             be_kv_pool* dst_pool, be_workspace* ws, const int32_t* src_slots,
                             const int32_t* dst_slots, int n_pages, int n_recompute,
                             int head_tokens, const void* d_head_rows, void* stream) {
  if (ctx == nullptr || blk == nullptr || src_pool == nullptr || dst_pool == nullptr ||
      ws == nullptr || n_pages < 0 || n_recompute < 0 || n_recompute > n_pages ||
      (n_pages > 0 && (src_slots == nullptr || dst_slots == nullptr)))
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_kv_migrate: bad arguments") : BE_ERR_INVALID;
  // with tail pages copied, the head must fill its last recomputed page (no token uncovered)
  const int head_min = n_recompute < n_pages ? n_recompute * 16 : (n_recompute - 1) * 16 + 1;
  if (n_recompute > 0 && (d_head_rows == nullptr || head_tokens < head_min ||
                          head_tokens > n_recompute * 16))
    return fail(ctx, BE_ERR_INVALID,
                "be_kv_migrate: %d recompute pages need %d..%d head tokens (got %d)",
                n_recompute, head_min, n_recompute * 16, head_tokens);
  if (dst_pool->ctx != ctx || blk->ctx != ctx)
    return fail(ctx, BE_ERR_INVALID, "be_kv_migrate: block and destination pool must be on ctx");
  cudaSetDevice(ctx->device);
  if (ctx->side == nullptr) {
    BE_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    BE_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    BE_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  }
  cudaStream_t st = pick_stream(ctx, stream);
  const int n_copy = n_pages - n_recompute;
  int rc;
  // tail pages: copy engine (peer copy over NVLink when the pools are on different GPUs), on the
  // side stream so it overlaps the recompute
  if (n_copy > 0) {
    BE_CUDA(ctx, cudaEventRecord(ctx->ev_fork, st));
    BE_CUDA(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    if ((rc = be_kv_copy_pages(ctx, src_pool, dst_pool, src_slots + n_recompute,
                               dst_slots + n_recompute, n_copy, ctx->side)) != BE_OK)
      return rc;
  }
  // head pages: chunked prefill of the head tokens through the block on the destination, K/V
  // appended straight into the destination pages (outputs discarded: dst_row -1)
  if (n_recompute > 0) {
    std::vector<be_token> toks(head_tokens);
    for (int t = 0; t < head_tokens; ++t)
      toks[t] = be_token{t, -1, dst_slots[t >> 4] * 16 + (t & 15), t, 0};
    if ((rc = be_exec_batch(ctx, blk, dst_pool, ws, BE_PHASE_PREFILL, head_tokens, toks.data(),
                            1, n_recompute, dst_slots, d_head_rows, nullptr, st)) != BE_OK)
      return rc;
  }
  if (n_copy > 0) {
    BE_CUDA(ctx, cudaEventRecord(ctx->ev_join, ctx->side));
    BE_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_join, 0));
  }
  return BE_OK;
}

// ------------------------------------------------------------------------------ row kernels
extern "C" int be_gather_rows(be_ctx* ctx, const void* arena, const int32_t* src, int rows, int d,
                              void* out, void* stream) {
  if (ctx == nullptr || rows < 0 || d % 8 != 0) return BE_ERR_INVALID;
  cudaError_t e = bx::launch_gather(static_cast<const bf16*>(arena), src, 1, rows, d,
                                    static_cast<bf16*>(out), nullptr, nullptr,
                                    pick_stream(ctx, stream), nullptr, 0);
  return e == cudaSuccess ? BE_OK : fail(ctx, BE_ERR_CUDA, "gather: %s", cudaGetErrorString(e));
}

extern "C" int be_scatter_rows(be_ctx* ctx, const void* rows_in, const int32_t* dst, int rows,
                               int d, void* arena, void* stream) {
  if (ctx == nullptr || rows < 0 || d % 8 != 0) return BE_ERR_INVALID;
  cudaError_t e = bx::launch_scatter(static_cast<const bf16*>(rows_in), dst, 1, rows, d,
                                     static_cast<bf16*>(arena), pick_stream(ctx, stream), nullptr, 0);
  return e == cudaSuccess ? BE_OK : fail(ctx, BE_ERR_CUDA, "scatter: %s", cudaGetErrorString(e));
}

extern "C" int be_cosine(be_ctx* ctx, const void* pred, const void* actual, int rows, int d,
                         float thr, float* cos_out, int32_t* accept, void* stream) {
  if (ctx == nullptr || rows < 0 || d % 8 != 0 || cos_out == nullptr) return BE_ERR_INVALID;
  cudaError_t e = bx::launch_cosine(static_cast<const bf16*>(pred), static_cast<const bf16*>(actual),
                                    rows, d, thr, cos_out, accept, pick_stream(ctx, stream));
  return e == cudaSuccess ? BE_OK : fail(ctx, BE_ERR_CUDA, "cosine: %s", cudaGetErrorString(e));
}

extern "C" int be_synth_rows(be_ctx* ctx, void* dst, int64_t n, uint64_t seed, const char* sid,
                             float scale, void* stream) {
  if (ctx == nullptr || dst == nullptr || sid == nullptr || n < 0) return BE_ERR_INVALID;
  cudaError_t e = bx::launch_synth_rows(static_cast<bf16*>(dst), n, stream_key(seed, sid), scale,
                                        pick_stream(ctx, stream));
  return e == cudaSuccess ? BE_OK : fail(ctx, BE_ERR_CUDA, "synth: %s", cudaGetErrorString(e));
}

extern "C" int be_pack_weight(be_ctx* ctx, const void* src, void* dst, int N, int K,
                              void* stream) {
  if (ctx == nullptr || src == nullptr || dst == nullptr || N % 128 != 0 || K % 64 != 0)
    return BE_ERR_INVALID;
  cudaError_t e = bx::launch_pack_weight(static_cast<const bf16*>(src), static_cast<bf16*>(dst), N,
                                         K, pick_stream(ctx, stream));
  return e == cudaSuccess ? BE_OK : fail(ctx, BE_ERR_CUDA, "pack: %s", cudaGetErrorString(e));
}

// ------------------------------------------------------------------------------ stitches
// A stitch maps activations of width dim_in to dim_out when a chain step is served by an
// equivalent block of another width (Zoo::candidate_instances, zoo.cpp:568-589; priced by
// CostModel::stitch_us): one linear layer, y = x W^T, W [dim_out][dim_in] synthetic from stream
// "stitch:<name>" (same counter-mode generator as block weights), run on the tcgen05 GEMM.
struct be_stitch {
  be_ctx* ctx = nullptr;
  int dim_in = 0, dim_out = 0;
  bf16* w = nullptr;  // packed tile layout
};

extern "C" int be_stitch_load(be_ctx* ctx, int dim_in, int dim_out, const char* name,
                              uint64_t seed, float scale, be_stitch** out) {
  if (ctx == nullptr || name == nullptr || out == nullptr || dim_in <= 0 || dim_in % 64 != 0 ||
      dim_out <= 0 || dim_out % 128 != 0)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_stitch_load: dims must be multiples of 64 (in) "
                                           "and 128 (out)")
               : BE_ERR_INVALID;
  cudaSetDevice(ctx->device);
  auto* s = new be_stitch();
  s->ctx = ctx;
  s->dim_in = dim_in;
  s->dim_out = dim_out;
  if (cudaMalloc(&s->w, (size_t)dim_in * dim_out * sizeof(bf16)) != cudaSuccess) {
    delete s;
    return fail(ctx, BE_ERR_NOMEM, "be_stitch_load: allocation failed");
  }
  bx::launch_synth_weight(s->w, dim_out, dim_in, stream_key(seed, std::string("stitch:") + name),
                          0, scale, 0, 64, nullptr, ctx->stream);
  const cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    cudaFree(s->w);
    delete s;
    return fail(ctx, BE_ERR_CUDA, "be_stitch_load: %s", cudaGetErrorString(e));
  }
  *out = s;
  return BE_OK;
}

extern "C" int be_stitch_free(be_stitch* s) {
  if (s == nullptr) return BE_ERR_INVALID;
  cudaSetDevice(s->ctx->device);
  if (s->w) cudaFree(s->w);
  delete s;
  return BE_OK;
}

extern "C" int be_gemm_bf16(be_ctx* ctx, const void* w, const void* x, void* out, int N, int K,
                            int ntok, int grid_cap, void* stream);

extern "C" int be_stitch_rows(be_ctx* ctx, const be_stitch* s, const void* d_in, int rows,
                              void* d_out, void* stream) {
  if (ctx == nullptr || s == nullptr || d_in == nullptr || d_out == nullptr || rows <= 0)
    return ctx ? fail(ctx, BE_ERR_INVALID, "be_stitch_rows: bad arguments") : BE_ERR_INVALID;
  cudaSetDevice(ctx->device);
  return be_gemm_bf16(ctx, s->w, d_in, d_out, s->dim_out, s->dim_in, rows, 0, stream);
}

extern "C" int be_gemm_bf16(be_ctx* ctx, const void* w, const void* x, void* out, int N, int K,
                            int ntok, int grid_cap, void* stream) {
  if (ctx == nullptr || N % 128 != 0 || K % 64 != 0 || ntok <= 0 || grid_cap < 0)
    return BE_ERR_INVALID;
  const int bn = bx::gemm_pick_bn(ntok);
  CUtensorMap mx;
  int rc;
  if ((rc = make_map(ctx, &mx, x, ntok, K, bn)) != BE_OK) return rc;
  const bx::GemmPlan p =
      bx::gemm_plan(N, K, ntok, bn, ctx->num_sms, (size_t)1 << 40, 1 << 16, grid_cap);
  if (p.ws_needed > ctx->gemm_ws_elems) {
    if (ctx->gemm_ws) cudaFree(ctx->gemm_ws);
    ctx->gemm_ws = nullptr;
    BE_CUDA(ctx, cudaMalloc(&ctx->gemm_ws, p.ws_needed * sizeof(float)));
    ctx->gemm_ws_elems = p.ws_needed;
  }
  const int tiles = (N / 128) * ((ntok + bn - 1) / bn);
  if (tiles > (1 << 16)) return fail(ctx, BE_ERR_INVALID, "gemm: too many tiles");
  if (ctx->gemm_counters == nullptr) {
    BE_CUDA(ctx, cudaMalloc(&ctx->gemm_counters, (1 << 16) * sizeof(int)));
    BE_CUDA(ctx, cudaMemset(ctx->gemm_counters, 0, (1 << 16) * sizeof(int)));
  }
  bx::GemmLaunch L{};
  L.w_packed = static_cast<const bf16*>(w);
  L.map_x = &mx;
  L.N = N;
  L.K = K;
  L.bn = bn;
  L.grid = p.grid;
  L.rr = p.rr;
  L.pdl = ctx->use_pdl;
  L.epi.mode = bx::kStore;
  L.epi.ntok = ntok;
  L.epi.out = static_cast<bf16*>(out);
  L.epi.ldo = N;
  L.epi.ws = ctx->gemm_ws;
  L.epi.counters = ctx->gemm_counters;
  unsigned long long* trace = nullptr;
  const bool tracing = getenv("BE_GEMM_TRACE") != nullptr;
  if (tracing) {
    BE_CUDA(ctx, cudaMalloc(&trace, (size_t)p.grid * 8 * sizeof(unsigned long long)));
    BE_CUDA(ctx, cudaMemset(trace, 0, (size_t)p.grid * 8 * sizeof(unsigned long long)));
    L.epi.trace = trace;
  }
  cudaError_t e = bx::launch_gemm(L, pick_stream(ctx, stream));
  if (tracing) {
    // diagnostics: per-phase globaltimer stamps across CTAs, microseconds from the first entry
    std::vector<unsigned long long> h((size_t)p.grid * 8);
    cudaStreamSynchronize(pick_stream(ctx, stream));
    cudaMemcpy(h.data(), trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(trace);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < p.grid; ++c) t0 = h[c * 8] && h[c * 8] < t0 ? h[c * 8] : t0;
    const char* names[8] = {"entry", "setup", "pdl_wait", "last_load", "last_tfull", "epi_done",
                            "role", "exit"};
    fprintf(stderr, "gemm trace N=%d K=%d ntok=%d grid=%d\n", N, K, ntok, p.grid);
    // the five slowest final epilogues: role 1000000+n = owner of an n-way partial tile,
    // 2000000 = non-owner contributor, 0 = full tile
    std::vector<int> order(p.grid);
    for (int c = 0; c < p.grid; ++c) order[c] = c;
    std::sort(order.begin(), order.end(), [&](int a, int b2) { return h[a * 8 + 5] > h[b2 * 8 + 5]; });
    for (int i = 0; i < 5 && i < p.grid; ++i) {
      const int c = order[i];
      fprintf(stderr, "  slow cta %3d: last_tfull %.2f epi_done %.2f role %llu\n", c,
              (h[c * 8 + 4] - t0) / 1e3, (h[c * 8 + 5] - t0) / 1e3,
              (unsigned long long)h[c * 8 + 6]);
    }
    for (int c = 0; c < p.grid; ++c) h[c * 8 + 6] = 0;
    for (int k = 0; k < 8; ++k) {
      std::vector<double> v;
      for (int c = 0; c < p.grid; ++c)
        if (h[c * 8 + k]) v.push_back((h[c * 8 + k] - t0) / 1e3);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      fprintf(stderr, "  %-12s min %8.2f  med %8.2f  max %8.2f us (n=%zu)\n", names[k], v.front(),
              v[v.size() / 2], v.back(), v.size());
    }
    int inverted = 0;
    for (int c = 0; c < p.grid; ++c)
      if (h[c * 8 + 7] && h[c * 8 + 5] && h[c * 8 + 7] < h[c * 8 + 5]) ++inverted;
    fprintf(stderr, "  CTAs with exit stamp < epilogue-done stamp: %d; cta0 epi_done %.2f exit %.2f\n",
            inverted, (h[5] - t0) / 1e3, (h[7] - t0) / 1e3);
    int worst = 0;
    for (int c = 0; c < p.grid; ++c)
      if (h[c * 8 + 5] > h[worst * 8 + 5]) worst = c;
    fprintf(stderr, "  slowest epilogue cta %d:", worst);
    for (int k = 0; k < 8; ++k)
      fprintf(stderr, " %s=%.2f", names[k], h[worst * 8 + k] ? (h[worst * 8 + k] - t0) / 1e3 : -1.0);
    fprintf(stderr, "\n");
  }
  return e == cudaSuccess ? BE_OK : fail(ctx, BE_ERR_CUDA, "gemm: %s", cudaGetErrorString(e));
}

// Device time per launch of the GEMM, measured as one CUDA-graph replay of `reps` launches that
// cycle through `n_w` packed weight copies (so the weights come from HBM, not L2).
extern "C" int be_bench_gemm(be_ctx* ctx, const void* const* w_packed, int n_w, const void* x,
                             void* out, int N, int K, int ntok, int reps, float* us_per_launch) {
  if (ctx == nullptr || w_packed == nullptr || n_w <= 0 || reps <= 0 || us_per_launch == nullptr)
    return BE_ERR_INVALID;
  cudaStream_t st = ctx->stream;
  int rc = be_gemm_bf16(ctx, w_packed[0], x, out, N, K, ntok, 0, st);  // configure + allocate
  if (rc != BE_OK) return rc;
  BE_CUDA(ctx, cudaStreamSynchronize(st));
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  BE_CUDA(ctx, cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int r = 0; r < reps && rc == BE_OK; ++r)
    rc = be_gemm_bf16(ctx, w_packed[r % n_w], x, out, N, K, ntok, 0, st);
  cudaStreamEndCapture(st, &g);
  if (rc != BE_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  BE_CUDA(ctx, cudaGraphInstantiate(&ge, g, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaGraphLaunch(ge, st);  // warm
  cudaEventRecord(e0, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  BE_CUDA(ctx, cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *us_per_launch = ms * 1e3f / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return BE_OK;
}

extern "C" int be_attention(be_ctx* ctx, const void* q, const void* pool, int n_layers, int H,
                            int hd, int layer, const int32_t* pt, int pt_stride,
                            const int32_t* row_pt, const int32_t* row_ctx, int rows, int splits,
                            void* out, void* stream) {
  if (ctx == nullptr || rows < 0 || (hd != 64 && hd != 128) || splits < 1) return BE_ERR_INVALID;
  cudaSetDevice(ctx->device);
  if (splits > 1) {  // split-K partials: the context's own scratch (one per GPU / context)
    const size_t need = (size_t)rows * H * splits * (hd + 2);
    if (need > ctx->attn_part_elems) {
      BE_CUDA(ctx, cudaStreamSynchronize(pick_stream(ctx, stream)));
      if (ctx->attn_part) cudaFree(ctx->attn_part);
      ctx->attn_part = nullptr;
      ctx->attn_part_elems = 0;
      BE_CUDA(ctx, cudaMalloc(&ctx->attn_part, need * sizeof(float)));
      ctx->attn_part_elems = need;
    }
  }
  bx::AttnParams ap{};
  ap.q = static_cast<const bf16*>(q);
  ap.pool = static_cast<const bf16*>(pool);
  ap.layer_elems = 2LL * H * 16 * hd;
  ap.page_elems = ap.layer_elems * n_layers;
  ap.layer = layer;
  ap.page_table = pt;
  ap.pt_stride = pt_stride;
  ap.row_pt = row_pt;
  ap.row_ctx = row_ctx;
  ap.meta_stride = 1;
  ap.ctx_add = 0;
  ap.H = H;
  ap.scale_log2 = (1.0f / sqrtf((float)hd)) * 1.4426950408889634f;
  ap.out = static_cast<bf16*>(out);
  ap.part = ctx->attn_part;
  ap.splits = splits;
  cudaError_t e = bx::launch_attention(ap, rows, hd, pick_stream(ctx, stream));
  return e == cudaSuccess ? BE_OK : fail(ctx, BE_ERR_CUDA, "attention: %s", cudaGetErrorString(e));
}
