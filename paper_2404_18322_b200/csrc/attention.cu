// Paged attention over a block-local KV pool (K3 attention core).
//
// Pool layout (one page = 16 tokens of one (request, block) segment, all layers of the block):
//   pool[page][layer][K|V][head][16][head_dim]  bf16
// so one head's 16 keys of a page are one contiguous 16*hd*2-byte run (4 KB at hd=128) and a
// warp streams it with 16-byte vector loads. Each query row (a decode token, or one prompt
// token of a prefill) reads the pages named by its row of the page table, up to ctx_len tokens
// (causal by construction: a prefill token's ctx_len is its position + 1).
//
// Grid (rows, heads, splits); 4 warps per CTA split the row's pages round-robin; each warp keeps
// an online-softmax state (running max m, sum l, o[hd] spread over lanes) in fp32; warps merge
// through shared memory; with splits > 1 the CTA writes an unnormalised partial and
// attn_combine merges the splits (flash-decoding).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cfloat>

#include "ptx.cuh"

namespace bx {

struct AttnParams {
  const __nv_bfloat16* q;     // [rows][H*hd] (q/k head dims pair-interleaved, see gemm QKV)
  const __nv_bfloat16* pool;  // KV pool
  long long page_elems;       // elements per page
  long long layer_elems;      // elements per layer inside a page
  int layer;
  const int* page_table;      // [n_pt][pt_stride]
  int pt_stride;
  const int* row_pt;          // row r -> page-table row at row_pt[r * meta_stride]
  const int* row_ctx;         // row r -> visible tokens at row_ctx[r * meta_stride] (+ ctx_add)
  int meta_stride;            // 1 for plain arrays, 5 for be_token records
  int ctx_add;                // 0 for ctx arrays, 1 when row_ctx points at positions
  int H;
  float scale_log2;           // softmax scale * log2(e)
  __nv_bfloat16* out;         // [rows][H*hd]
  float* part;                // [rows][H][splits][hd + 2] partials when splits > 1
  int splits;
  // grouped batch: rows [g*grp_rows, (g+1)*grp_rows) read block g's pool pools[g]
  int n_grp;
  int grp_rows;
  const __nv_bfloat16* pools[8];
  unsigned long long* tl;     // diagnostics: timeline slots of decode and combine (or nullptr)
  int tl_cap;
};

template <int HD>
__global__ void __launch_bounds__(128) attn_decode_kernel(AttnParams P) {
  constexpr int LPT = HD / 8;      // lanes per token (16 B = 8 bf16 per lane)
  constexpr int TPL = 32 / LPT;    // tokens per warp-load
  constexpr int NLD = 16 / TPL;    // warp-loads per 16-token page
  const int row = blockIdx.x;
  const int head = blockIdx.y;
  const int split = blockIdx.z;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int sub = lane % LPT;      // which 8-dim chunk
  const int tg = lane / LPT;       // token group inside a warp-load
  if (threadIdx.x == 0) {
    tl_start(P.tl, P.tl_cap);
    tl_go(P.tl, P.tl_cap);
  }

  const int ctx = P.row_ctx[(size_t)row * P.meta_stride] + P.ctx_add;
  const int npages = (ctx + 15) >> 4;
  const int p_begin = (int)((long long)split * npages / P.splits);
  const int p_end = (int)((long long)(split + 1) * npages / P.splits);
  const int* pt = P.page_table + (size_t)P.row_pt[(size_t)row * P.meta_stride] * P.pt_stride;
  const __nv_bfloat16* pool = P.n_grp > 1 ? P.pools[row / P.grp_rows] : P.pool;

  // q chunk for this lane, prescaled so scores are in log2 units
  float q[8];
  {
    const uint4 qv = *reinterpret_cast<const uint4*>(P.q + (size_t)row * P.H * HD + head * HD + sub * 8);
    const __nv_bfloat16* qb = reinterpret_cast<const __nv_bfloat16*>(&qv);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = __bfloat162float(qb[i]) * P.scale_log2;
  }

  float m = -FLT_MAX, l = 0.f;
  float o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = 0.f;

  const size_t head_off = (size_t)P.layer * P.layer_elems + (size_t)head * 16 * HD;
  const size_t v_off = (size_t)P.H * 16 * HD;

  for (int p = p_begin + warp; p < p_end; p += 4) {
    const __nv_bfloat16* kp = pool + (size_t)pt[p] * P.page_elems + head_off;
    const __nv_bfloat16* vp = kp + v_off;
    uint4 kr[NLD], vr[NLD];
#pragma unroll
    for (int j = 0; j < NLD; ++j) {
      kr[j] = __ldcs(reinterpret_cast<const uint4*>(kp) + j * 32 + lane);
    }
#pragma unroll
    for (int j = 0; j < NLD; ++j) {
      vr[j] = __ldcs(reinterpret_cast<const uint4*>(vp) + j * 32 + lane);
    }
    float s[NLD];
    float pmax = -FLT_MAX;
#pragma unroll
    for (int j = 0; j < NLD; ++j) {
      const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(&kr[j]);
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = fmaf(q[i], __bfloat162float(kb[i]), acc);
#pragma unroll
      for (int off = LPT / 2; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      const int tok = p * 16 + j * TPL + tg;
      s[j] = tok < ctx ? acc : -FLT_MAX;
      pmax = fmaxf(pmax, s[j]);
    }
#pragma unroll
    for (int off = LPT; off < 32; off <<= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, off));
    const float m_new = fmaxf(m, pmax);
    const float corr = exp2f(m - m_new);
    float psum = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] *= corr;
#pragma unroll
    for (int j = 0; j < NLD; ++j) {
      const float pj = s[j] == -FLT_MAX ? 0.f : exp2f(s[j] - m_new);
      psum += pj;
      const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&vr[j]);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = fmaf(pj, __bfloat162float(vb[i]), o[i]);
    }
#pragma unroll
    for (int off = LPT; off < 32; off <<= 1) psum += __shfl_xor_sync(0xffffffffu, psum, off);
    l = l * corr + psum;
    m = m_new;
  }
  // the next (PDL-launched) GEMM may start streaming its weights under this kernel's tail
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // merge token groups inside the warp (lanes with equal `sub`)
#pragma unroll
  for (int off = LPT; off < 32; off <<= 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] += __shfl_xor_sync(0xffffffffu, o[i], off);
  }

  __shared__ float s_m[4], s_l[4];
  __shared__ float s_o[4][HD];
  if (lane == 0) {
    s_m[warp] = m;
    s_l[warp] = l;
  }
  if (lane < LPT) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s_o[warp][sub * 8 + i] = o[i];
  }
  __syncthreads();
  if (threadIdx.x < HD) {
    const int dim = threadIdx.x;
    float M = fmaxf(fmaxf(s_m[0], s_m[1]), fmaxf(s_m[2], s_m[3]));
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float c = s_m[w] == -FLT_MAX ? 0.f : exp2f(s_m[w] - M);
      L += s_l[w] * c;
      O += s_o[w][dim] * c;
    }
    if (P.splits == 1) {
      P.out[(size_t)row * P.H * HD + head * HD + dim] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
    } else {
      float* pp = P.part + (((size_t)row * P.H + head) * P.splits + split) * (HD + 2);
      pp[2 + dim] = O;
      if (dim == 0) {
        pp[0] = M;
        pp[1] = L;
      }
    }
  }
  if (threadIdx.x == 0) tl_end(P.tl, P.tl_cap);
}

template <int HD>
__global__ void attn_combine_kernel(AttnParams P) {
  const int row = blockIdx.x;
  const int head = blockIdx.y;
  const int dim = threadIdx.x;
  unsigned long long* tl = P.tl != nullptr ? P.tl + 1 : nullptr;  // the combine's own slot
  if (dim == 0) {
    tl_start(tl, P.tl_cap);
    tl_go(tl, P.tl_cap);
  }
  const float* pp = P.part + (((size_t)row * P.H + head) * P.splits) * (HD + 2);
  float M = -FLT_MAX;
  for (int s = 0; s < P.splits; ++s) M = fmaxf(M, pp[s * (HD + 2)]);
  float L = 0.f, O = 0.f;
  for (int s = 0; s < P.splits; ++s) {
    const float ms = pp[s * (HD + 2)];
    const float c = ms == -FLT_MAX ? 0.f : exp2f(ms - M);
    L += pp[s * (HD + 2) + 1] * c;
    O += pp[s * (HD + 2) + 2 + dim] * c;
  }
  P.out[(size_t)row * P.H * HD + head * HD + dim] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
  if (dim == 0) tl_end(tl, P.tl_cap);
}

cudaError_t launch_attention(const AttnParams& P, int rows, int head_dim, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  dim3 grid(rows, P.H, P.splits);
  if (head_dim == 128) {
    attn_decode_kernel<128><<<grid, 128, 0, stream>>>(P);
    if (P.splits > 1) attn_combine_kernel<128><<<dim3(rows, P.H), 128, 0, stream>>>(P);
  } else if (head_dim == 64) {
    attn_decode_kernel<64><<<grid, 128, 0, stream>>>(P);
    if (P.splits > 1) attn_combine_kernel<64><<<dim3(rows, P.H), 64, 0, stream>>>(P);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace bx
