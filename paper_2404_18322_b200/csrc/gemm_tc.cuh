// Block-forward GEMM on tcgen05: out^T[f, t] = sum_k W[f, k] * X[t, k] ("swap-AB": weight rows
// fill the 128-row UMMA M dimension, the batch's tokens are the UMMA N dimension, 16..256).
// Operands arrive by TMA (128B swizzle, K-major) through an mbarrier ring; one elected thread
// issues tcgen05.mma into a TMEM accumulator; four warps drain TMEM in a fused epilogue:
//   kStore   out = bf16(acc)                                   (plain projection)
//   kResid   x += acc, xb = bf16(x)                            (O / down proj + residual)
//   kSwiGLU  h = silu(gate) * up  (gate/up rows interleaved)   (FFN gate/up)
//   kQKV     RoPE(q,k) + q store + paged KV append of k, v     (attention input proj)
// The RMSNorm of the input row is fused as a per-token scale (rstd) applied to acc; the norm
// weight gamma is folded into W at load time; the per-token statistics come from the producer of
// the residual stream (see ss_in / ss_out), so no separate norm kernel runs. Split-K partials meet in an fp32 workspace
// (L2 resident) and the last CTA of a tile runs the epilogue.
#pragma once
#include <cuda.h>
#include "ptx.cuh"

namespace bx {

// kResidOut: the block's last GEMM - residual add, then K2 (the scatter) fused: the bf16 row of
// token t goes straight to out[tok[t].dst_row] (dst_row < 0: not stored); no fp32 / stats copy
// k*Lora: the same epilogues plus a per-token low-rank adapter delta added to the (normalised)
// accumulator before anything else: v[t][f] += <B_{a(t)}[f], u[t][seg(f)]> (segmented LoRA: the
// tokens of one launch may belong to different adapters; u from lora_shrink_kernel)
enum EpiMode : int {
  kStore = 0, kResid = 1, kSwiGLU = 2, kQKV = 3, kResidOut = 4,
  kQKVLora = 5, kResidLora = 6, kResidOutLora = 7
};
constexpr int kMaxGroup = 8;  // blocks per grouped batch
constexpr int kLoraRank = 16;  // LoRA rank r of every adapter
constexpr int kMaxLora = 8;    // adapters per launch
struct LoraTable {
  const __nv_bfloat16* p[kMaxLora];
};

struct EpiParams {
  int mode;
  int ntok;                // valid tokens (columns)
  // fused RMSNorm without a stats kernel: the producer of the residual stream (gather, or a
  // kResid epilogue) writes per-(token, 32-feature group) sums of squares ss[t][g]; a GEMM with
  // ss_in reduces them to rstd[t] = 1/sqrt(sum/d + eps) before its first accumulator is ready
  const float* ss_in;      // [ntok][ss_groups] or nullptr (no norm)
  const float* rs_in;      // [ntok] rstd already reduced (round-robin launches), or nullptr
  float* ss_out;           // kResid: [ntok][ss_groups] written for the next component, or nullptr
  int ss_groups;           // d_model / 32
  float norm_eps;
  __nv_bfloat16* out;      // kStore/kSwiGLU/kQKV(q): [ntok][ldo]
  int ldo;
  float* xres;             // kResid: fp32 residual stream [ntok][ldr]
  __nv_bfloat16* xres_b;   // kResid: bf16 shadow of the residual (next GEMM's B operand)
  int ldr;
  // kQKV
  const int* tok;          // [ntok] be_token records {src, dst, kv_slot, pos, pt_row}:
                           //   kv_slot = page_slot * 16 + pos % 16, pos = RoPE position
  __nv_bfloat16* kv_pool;  // paged KV pool of the block instance
  long long page_elems;    // elements per page: L * 2 * H * 16 * hd
  long long layer_elems;   // elements per layer inside a page: 2 * H * 16 * hd
  int layer;
  int d_model;
  int head_dim;
  const float2* rope;      // [max_pos][head_dim/2] (cos, sin)
  // stream-K partial tiles
  float* ws;               // [grid][2][BN][128] fp32 partials (first/last segment per CTA)
  int* counters;           // [tiles] arrival counters (self-resetting)
  unsigned long long* trace;  // diagnostics: [grid][8] globaltimer stamps, nullptr = off
  // grouped batch: n_grp independent blocks of one shape side by side, token rows
  // [g*grp_rows, (g+1)*grp_rows) belonging to block g (grp_rows == BN): the GEMM of n-tile g
  // streams wgrp[g] and the QKV epilogue appends to kvgrp[g] (n_grp <= 1: wpk / kv_pool)
  int n_grp;
  int grp_rows;
  const __nv_bfloat16* wgrp[kMaxGroup];
  __nv_bfloat16* kvgrp[kMaxGroup];
  unsigned long long* tl;     // diagnostics: kernel timeline slot (ptx.cuh tl_*), nullptr = off
  int tl_cap;
  // k*Lora modes: u [ntok][ustride] fp32, adapter per token (-1: none), B_a [N][kLoraRank] bf16
  // rows in the GEMM's physical row order; segment f / lora_seg picks u's r-slice (q / k / v)
  const float* lora_u;
  int lora_ustride;
  int lora_seg;
  const int* lora_idx;
  LoraTable lora_b;
};

#ifndef BE_GEMM_WIDE_EPI16
#define BE_GEMM_WIDE_EPI16 1  // stream-K launches of 128/256-token tiles: four warps per quarter
#endif
// epilogue warps per CTA: two per TMEM lane quarter (4 -> 8 warps: decode step +4-5%); four per
// quarter for stream-K launches of 128/256-token tiles (C5's 256-row decode: the owners' 128
// columns per thread were the launch tail; +1.4% C5), not for the 16-64-token decode tiles (-1%
// .. +2% across boxes, spills in the LoRA modes) nor for the round-robin prefill (slower).
template <int BN, bool RR = false>
__host__ __device__ constexpr int epi_warps() {
  return BE_GEMM_WIDE_EPI16 && BN >= 128 && !RR ? 16 : 8;
}
constexpr int kBM = 128;
constexpr int kBK = 64;

template <int BN>
struct GemmSmem {
  static constexpr int kABytes = kBM * kBK * 2;  // 16 KB
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
};

// Ring depth: up to 8 stages / ~200 KB, one CTA per SM. Measured slower: deeper rings
// (12 x 18-24 KB), ~100 KB rings with two CTAs per SM, and ~100 KB rings leaving room for the
// next PDL-launched GEMM beside this one.
#ifndef BE_GEMM_CTAS
#define BE_GEMM_CTAS 1  // experiments: 2 (with a <= 100 KB ring) lets the next PDL launch co-reside
#endif
#ifndef BE_GEMM_RING_KB
#define BE_GEMM_RING_KB 96  // ring of a CTA that shares its SM (BE_GEMM_CTAS = 2)
#endif
// resident CTAs per SM for a tile width: the co-residency experiment covers the decode widths
template <int BN>
__host__ __device__ constexpr int gemm_ctas() {
  return BN <= 64 ? BE_GEMM_CTAS : 1;
}
#ifndef BE_GEMM_MAX_STAGES
#define BE_GEMM_MAX_STAGES 8
#endif
#ifndef BE_GEMM_RING_MAX_KB
#define BE_GEMM_RING_MAX_KB 200
#endif
template <int BN>
__host__ __device__ constexpr int gemm_stages_deep() {
  const int ring_kb = gemm_ctas<BN>() > 1 ? BE_GEMM_RING_KB : BE_GEMM_RING_MAX_KB;
  const int s = (ring_kb * 1024) / GemmSmem<BN>::kStageBytes;
  return s > BE_GEMM_MAX_STAGES ? BE_GEMM_MAX_STAGES : (s < 2 ? 2 : s);
}

template <int BN>
__host__ __device__ constexpr uint32_t tmem_cols() {
  return BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : (BN <= 256 ? 256 : 512)));
}

// Host-side launch description.
struct GemmLaunch {
  const __nv_bfloat16* w_packed;  // weights [N][K] in the packed tile layout (ptx.cuh)
  const CUtensorMap* map_x;  // activations [rows][K] bf16, box {64, BN}
  int N, K;
  int bn;                    // 16/32/64/128/256
  int grid;                  // persistent CTAs (stream-K ranges)
  int pdl;                   // launch with programmatic stream serialization
  int rr;                    // whole tiles dealt round-robin (large M), see gemm_plan
  EpiParams epi;
};

struct GemmPlan {
  int grid;
  size_t ws_needed;  // fp32 elements of split-tile partials
  long long tiles;   // arrival counters needed
  int rr;            // 1: whole tiles round-robin over the CTAs (no split, no partials)
};

// Launches on `stream`; returns cudaError_t.
cudaError_t launch_gemm(const GemmLaunch& L, cudaStream_t stream);
// rstd[t] = 1/sqrt(sum_g ss[t][g] / (32 G) + eps) for ntok tokens, in tile_rstd's exact order
// (prefill: the round-robin GEMM tiles of one token tile would otherwise each reduce it again)
cudaError_t launch_rstd(const float* ss, int groups, int ntok, float eps, float* rstd,
                        cudaStream_t stream);

// BN for a token count; persistent grid and workspace need for the stream-K schedule.
int gemm_pick_bn(int ntok);
GemmPlan gemm_plan(int N, int K, int ntok, int bn, int num_sms, size_t ws_elems, int n_counters,
                   int grid_cap);

}  // namespace bx
