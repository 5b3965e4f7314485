// tcgen05 / TMEM / TMA block-forward GEMM (see gemm_tc.cuh for the contract).
//
// Persistent stream-K schedule: the (tile, k-block) iteration space of the whole GEMM is cut
// into gridDim.x equal contiguous ranges, one per CTA (grid <= #SMs, one CTA per SM), so every
// SM streams the same number of weight bytes whatever the tile count (no wave quantisation:
// 172 gate/up tiles or 32 O-proj tiles both spread over all 148 SMs). A CTA range may start or
// end inside a tile; such partial tiles meet in an fp32 workspace (L2-resident) and the last
// contributor to arrive runs the fused epilogue (no CTA ever waits on another).
//
// Warp roles (64 + 32 * epi_warps<BN>() threads): warp 0 = TMA producer (one elected lane), warp
// 1 = MMA issuer (one elected lane) + TMEM allocator, warps 2.. = epilogue: warp w drains TMEM
// lanes 32*(w%4).. (the lane quarter a warp may access), the warps sharing a quarter splitting
// the tile's token columns, so several epilogue warps per SM sub-partition hide each other's
// latencies (the owners' fixup + epilogue is each decode launch's exposed tail).
// Two TMEM accumulators ping-pong so the MMA of the next tile overlaps the epilogue of this one.
// Programmatic dependent launch: weight tiles (which no earlier kernel writes) are requested
// before griddepcontrol.wait, so the weight stream starts under the previous kernel's tail.
#include "gemm_tc.cuh"

namespace bx {


__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void stamp(const EpiParams& E, int idx) {
  if (E.trace != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    E.trace[blockIdx.x * 8 + idx] = t;
  }
}
#ifdef BE_EXP_RR_TRACE  // experiments (scripts/rr_trace.py): per-tile stamps of CTA 0 in
                        // round-robin launches of the epilogue mode named by the macro's value
__device__ unsigned long long g_rr_trace[64][6];
__device__ unsigned long long g_rr_ld[64];
__device__ __forceinline__ void rr_stamp(int seg, int k) {
  if (blockIdx.x == 0 && seg < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_rr_trace[seg][k] = t;
  }
}
extern "C" int be_exp_rr_trace(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_rr_trace, sizeof(g_rr_trace));
}
extern "C" int be_exp_rr_ld(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_rr_ld, sizeof(g_rr_ld));
}
#define RR_STAMP(seg, k) \
  if (RR && MODE == BE_EXP_RR_TRACE) rr_stamp(seg, k)
#else
#define RR_STAMP(seg, k)
#endif
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&p);
}

// Fused epilogue over 16 consecutive token columns [t0, t0+16) of this thread's feature row f
// (all lanes of a warp share t0; lanes hold consecutive features). Stores are vectorised across
// lane pairs: for token pair (2p, 2p+1) one shuffle gives the even lane features (f, f+1) of
// token 2p and the odd lane features (f-1, f) of token 2p+1, so every store is a bf16x2 / float2.
// rs: the chunk's 16 per-token RMSNorm scales (shared memory), nullptr = no norm.
// LoRA delta of feature row f for the chunk's tokens: v[i] += <B_a[f][0..r), u[t][seg*r ..)>.
// B rows are 32 bytes (r = 16 bf16), u slices are broadcast loads shared by the warp. A chunk's
// 16 tokens usually belong to one adapter (batches are segmented by tenant): then B's row is
// loaded once and the u slices of 4 tokens at a time are all in flight together.
__device__ __forceinline__ float lora_dot(const float (&b)[kLoraRank], const float4* u) {
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < kLoraRank / 4; ++q) {
    const float4 uu = u[q];
    acc += b[4 * q] * uu.x + b[4 * q + 1] * uu.y + b[4 * q + 2] * uu.z + b[4 * q + 3] * uu.w;
  }
  return acc;
}
__device__ __forceinline__ void lora_brow(const EpiParams& E, int a, int f, float (&b)[kLoraRank]) {
  const uint4* p = reinterpret_cast<const uint4*>(E.lora_b.p[a] + (size_t)f * kLoraRank);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint4 w = __ldg(p + h);
    const __nv_bfloat162* bb = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 x = __bfloat1622float2(bb[q]);
      b[8 * h + 2 * q] = x.x;
      b[8 * h + 2 * q + 1] = x.y;
    }
  }
}
// lu: the tile's u slices in shared memory, [BN][kLoraRank] from token n0; li: adapters [BN]
__device__ __forceinline__ void lora_add(const EpiParams& E, int f, int tt0, int nvalid,
                                         float (&v)[16], const float* lu, const int* li) {
  const int lane = threadIdx.x & 31;
  const int my_a = (lane & 15) < nvalid ? li[tt0 + (lane & 15)] : -1;
  const int a0 = __shfl_sync(0xffffffffu, my_a, 0);
  const bool uniform = __all_sync(0xffffffffu, (lane & 15) >= nvalid || my_a == a0);
  const float4* ub = reinterpret_cast<const float4*>(lu + (size_t)tt0 * kLoraRank);
  if (uniform) {
    if (a0 < 0) return;
    float b[kLoraRank];
    lora_brow(E, a0, f, b);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < nvalid) v[i] += lora_dot(b, ub + i * (kLoraRank / 4));
    return;
  }
  // mixed adapters in the chunk: per token, static indices so v stays in registers
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i >= nvalid) break;  // warp-uniform
    const int a = __shfl_sync(0xffffffffu, my_a, i);
    if (a < 0) continue;
    float b[kLoraRank];
    lora_brow(E, a, f, b);
    v[i] += lora_dot(b, ub + i * (kLoraRank / 4));
  }
}

template <int MODE>
__device__ __forceinline__ void epilogue_chunk(const EpiParams& E, int f, int t0, float (&v)[16],
                                               const float* rs, const float* lu = nullptr,
                                               const int* li = nullptr, int n0 = 0) {
  // the adapter modes run their base epilogue after adding the LoRA delta
  constexpr int BASE = MODE == kQKVLora ? kQKV
                       : MODE == kResidLora ? kResid
                       : MODE == kResidOutLora ? kResidOut : MODE;
  constexpr bool kLora = MODE >= kQKVLora;
  const int lane = threadIdx.x & 31;
  const bool odd = (lane & 1) != 0;
  const int nvalid = E.ntok - t0 < 16 ? E.ntok - t0 : 16;  // warp-uniform, >= 1
  if (BASE != kQKV && rs != nullptr) {
    // fused RMSNorm row scale (gamma folded into the weights)
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] *= rs[i];
  }
  if constexpr (kLora && BASE != kQKV) lora_add(E, f, t0 - n0, nvalid, v, lu, li);
  if constexpr (BASE == kStore || BASE == kResid || BASE == kResidOut) {
    const int fe = f & ~1;
    float sq[8];  // kResid: this lane's x^2 + x'^2 of token pair p
    float2 xv[8];
    // kResidOut: the chunk's next-hop rows, one load per token (lane i < 16 -> token t0 + i),
    // all issued before the stores below (which might alias them for the compiler)
    int my_dst = -1;
    if constexpr (BASE == kResidOut)
      my_dst = (lane & 15) < nvalid ? __ldg(E.tok + (size_t)(t0 + (lane & 15)) * 5 + 1) : -1;
    if constexpr (BASE == kResid || BASE == kResidOut) {
      // all residual loads of the chunk in flight before the first store (the stores below may
      // alias them as far as the compiler knows, which would serialise 8 L2 round trips)
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int ti = 2 * p + (odd ? 1 : 0);
        xv[p] = ti < nvalid ? __ldcg(reinterpret_cast<const float2*>(E.xres + (size_t)(t0 + ti) * E.ldr + fe))
                            : make_float2(0.f, 0.f);
      }
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const float recv = __shfl_xor_sync(0xffffffffu, odd ? v[2 * p] : v[2 * p + 1], 1);
      const float lo = odd ? recv : v[2 * p];
      const float hi = odd ? v[2 * p + 1] : recv;
      const int t = t0 + 2 * p + (odd ? 1 : 0);
      const bool valid = 2 * p + (odd ? 1 : 0) < nvalid;
      if constexpr (BASE == kStore) {
        if (valid)
          *reinterpret_cast<uint32_t*>(E.out + (size_t)t * E.ldo + fe) = pack_bf16x2(lo, hi);
      } else if constexpr (BASE == kResidOut) {
        const int drow = __shfl_sync(0xffffffffu, my_dst, 2 * p + (odd ? 1 : 0));  // dst_row
        if (valid && drow >= 0)
          *reinterpret_cast<uint32_t*>(E.out + (size_t)drow * E.ldo + fe) =
              pack_bf16x2(xv[p].x + lo, xv[p].y + hi);
      } else {
        sq[p] = 0.f;
        if (valid) {
          float2 x = xv[p];
          x.x += lo;
          x.y += hi;
          *reinterpret_cast<float2*>(E.xres + (size_t)t * E.ldr + fe) = x;
          *reinterpret_cast<uint32_t*>(E.xres_b + (size_t)t * E.ldr + fe) = pack_bf16x2(x.x, x.y);
          sq[p] = x.x * x.x + x.y * x.y;
        }
      }
    }
    if constexpr (BASE == kResid) {
      if (E.ss_out != nullptr) {
        // Sum of squares per token over the warp's 32 features: token 2p + parity lives in the 16
        // lanes of that parity. Transposed butterfly: each xor step halves the values a lane
        // keeps (8 shuffles in all, fixed order), ending with lane bits 4..2 naming p.
        const unsigned full = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool up = lane & 16;
          const float send = up ? sq[i] : sq[i + 4];
          const float keep = up ? sq[i + 4] : sq[i];
          sq[i] = keep + __shfl_xor_sync(full, send, 16);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const bool up = lane & 8;
          const float send = up ? sq[i] : sq[i + 2];
          const float keep = up ? sq[i + 2] : sq[i];
          sq[i] = keep + __shfl_xor_sync(full, send, 8);
        }
        {
          const bool up = lane & 4;
          const float send = up ? sq[0] : sq[1];
          const float keep = up ? sq[1] : sq[0];
          sq[0] = keep + __shfl_xor_sync(full, send, 4);
        }
        sq[0] += __shfl_xor_sync(full, sq[0], 2);
        const int p = ((lane >> 2) & 1) | (((lane >> 3) & 1) << 1) | (((lane >> 4) & 1) << 2);
        const int ti = 2 * p + (odd ? 1 : 0);
        if ((lane & 2) == 0 && ti < nvalid)
          E.ss_out[(size_t)(t0 + ti) * E.ss_groups + (f >> 5)] = sq[0];
      }
    }
  } else if constexpr (BASE == kSwiGLU) {
    // even lane holds gate_j, odd lane holds up_j (rows interleaved at load time)
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const float recv = __shfl_xor_sync(0xffffffffu, odd ? v[2 * p] : v[2 * p + 1], 1);
      const float g = odd ? recv : v[2 * p];
      const float u = odd ? v[2 * p + 1] : recv;
      const int ti = 2 * p + (odd ? 1 : 0);
      if (ti >= nvalid) continue;
      E.out[(size_t)(t0 + ti) * E.ldo + (f >> 1)] = __float2bfloat16_rn(silu(g) * u);
    }
  } else {  // kQKV: rstd, RoPE on q/k, q to the q buffer, k/v to their paged KV slots
    const int d = E.d_model;
    const int sec = f / d;  // warp-uniform (d % 32 == 0)
    const int fi = f - sec * d;
    const int head = fi / E.head_dim;
    const int e = fi - head * E.head_dim;
    // token metadata of the chunk: lane i (< 16) fetches token t0+i, broadcast by shuffles
    const int ti_l = lane & 15;
    const bool have = ti_l < nvalid;
    const int my_slot = have ? __ldg(E.tok + (size_t)(t0 + ti_l) * 5 + 2) : 0;
    const int my_pos = have ? __ldg(E.tok + (size_t)(t0 + ti_l) * 5 + 3) : 0;
    if (rs != nullptr) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] *= rs[i];
    }
    if constexpr (kLora) lora_add(E, f, t0 - n0, nvalid, v, lu, li);
    if (sec < 2) {
      // rows are pair-interleaved per head: even = dim j, odd = dim j + hd/2 (rotate_half).
      // All 16 (cos, sin) loads are issued before the first use: one L2 round trip per chunk.
      float2 cs[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int pos = __shfl_sync(0xffffffffu, my_pos, i);
        const int pc = i < nvalid && pos > 0 ? pos : 0;  // padding rows of a grouped batch: -1
        cs[i] = __ldg(E.rope + (size_t)pc * (E.head_dim >> 1) + (e >> 1));
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float other = __shfl_xor_sync(0xffffffffu, v[i], 1);
        if (i < nvalid)
          v[i] = odd ? v[i] * cs[i].x + other * cs[i].y : v[i] * cs[i].x - other * cs[i].y;
      }
    }
    const int ee = e & ~1;
    const int H = d / E.head_dim;
    __nv_bfloat16* kvp = E.n_grp > 1 ? E.kvgrp[t0 / E.grp_rows] : E.kv_pool;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const float recv = __shfl_xor_sync(0xffffffffu, odd ? v[2 * p] : v[2 * p + 1], 1);
      const float lo = odd ? recv : v[2 * p];
      const float hi = odd ? v[2 * p + 1] : recv;
      const int ti = 2 * p + (odd ? 1 : 0);
      const int slot = __shfl_sync(0xffffffffu, my_slot, ti);
      if (ti >= nvalid) continue;
      if (sec == 0) {
        *reinterpret_cast<uint32_t*>(E.out + (size_t)(t0 + ti) * E.ldo + (fi & ~1)) =
            pack_bf16x2(lo, hi);
      } else if (slot >= 0) {  // padding rows (slot -1) own no KV
        const long long page = slot >> 4;
        const size_t idx = (size_t)(page * E.page_elems + (long long)E.layer * E.layer_elems) +
                           ((size_t)((sec - 1) * H + head) * 16 + (slot & 15)) * E.head_dim + ee;
        *reinterpret_cast<uint32_t*>(kvp + idx) = pack_bf16x2(lo, hi);
      }
    }
  }
}

// kQKV epilogue of one 16-token chunk with the chunk's RoPE (cos, sin) already in registers and
// its (position, KV slot) pairs in shared memory (prefill, whole tiles): same arithmetic and
// stores as epilogue_chunk<kQKV>, no per-token branches before the stores.
__device__ __forceinline__ void qkv_chunk_rr(const EpiParams& E, int f, int t0, float (&v)[16],
                                             const float* rs, const float2 (&cs)[16],
                                             const int2* meta) {
  const int lane = threadIdx.x & 31;
  const bool odd = (lane & 1) != 0;
  const int nvalid = E.ntok - t0 < 16 ? E.ntok - t0 : 16;
  const int d = E.d_model;
  const int sec = f / d;
  const int fi = f - sec * d;
  const int head = fi / E.head_dim;
  const int e = fi - head * E.head_dim;
  if (rs != nullptr) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] *= rs[i];
  }
  if (sec < 2) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float other = __shfl_xor_sync(0xffffffffu, v[i], 1);
      v[i] = odd ? v[i] * cs[i].x + other * cs[i].y : v[i] * cs[i].x - other * cs[i].y;
    }
  }
  const int ee = e & ~1;
  const int H = d / E.head_dim;
  __nv_bfloat16* kvp = E.n_grp > 1 ? E.kvgrp[t0 / E.grp_rows] : E.kv_pool;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const float recv = __shfl_xor_sync(0xffffffffu, odd ? v[2 * p] : v[2 * p + 1], 1);
    const float lo = odd ? recv : v[2 * p];
    const float hi = odd ? v[2 * p + 1] : recv;
    const int ti = 2 * p + (odd ? 1 : 0);
    if (ti >= nvalid) continue;
    if (sec == 0) {
      *reinterpret_cast<uint32_t*>(E.out + (size_t)(t0 + ti) * E.ldo + (fi & ~1)) =
          pack_bf16x2(lo, hi);
    } else {
      const int slot = meta[ti].y;
      if (slot >= 0) {
        const long long page = slot >> 4;
        const size_t idx = (size_t)(page * E.page_elems + (long long)E.layer * E.layer_elems) +
                           ((size_t)((sec - 1) * H + head) * 16 + (slot & 15)) * E.head_dim + ee;
        *reinterpret_cast<uint32_t*>(kvp + idx) = pack_bf16x2(lo, hi);
      }
    }
  }
}

// rs[j] = 1/sqrt(sum_g ss[n0 + j][g] / d + eps) for the BN tokens of a tile; epilogue warp ew of
// epi_warps<BN>() takes tokens ew, ew + epi_warps<BN>(), ...; each lane sums groups lane, lane+32, ... then
// the warp reduces in a fixed order (bit-reproducible).
// All loads are issued before any reduction (one L2 round trip): a token's groups are read as
// float4s, lane l taking float4s l and l + 32 (ss_groups <= 256, i.e. d_model <= 8192).
template <int BN, int kEpiWarps>
__device__ __forceinline__ void tile_rstd(const EpiParams& E, int n0, int q, float* rs) {
  const int lane = threadIdx.x & 31;
  const int G = E.ss_groups;
  const int G4 = G >> 2;
  const float inv_d = 1.0f / (float)(G * 32);
  constexpr int J = (BN + kEpiWarps - 1) / kEpiWarps;  // tokens per warp
  // wide tiles (BN > 64) in rounds of 16 tokens: all 64 at once would exceed the register file
  constexpr int JC = J < 16 ? J : 16;
#pragma unroll 1
  for (int j0 = 0; j0 < J; j0 += JC) {
    float s[JC];
#pragma unroll
    for (int jj = 0; jj < JC; ++jj) {
      const int tt = q + kEpiWarps * (j0 + jj);
      const int t = n0 + tt;
      const float4* p = reinterpret_cast<const float4*>(E.ss_in + (size_t)t * G);
      const bool ok = tt < BN && t < E.ntok;
      const float4 a = (ok && lane < G4) ? __ldcg(p + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 b = (ok && lane + 32 < G4) ? __ldcg(p + lane + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
      s[jj] = ((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w));
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
      for (int jj = 0; jj < JC; ++jj) s[jj] += __shfl_xor_sync(0xffffffffu, s[jj], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int jj = 0; jj < JC; ++jj) {
        const int tt = q + kEpiWarps * (j0 + jj);
        if (tt < BN) rs[tt] = n0 + tt < E.ntok ? rsqrtf(s[jj] * inv_d + E.norm_eps) : 0.f;
      }
    }
  }
}

struct SkRange {
  long long total;  // iterations = tiles * nkb
  int G;            // CTAs
  // 32-bit arithmetic when total * G fits (every shape here): a 64-bit division is a long
  // emulated sequence on the epilogue's critical path
  __device__ __forceinline__ bool narrow() const { return total * G < (1ll << 32); }
  __device__ __forceinline__ long long begin(int c) const {
    return narrow() ? (long long)((unsigned)c * (unsigned)total / (unsigned)G)
                    : (long long)c * total / G;
  }
  // CTA whose range holds iteration it
  __device__ __forceinline__ int cta_of(long long it) const {
    return narrow() ? (int)(((unsigned)(it + 1) * (unsigned)G - 1u) / (unsigned)total)
                    : (int)(((it + 1) * G - 1) / total);
  }
};

// RR: many token tiles (prefill): CTA c takes whole tiles c, c + G, c + 2G, ... so the CTAs in
// flight share a few token tiles and all weight tiles stay L2-resident; the per-CTA iteration
// range [it_begin, it_end) is then virtual (its own tiles back to back).
template <int BN, int STAGES, int CTAS, int MODE, bool RR>
__global__ void __launch_bounds__(64 + 32 * epi_warps<BN, RR>(), CTAS)
    gemm_sk_kernel(const __nv_bfloat16* __restrict__ wpk,
                   const __grid_constant__ CUtensorMap map_x, int K, int m_tiles, int n_tiles,
                   int rr_gm, EpiParams E) {
  using S = GemmSmem<BN>;
  constexpr uint32_t kTmemCols = tmem_cols<2 * BN>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * S::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * S::kBBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* fixbar = tempty + 2;     // the owner's staged partials (split-tile fixup)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(fixbar + 2);  // keeps rs/lu 16B-aligned
  float* rs_smem = reinterpret_cast<float*>(tmem_holder + 4);  // [2][BN] per-token rstd
  float* lu_smem = rs_smem + 2 * BN;                           // k*Lora: [BN][r] u slices
  int* li_smem = reinterpret_cast<int*>(lu_smem + BN * kLoraRank);  // k*Lora: [BN] adapters
  // RR kQKV (never a LoRA mode): [2][BN] (position, KV slot) of the tile's tokens, staged under
  // the mainloop, in the LoRA u region
  int2* meta_smem = reinterpret_cast<int2*>(lu_smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nkb = K / kBK;
  SkRange R{(long long)m_tiles * n_tiles * nkb, (int)gridDim.x};
  const int n_my_tiles =
      RR ? (m_tiles * n_tiles > (int)blockIdx.x
                ? (m_tiles * n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x
                : 0)
         : 0;
  const long long it_begin = RR ? 0 : R.begin(blockIdx.x);
  const long long it_end = RR ? (long long)n_my_tiles * nkb : R.begin(blockIdx.x + 1);
  // real tile of a (virtual) tile index of this CTA's range
  auto real_tile = [&](int vt) { return RR ? (int)blockIdx.x + vt * (int)gridDim.x : vt; };
  // (m, n) of a tile. Stream-K: m fastest. RR: grouped raster - bands of rr_gm weight tiles,
  // token tiles within a band, m fastest inside it - so the ~148 tiles in flight share a few
  // weight tiles AND a few token tiles in L2 (m fastest over all m would re-stream the whole
  // weight matrix from HBM once per token tile).
  auto tile_mn = [&](int tile, int& m, int& n) {
    if (!RR) {
      m = tile % m_tiles;
      n = tile / m_tiles;
      return;
    }
    const int band = tile / (rr_gm * n_tiles);
    const int r = tile - band * rr_gm * n_tiles;
    const int w = m_tiles - band * rr_gm < rr_gm ? m_tiles - band * rr_gm : rr_gm;
    n = r / w;
    m = band * rr_gm + (r - n * w);
  };

  if (threadIdx.x == 0) {
    stamp(E, 0);
    tl_start(E.tl, E.tl_cap);
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], epi_warps<BN, RR>());
    }
    mbar_init(fixbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_launch_dependents();
  if (threadIdx.x == 0) stamp(E, 1);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer: packed weight tiles by bulk copy, activations by TMA
      const long long n_it = it_end - it_begin;
      const int pre = (int)(n_it < STAGES ? n_it : STAGES);
      // (tile, k-block) cursors advanced incrementally: no 64-bit division per load
      struct Cur {
        int tile, kb, m, n;
      };
      const int vt0 = (int)(it_begin / nkb);
      const int tile0 = real_tile(vt0);
      Cur cw{tile0, (int)(it_begin - (long long)vt0 * nkb), 0, 0};
      tile_mn(tile0, cw.m, cw.n);
      Cur cb = cw;
      auto step = [&](Cur& c) {
        if (++c.kb == nkb) {
          c.kb = 0;
          if constexpr (RR) {
            c.tile += (int)gridDim.x;
            tile_mn(c.tile, c.m, c.n);
          } else {
            ++c.tile;
            if (++c.m == m_tiles) {
              c.m = 0;
              ++c.n;
            }
          }
        }
      };
      auto wtile = [&](const Cur& c) {
        const __nv_bfloat16* wb = E.n_grp > 1 ? E.wgrp[c.n] : wpk;  // grouped batch
        return wb + ((size_t)c.m * nkb + c.kb) * (kBM * kBK);
      };
      constexpr uint32_t stage_bytes = S::kStageBytes;
      // weights: streamed once (evict first) unless RR's band shares them across token tiles
      constexpr uint64_t kWPolicy = RR ? kEvictLast : kEvictFirst;
      // weights first: nothing upstream writes them, so they stream under the previous kernel
      for (int i = 0; i < pre; ++i, step(cw)) {
        mbar_arrive_expect_tx(&full[i], stage_bytes);
        bulk_load(sA + i * S::kABytes, wtile(cw), S::kABytes, &full[i], kWPolicy);
      }
      pdl_wait();  // activations are produced by the previous kernel
      stamp(E, 2);
      tl_go(E.tl, E.tl_cap);
      for (int i = 0; i < pre; ++i, step(cb))
        tma_load_2d(&map_x, &full[i], sB + i * S::kBBytes, cb.kb * kBK, cb.n * BN, kEvictLast);
      int s = pre % STAGES;
      uint32_t ph = (uint32_t)(pre / STAGES) & 1u;
      for (long long i = pre; i < n_it; ++i, step(cw)) {
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        bulk_load(sA + s * S::kABytes, wtile(cw), S::kABytes, &full[s], kWPolicy);
        tma_load_2d(&map_x, &full[s], sB + s * S::kBBytes, cw.kb * kBK, cw.n * BN, kEvictLast);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1u;
        }
      }
      stamp(E, 3);
    }
    __syncwarp();  // reconverge before the CTA barrier (barriers are .aligned)
  } else if (warp == 1) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = make_idesc_bf16(kBM, BN);
    int s = 0;  // ring slot and its phase, advanced incrementally
    uint32_t ph = 0;
    int seg = 0;
    int kb0 = (int)(it_begin % nkb);
    for (long long it = it_begin; it < it_end; ++seg) {
      const long long left = it_end - it;
      const int kb1 = (int)((nkb - kb0) < left ? nkb : kb0 + left);
      const int a = seg & 1;
      const uint32_t u = (uint32_t)(seg >> 1);
      if (lane == 0) RR_STAMP(seg, 0);
      mbar_wait(&tempty[a], (u & 1u) ^ 1u);
      tc_fence_after();
      if (lane == 0) RR_STAMP(seg, 1);
      const uint32_t tacc = tmem_base + (uint32_t)(a * BN);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(sA + s * S::kABytes);
          const uint32_t b_addr = smem_u32(sB + s * S::kBBytes);
#ifndef BE_EXP_NO_MMA  // experiments: data movement alone
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            umma_bf16(tacc, make_sdesc_k128(a_addr + k * 32), make_sdesc_k128(b_addr + k * 32),
                      idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
#else
          (void)a_addr;
          (void)b_addr;
          (void)tacc;
#endif
          umma_commit(&empty[s]);
          if (kb == kb1 - 1) {
            umma_commit(&tfull[a]);
            RR_STAMP(seg, 5);
          }
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1u;
        }
      }
      it += kb1 - kb0;
      kb0 = 0;  // later segments start at a tile's first k-block
    }
  } else {
    // ---------------- epilogue warps 2 .. 1 + epi_warps<BN>()
    pdl_wait();
    constexpr int kEpiWarps = epi_warps<BN, RR>();
    constexpr int kEpiThreads = 32 * kEpiWarps;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int ew = warp - 2;  // epilogue warp 0..kEpiWarps-1
    // the tile's token columns split between the warps sharing a lane quarter (16-column chunks)
    constexpr int kHalves = BN / 16 < kEpiWarps / 4 ? BN / 16 : kEpiWarps / 4;
    constexpr int CW = BN / kHalves;
    const int half = ew / 4;
    const int cb = half < kHalves ? half * CW : BN;  // this warp's columns [cb, ce)
    const int ce = half < kHalves ? cb + CW : BN;
    int seg = 0;
    for (long long it = it_begin; it < it_end; ++seg) {
      const int vt = (int)((unsigned)it / (unsigned)nkb);  // it < 2^31
      const int kb0 = (int)it - vt * nkb;
      const int tile = real_tile(vt);
      const long long left = it_end - it;
      const int kb1 = (int)((nkb - kb0) < left ? nkb : kb0 + left);
      it += kb1 - kb0;
      int m_tile, n_tile;
      tile_mn(tile, m_tile, n_tile);
      const int m0 = m_tile * kBM, n0 = n_tile * BN;
      const int f = m0 + q * 32 + lane;
      const int a = seg & 1;
      const uint32_t u = (uint32_t)(seg >> 1);
#ifdef BE_EXP_NO_FIXUP  // experiments: owners finish their own share, no partials (wrong sums)
      const bool owner_only = !(kb0 == 0 && kb1 == nkb) &&
                              (int)blockIdx.x == R.cta_of((long long)tile * nkb);
      const bool whole = (kb0 == 0 && kb1 == nkb) || owner_only;
#else
      const bool whole = kb0 == 0 && kb1 == nkb;
#endif
      const bool runs_epilogue = whole || (int)blockIdx.x == R.cta_of((long long)tile * nkb);
      if constexpr (RR && MODE == kQKV) {
        // the tile's token positions / KV slots for the RoPE and KV stores below (one L2 round
        // trip per tile instead of one per 16-token chunk); double-buffered like rs
        int2* meta = meta_smem + (seg & 1) * BN;
        for (int k = threadIdx.x - 64; k < BN; k += kEpiThreads) {
          const int t = n0 + k;
          meta[k] = t < E.ntok ? make_int2(__ldg(E.tok + (size_t)t * 5 + 3),
                                           __ldg(E.tok + (size_t)t * 5 + 2))
                               : make_int2(0, -1);
        }
        if (E.ss_in == nullptr) named_bar_sync(2, kEpiThreads);
      }
      float* rs = nullptr;
      if (E.ss_in != nullptr && runs_epilogue) {
        // the norm statistics of this tile's tokens, computed under the mainloop (or reduced
        // once per token by launch_rstd for round-robin launches)
        rs = rs_smem + (seg & 1) * BN;
        if (E.rs_in != nullptr) {
          for (int k = threadIdx.x - 64; k < BN; k += kEpiThreads)
            rs[k] = n0 + k < E.ntok ? __ldg(E.rs_in + n0 + k) : 0.f;
        } else {
          tile_rstd<BN, kEpiWarps>(E, n0, ew, rs);
        }
        named_bar_sync(2, kEpiThreads);
      }
      if constexpr (MODE >= kQKVLora) {
        if (runs_epilogue) {
          // the tile's LoRA u slices (its 128 rows lie in one q / k / v segment) and adapters
          named_bar_sync(3, kEpiThreads);  // the previous tile's readers are done with the buffer
          const int et = threadIdx.x - 64;  // epilogue thread
          const int sg = m0 / E.lora_seg;
          float4* lu4 = reinterpret_cast<float4*>(lu_smem);
          for (int k = et; k < BN * (kLoraRank / 4); k += kEpiThreads) {
            const int tt = k / (kLoraRank / 4), qq = k % (kLoraRank / 4);
            lu4[k] = n0 + tt < E.ntok
                         ? __ldg(reinterpret_cast<const float4*>(
                               E.lora_u + (size_t)(n0 + tt) * E.lora_ustride + sg * kLoraRank) + qq)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          for (int k = et; k < BN; k += kEpiThreads) li_smem[k] = n0 + k < E.ntok ? __ldg(E.lora_idx + n0 + k) : -1;
          named_bar_sync(3, kEpiThreads);
        }
      }
      if (warp == 2 && lane == 0) RR_STAMP(seg, 2);
      mbar_wait(&tfull[a], u & 1u);
      tc_fence_after();
      if (warp == 2 && lane == 0) RR_STAMP(seg, 3);
      if (warp == 2 && lane == 0) stamp(E, 4);  // overwritten: the last segment's accumulator
      __syncwarp();
#if defined(BE_EXP_NO_EPI) || defined(BE_EXP_NO_EPI_MODE)
      // experiments: the mainloop alone (no partials, no fixup, no stores), for every mode or
      // for one epilogue mode only
#ifdef BE_EXP_NO_EPI_MODE
      if (MODE == BE_EXP_NO_EPI_MODE) {
#else
      if (true) {
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
        continue;
      }
#endif
      const uint32_t t_lane = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * BN);
      if (RR && MODE == kQKV) {
        // prefill QKV: the next chunk's RoPE (cos, sin) loads are in flight while this chunk
        // is rotated and stored
        const int2* meta = meta_smem + (seg & 1) * BN;
        const bool rope = f / E.d_model < 2;  // q / k rows (warp-uniform)
        const int e2 = ((f % E.d_model) % E.head_dim) >> 1;
        float2 csa[16], csb[16];
        auto load_cs = [&](int c0, float2 (&cs)[16]) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int pos = meta[c0 + i].x;
            cs[i] = __ldg(E.rope + (size_t)(pos > 0 ? pos : 0) * (E.head_dim >> 1) + e2);
          }
        };
        if (rope && cb < ce && n0 + cb < E.ntok) load_cs(cb, csa);
#pragma unroll 1
        for (int c0 = cb; c0 < ce; c0 += 32) {
          if (n0 + c0 >= E.ntok) break;
          float acc[16];
          if (rope && c0 + 16 < ce && n0 + c0 + 16 < E.ntok) load_cs(c0 + 16, csb);
          tmem_ld16(t_lane + c0, acc);
          qkv_chunk_rr(E, f, n0 + c0, acc, rs ? rs + c0 : nullptr, csa, meta + c0);
          if (c0 + 16 >= ce || n0 + c0 + 16 >= E.ntok) break;
          if (rope && c0 + 32 < ce && n0 + c0 + 32 < E.ntok) load_cs(c0 + 32, csa);
          tmem_ld16(t_lane + c0 + 16, acc);
          qkv_chunk_rr(E, f, n0 + c0 + 16, acc, rs ? rs + c0 + 16 : nullptr, csb, meta + c0 + 16);
        }
      } else if (whole) {
#pragma unroll 1
        for (int c0 = cb; c0 < ce; c0 += 16) {
          if (n0 + c0 >= E.ntok) break;
          float acc[16];
          tmem_ld16(t_lane + c0, acc);
          epilogue_chunk<MODE>(E, f, n0 + c0, acc, rs ? rs + c0 : nullptr, lu_smem, li_smem, n0);
        }
      } else {
        // Partial tile. Its owner is the CTA holding the tile's first k-block (c_first): for
        // that CTA the tile is its LAST segment, so it finishes last. Every other contributor
        // holds the tile as its FIRST (or only) segment: it writes its partial to its single
        // slot and releases one count on the tile's counter, usually long before the owner
        // gets there. The owner never writes its own partial: it acquires the counter (all
        // contributors are resident: grid <= #SMs, one CTA per SM), reads the partials with
        // every load in flight and runs the epilogue. Sum order is contributor order.
        const long long tile_it0 = (long long)tile * nkb;
        const int c_first = R.cta_of(tile_it0);
        const int c_last = R.cta_of(tile_it0 + nkb - 1);
        const int n_contrib = c_last - c_first + 1;
        // partial layout [BN/4][128 rows] of float4 (4 consecutive tokens of one feature row): a
        // warp instruction moves 32 consecutive rows = 512 contiguous bytes (4 L2 lines, not 32)
        const int row = q * 32 + lane;
        auto part4 = [&](int c) {
          return reinterpret_cast<float4*>(E.ws + (size_t)c * BN * kBM);
        };
        int* ctr = E.counters + tile;
        if (E.trace != nullptr && warp == 2 && lane == 0)  // diagnostics: last segment's role
          E.trace[blockIdx.x * 8 + 6] = (int)blockIdx.x == c_first ? 1000000 + n_contrib : 2000000;
#ifdef BE_EXP_NO_FIXUP
        if (true) {
        } else
#endif
        if ((int)blockIdx.x != c_first) {
          float4* slot = part4(blockIdx.x) + row;
#pragma unroll 1
          for (int c0 = cb; c0 < ce; c0 += 16) {
            if (n0 + c0 >= E.ntok) break;
            float acc[16];
            tmem_ld16(t_lane + c0, acc);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              __stcg(slot + ((c0 >> 2) + j) * kBM,
                     make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]));
          }
          // the CTA barrier orders the epilogue threads' stores before one release at GPU scope
          // (release is cumulative; no sequentially-consistent fence on the hot path)
          named_bar_sync(1, kEpiThreads);
          if (warp == 2 && lane == 0)
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ctr) : "memory");
        } else {
          if (warp == 2 && lane == 0) {
            int seen = 0;
            do {
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
            } while (seen < n_contrib - 1);
            *ctr = 0;  // reset for the next launch / graph replay (ordered by kernel boundary)
          }
          __syncwarp();
          named_bar_sync(1, kEpiThreads);  // everyone's loads are ordered after the acquire
          if constexpr (BN <= 64) {
            // whole tile in registers; the contributors' partials are staged into the ring
            // (idle now: this is the CTA's last segment and its MMAs are complete) by bulk
            // copies, every partial of a round in flight at once - one L2 round trip per round
            // instead of one per contributor - and summed from shared memory in contributor
            // order (deterministic)
            float acc[CW];  // this warp's columns [cb, cb + CW) (a warp past kHalves has none)
            const bool mine = half < kHalves;
            if (mine) {
#pragma unroll
              for (int c = 0; c < CW; c += 16)
                tmem_ld16(t_lane + cb + c, *reinterpret_cast<float(*)[16]>(acc + c));
            }
            constexpr int kPartBytes = BN * kBM * 4;
            constexpr int kPerRound = STAGES * S::kStageBytes / kPartBytes;
            static_assert(kPerRound >= 1, "ring smaller than one partial tile");
            const float4* staged = reinterpret_cast<const float4*>(smem);
            uint32_t fph = 0;
            for (int o0 = 1; o0 < n_contrib; o0 += kPerRound) {
              const int nr = n_contrib - o0 < kPerRound ? n_contrib - o0 : kPerRound;
              if (warp == 2 && lane == 0) {
                // the acquire above ordered the contributors' stores; order the async-proxy
                // reads after it
                asm volatile("fence.proxy.async.global;" ::: "memory");
                mbar_arrive_expect_tx(fixbar, (uint32_t)(nr * kPartBytes));
                for (int j = 0; j < nr; ++j)
                  bulk_load(smem + j * kPartBytes, part4(c_first + o0 + j), kPartBytes, fixbar,
                            kEvictFirst);
              }
              mbar_wait(fixbar, fph);
              fph ^= 1u;
              for (int j = 0; mine && j < nr; ++j) {
                const float4* p = staged + (size_t)j * (kPartBytes / 16) + row + (cb / 4) * kBM;
#pragma unroll
                for (int k = 0; k < CW / 4; ++k) {
                  const float4 v = p[k * kBM];
                  acc[4 * k] += v.x;
                  acc[4 * k + 1] += v.y;
                  acc[4 * k + 2] += v.z;
                  acc[4 * k + 3] += v.w;
                }
              }
              if (o0 + kPerRound < n_contrib) named_bar_sync(1, kEpiThreads);  // ring reused
            }
#pragma unroll
            for (int c = 0; c < CW; c += 16) {
              if (!mine || n0 + cb + c >= E.ntok) break;
              epilogue_chunk<MODE>(E, f, n0 + cb + c, *reinterpret_cast<float(*)[16]>(acc + c),
                                   rs ? rs + cb + c : nullptr, lu_smem, li_smem, n0);
            }
          } else {
#pragma unroll 1
          for (int c0 = cb; c0 < ce; c0 += 16) {
            if (n0 + c0 >= E.ntok) break;
            float acc[16];
            tmem_ld16(t_lane + c0, acc);  // the owner's share is contributor 0
            for (int o0 = 1; o0 < n_contrib; o0 += 4) {
              float4 v[4][4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int o = o0 + j;
                const float4* p = part4(c_first + (o < n_contrib ? o : 0)) + row + (c0 >> 2) * kBM;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  v[j][k] = o < n_contrib ? __ldcg(p + k * kBM) : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  acc[4 * k] += v[j][k].x;
                  acc[4 * k + 1] += v[j][k].y;
                  acc[4 * k + 2] += v[j][k].z;
                  acc[4 * k + 3] += v[j][k].w;
                }
              }
            }
            epilogue_chunk<MODE>(E, f, n0 + c0, acc, rs ? rs + c0 : nullptr, lu_smem, li_smem, n0);
          }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (warp == 2 && lane == 0) RR_STAMP(seg, 4);
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
    if (warp == 2 && lane == 0) stamp(E, 5);
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    stamp(E, 7);
    tl_end(E.tl, E.tl_cap);
  }
  if (warp == 1) tmem_free<kTmemCols>(tmem_base);
}

template <int BN, int MODE, bool RR>
static cudaError_t launch_bn_rr(const GemmLaunch& L, cudaStream_t stream) {
  constexpr int STAGES = gemm_stages_deep<BN>();
  constexpr int CTAS = gemm_ctas<BN>();  // resident CTAs per SM the register budget allows
  constexpr int smem = STAGES * GemmSmem<BN>::kStageBytes + 1024 /*align*/ + 256 /*barriers*/ +
                       2 * BN * 4 /*rstd*/ +
                       (MODE >= kQKVLora ? BN * (kLoraRank + 1) * 4 : 0) /*LoRA u, adapters*/ +
                       (RR && MODE == kQKV ? 2 * BN * 8 : 0) /*token metadata*/;
  auto kern = gemm_sk_kernel<BN, STAGES, CTAS, MODE, RR>;
  static unsigned long long configured = 0;  // per device: the attribute is device state
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> dev & 1ull)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured |= 1ull << dev;
  }
  const int m_tiles = L.N / kBM;
  const int n_tiles = (L.epi.ntok + BN - 1) / BN;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.grid, 1, 1);
  cfg.blockDim = dim3(64 + 32 * epi_warps<BN, RR>(), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = L.pdl ? 1 : 0;
  // RR band width in weight tiles (BE_GEMM_RR_GM: experiments; 0 = all of them, m fastest)
  static const int kRRGm = [] {
    const char* e = getenv("BE_GEMM_RR_GM");
    return e ? atoi(e) : 16;
  }();
  const int rr_gm = kRRGm > 0 && kRRGm < m_tiles ? kRRGm : m_tiles;
  return cudaLaunchKernelEx(&cfg, kern, L.w_packed, *L.map_x, L.K, m_tiles, n_tiles, rr_gm,
                            L.epi);
}

// the round-robin variant only for wide tiles (prefill-sized token counts)
template <int BN, int MODE>
static cudaError_t launch_bn(const GemmLaunch& L, cudaStream_t stream) {
  if constexpr (BN == 256 && MODE != kQKVLora && MODE != kResidLora && MODE != kResidOutLora) {
    if (L.rr) return launch_bn_rr<BN, MODE, true>(L, stream);
  }
  return launch_bn_rr<BN, MODE, false>(L, stream);
}

template <int MODE>
static cudaError_t launch_mode(const GemmLaunch& L, cudaStream_t stream) {
  switch (L.bn) {
    case 16: return launch_bn<16, MODE>(L, stream);
    case 32: return launch_bn<32, MODE>(L, stream);
    case 64: return launch_bn<64, MODE>(L, stream);
    case 128: return launch_bn<128, MODE>(L, stream);
    case 256: return launch_bn<256, MODE>(L, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemm(const GemmLaunch& L, cudaStream_t stream) {
  if (L.N % kBM != 0 || L.K % kBK != 0 || L.grid < 1) return cudaErrorInvalidValue;
  switch (L.epi.mode) {
    case kStore: return launch_mode<kStore>(L, stream);
    case kResid: return launch_mode<kResid>(L, stream);
    case kSwiGLU: return launch_mode<kSwiGLU>(L, stream);
    case kQKV: return launch_mode<kQKV>(L, stream);
    case kResidOut: return launch_mode<kResidOut>(L, stream);
    case kQKVLora: return launch_mode<kQKVLora>(L, stream);
    case kResidLora: return launch_mode<kResidLora>(L, stream);
    case kResidOutLora: return launch_mode<kResidOutLora>(L, stream);
    default: return cudaErrorInvalidValue;
  }
}

// one warp per token, the same lane split, float4 sums and butterfly order as tile_rstd
__global__ void __launch_bounds__(256) rstd_kernel(const float* __restrict__ ss, int G, int ntok,
                                                   float eps, float* __restrict__ rstd) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= ntok) return;
  const int G4 = G >> 2;
  const float4* p = reinterpret_cast<const float4*>(ss + (size_t)t * G);
  const float4 a = lane < G4 ? __ldcg(p + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 b = lane + 32 < G4 ? __ldcg(p + lane + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
  float s = ((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w));
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) rstd[t] = rsqrtf(s * (1.0f / (float)(G * 32)) + eps);
}

cudaError_t launch_rstd(const float* ss, int groups, int ntok, float eps, float* rstd,
                        cudaStream_t stream) {
  if (ntok <= 0) return cudaSuccess;
  rstd_kernel<<<(ntok + 7) / 8, 256, 0, stream>>>(ss, groups, ntok, eps, rstd);
  return cudaGetLastError();
}

int gemm_pick_bn(int ntok) {
  // BE_GEMM_BN256_MIN: smallest batch that takes 256-token tiles (4-stage ring) instead of
  // 128-token ones (6 stages); experiments only
  static const int kBn256Min = [] {
    const char* e = getenv("BE_GEMM_BN256_MIN");
    return e ? atoi(e) : 129;
  }();
  if (ntok <= 16) return 16;
  if (ntok <= 32) return 32;
  if (ntok <= 64) return 64;
  if (ntok <= 128 || ntok < kBn256Min) return 128;
  return 256;
}

GemmPlan gemm_plan(int N, int K, int ntok, int bn, int num_sms, size_t ws_elems, int n_counters,
                   int grid_cap) {
  GemmPlan p{};
  const int m_tiles = N / kBM;
  const int n_tiles = (ntok + bn - 1) / bn;
  const long long tiles = (long long)m_tiles * n_tiles;
  const int nkb = K / kBK;
  const long long total = tiles * nkb;
  // Grid: every SM streams (stream-K ranges over all 148), measured best since the partial fixup
  // became cheap (coalesced partials): all-SM stream-K beat whole tiles on 128 CTAs by 2.3% and
  // the min-CTA knob is flat (profiles/r01_gemm_sweep_gmin.log). BE_GEMM_WHOLE=1 / BE_GEMM_GMIN
  // restore the whole-tile preference / fewer even splits for experiments.
  static const int kMinStreamCtas = [] {
    const char* e = getenv("BE_GEMM_GMIN");
    return e ? atoi(e) : 148;
  }();
  static const bool kWholeTiles = [] {
    const char* e = getenv("BE_GEMM_WHOLE");
    return e ? atoi(e) != 0 : false;
  }();
  const long long sms = grid_cap > 0 && grid_cap < num_sms ? grid_cap : num_sms;
  long long g = sms;
  if (tiles >= sms) {
    const long long k = (tiles + sms - 1) / sms;  // whole tiles per CTA
    if (kWholeTiles && tiles % k == 0 && tiles / k >= kMinStreamCtas) g = tiles / k;
  } else if (tiles >= kMinStreamCtas) {
    if (kWholeTiles) g = tiles;  // one whole tile per CTA
  } else {
    const long long s = (kMinStreamCtas + tiles - 1) / tiles;  // even k-splits per tile
    g = tiles * s < sms ? tiles * s : sms;
  }
  // many token tiles (prefill): whole tiles dealt round-robin, the CTAs in flight share a few
  // token tiles (BE_GEMM_RR=0 keeps stream-K ranges)
  static const bool kRR = [] {
    const char* e = getenv("BE_GEMM_RR");
    return e ? atoi(e) != 0 : true;
  }();
  if (kRR && bn == 256 && n_tiles > 16 && tiles >= 4 * sms) {  // M > 4096: measured crossover
    p.grid = (int)sms;
    p.ws_needed = 0;
    p.tiles = tiles;
    p.rr = 1;
    return p;
  }
  if (g > total / 4) g = total / 4 > 0 ? total / 4 : 1;
  // partial-tile slots: one per CTA (its first segment; owners never publish theirs)
  while (g > 1 && (size_t)g * bn * kBM > ws_elems) g /= 2;
  (void)n_counters;
  p.grid = (int)g;
  p.ws_needed = (size_t)g * bn * kBM;
  p.tiles = tiles;
  return p;
}

}  // namespace bx
