// tcgen05 / TMEM / TMA block-forward GEMM (see gemm_tc.cuh for the contract).
#include "gemm_tc.cuh"

namespace bx {

// Applies the fused epilogue to 16 consecutive token columns [c0, c0+16) of this thread's
// feature row f. `t0` is the first token index of the chunk; all lanes of a warp share t0.
template <int BN>
__device__ __forceinline__ void epilogue_chunk(const EpiParams& E, int N, int f, int t0,
                                               const float (&acc)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int t = t0 + i;
    const bool valid = t < E.ntok;  // warp-uniform
    float v = acc[i];
    if (E.rstd != nullptr && valid) v *= E.rstd[t];
    if (E.mode == kResid) {
      if (valid) {
        float* px = E.xres + (size_t)t * E.ldr + f;
        const float nv = *px + v;
        *px = nv;
        E.xres_b[(size_t)t * E.ldr + f] = __float2bfloat16_rn(nv);
      }
    } else if (E.mode == kStore) {
      if (valid) E.out[(size_t)t * E.ldo + f] = __float2bfloat16_rn(v);
    } else if (E.mode == kSwiGLU) {
      const float other = __shfl_xor_sync(0xffffffffu, v, 1);
      if (valid && (lane & 1) == 0) {
        // even lane holds gate_j, odd lane holds up_j
        E.out[(size_t)t * E.ldo + (f >> 1)] = __float2bfloat16_rn(silu(v) * other);
      }
    } else {  // kQKV
      const int d = E.d_model;
      const int sec = f / d;  // 0 q, 1 k, 2 v (warp-uniform: d % 32 == 0)
      const int fi = f - sec * d;
      const int head = fi / E.head_dim;
      const int e = fi - head * E.head_dim;
      const float other = __shfl_xor_sync(0xffffffffu, v, 1);
      if (!valid) continue;
      float o = v;
      if (sec < 2) {
        // rows are pair-interleaved per head: even = dim j, odd = dim j + hd/2 (rotate_half)
        const float2 cs = E.rope[(size_t)E.tok[t * 5 + 3] * (E.head_dim >> 1) + (e >> 1)];
        o = (lane & 1) == 0 ? v * cs.x - other * cs.y : v * cs.x + other * cs.y;
      }
      if (sec == 0) {
        E.out[(size_t)t * E.ldo + fi] = __float2bfloat16_rn(o);
      } else {
        const int slot = E.tok[t * 5 + 2];
        const long long page = slot >> 4;
        const int tok = slot & 15;
        const int H = d / E.head_dim;
        const size_t idx = (size_t)(page * E.page_elems + (long long)E.layer * E.layer_elems) +
                           ((size_t)((sec - 1) * H + head) * 16 + tok) * E.head_dim + e;
        E.kv_pool[idx] = __float2bfloat16_rn(o);
      }
    }
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_w,
                   const __grid_constant__ CUtensorMap map_x, int N, int K, int ksplit,
                   EpiParams E) {
  using S = GemmSmem<BN>;
  constexpr uint32_t kTmemCols = tmem_cols<BN>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * S::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * S::kBBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* accum_full = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accum_full + 1);
  int* flag = reinterpret_cast<int*>(tmem_holder + 1);

  const int warp = threadIdx.x >> 5;
  const int m_tile = blockIdx.x;
  const int n_tile = blockIdx.y;
  const int split = blockIdx.z;
  const int m0 = m_tile * kBM;
  const int n0 = n_tile * BN;

  const int num_kb = K / kBK;
  const int kb_begin = (int)((long long)split * num_kb / ksplit);
  const int kb_end = (int)((long long)(split + 1) * num_kb / ksplit);
  const int nkb = kb_end - kb_begin;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], S::kStageBytes);
        const int kc = (kb_begin + i) * kBK;
        tma_load_2d(&map_w, &full[s], sA + s * S::kABytes, kc, m0, kEvictFirst);
        tma_load_2d(&map_x, &full[s], sB + s * S::kBBytes, kc, n0, kEvictLast);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = make_idesc_bf16(kBM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a_addr = smem_u32(sA + s * S::kABytes);
        const uint32_t b_addr = smem_u32(sB + s * S::kBBytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          // advance 16 bf16 (32 B) along K inside the 128B swizzle atom
          const uint64_t da = make_sdesc_k128(a_addr + k * 32);
          const uint64_t db = make_sdesc_k128(b_addr + k * 32);
          umma_bf16(tmem_base, da, db, idesc, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
        if (i == nkb - 1) umma_commit(accum_full);
      }
      __syncwarp();
    }
  }

  // ---------------- epilogue: all 4 warps, warp w owns TMEM lanes [32w, 32w+32)
  mbar_wait(accum_full, 0);
  tc_fence_after();
  const int f = m0 + warp * 32 + (threadIdx.x & 31);
  const uint32_t t_lane = tmem_base + ((uint32_t)(warp * 32) << 16);
  const int n_tiles = gridDim.y;

  if (ksplit == 1) {
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      if (n0 + c0 >= E.ntok) break;
      float acc[16];
      tmem_ld16(t_lane + c0, acc);
      epilogue_chunk<BN>(E, N, f, n0 + c0, acc);
    }
  } else {
    // publish this split's partial, last arriver reduces and runs the epilogue
    float* my_ws = E.ws + ((size_t)(split * n_tiles + n_tile) * BN) * N;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      if (n0 + c0 >= E.ntok) break;
      float acc[16];
      tmem_ld16(t_lane + c0, acc);
#pragma unroll
      for (int i = 0; i < 16; ++i) __stcg(my_ws + (size_t)(c0 + i) * N + f, acc[i]);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      int* ctr = E.counters + m_tile * n_tiles + n_tile;
      const int prev = atomicAdd(ctr, 1);
      const int last = prev == ksplit - 1;
      if (last) *ctr = 0;  // self-reset for the next launch / graph replay
      *flag = last;
    }
    __syncthreads();
    if (*flag) {
      __threadfence();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        if (n0 + c0 >= E.ntok) break;
        float acc[16];
        tmem_ld16(t_lane + c0, acc);
        for (int s2 = 0; s2 < ksplit; ++s2) {
          if (s2 == split) continue;
          const float* ws = E.ws + ((size_t)(s2 * n_tiles + n_tile) * BN) * N;
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] += __ldcg(ws + (size_t)(c0 + i) * N + f);
        }
        epilogue_chunk<BN>(E, N, f, n0 + c0, acc);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_free<kTmemCols>(tmem_base);
}

template <int BN>
static cudaError_t launch_bn(const GemmLaunch& L, cudaStream_t stream) {
  constexpr int STAGES = gemm_stages<BN>();
  constexpr int smem = STAGES * GemmSmem<BN>::kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
  auto kern = gemm_tc_kernel<BN, STAGES>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(L.N / kBM, (L.epi.ntok + BN - 1) / BN, L.ksplit);
  kern<<<grid, 128, smem, stream>>>(*L.map_w, *L.map_x, L.N, L.K, L.ksplit, L.epi);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmLaunch& L, cudaStream_t stream) {
  if (L.N % kBM != 0 || L.K % kBK != 0 || L.ksplit < 1 || L.ksplit > L.K / kBK)
    return cudaErrorInvalidValue;
  switch (L.bn) {
    case 16: return launch_bn<16>(L, stream);
    case 32: return launch_bn<32>(L, stream);
    case 64: return launch_bn<64>(L, stream);
    case 128: return launch_bn<128>(L, stream);
    case 256: return launch_bn<256>(L, stream);
    default: return cudaErrorInvalidValue;
  }
}

int gemm_pick_bn(int ntok) {
  if (ntok <= 16) return 16;
  if (ntok <= 32) return 32;
  if (ntok <= 64) return 64;
  if (ntok <= 128) return 128;
  return 256;
}

int gemm_pick_ksplit(int N, int K, int ntok, int bn, int num_sms) {
  const int tiles = (N / kBM) * ((ntok + bn - 1) / bn);
  const int nkb = K / kBK;
  if (tiles >= num_sms) return 1;
  // smallest split that fills the SMs, keeping >= 4 K-blocks per split
  int best = 1;
  for (int s = 1; s <= 16; ++s) {
    if (nkb / s < 4) break;
    best = s;
    if (tiles * s >= num_sms) break;
  }
  return best;
}

}  // namespace bx
