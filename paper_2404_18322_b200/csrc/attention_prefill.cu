// Causal prefill attention over the paged KV pool on tensor cores (K3 for prefill batches).
//
// The decode kernel (attention.cu) gives every query row its own pass over the row's pages:
// right for decode (one row per request), quadratic in KV traffic for a prompt. Here a CTA
// takes a tile of up to 64 query rows of one request (rows whose (page-table row, pos / 64) agree
// - consecutive prompt tokens) and one head, and streams that request's K/V in 64-token tiles
// (4 pages) through shared memory once for all 64 rows: S = Q K^T and O += P V on
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate), online softmax in registers (flash-attention
// style), causal mask on the diagonal tile. Warp w owns query rows 16w..16w+15 of the tile.
//
// Tiles are found on the device (the batch metadata lives there): tile_index_kernel marks rows
// that start a tile and compacts them with a block scan; the attention kernel is persistent over
// (tile, head) items.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cfloat>

#include "ptx.cuh"

namespace bx {

struct PrefillAttnParams {
  const __nv_bfloat16* q;     // [rows][H*hd] (q/k head dims pair-interleaved, see gemm QKV)
  const __nv_bfloat16* pool;  // KV pool
  long long page_elems;
  long long layer_elems;
  int layer;
  const int* page_table;      // [n_pt][pt_stride]
  int pt_stride;
  const int* tok;             // be_token records (stride 5): [2] kv_slot, [3] pos, [4] pt_row
  int rows;
  int H;
  float scale_log2;
  __nv_bfloat16* out;         // [rows][H*hd]
  int* tiles;                 // [rows + 2] tile start rows, the count at tiles[rows], a work
                              // counter at tiles[rows + 1]
};

// One CTA, up to 1024 threads: row r starts a tile if r == 0 or its (pt_row, pos >> shift)
// differs from row r-1's (64-row tiles here, 128 for the tcgen05 kernel); starts are compacted in
// order (block-wide scan in chunks).
__global__ void tile_index_kernel(const int* __restrict__ tok, int rows, int* __restrict__ tiles,
                                  int shift) {
  __shared__ int warp_sums[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r0 = 0; r0 < rows; r0 += blockDim.x) {
    const int r = r0 + threadIdx.x;
    int start = 0;
    if (r < rows) {
      const int key_pt = tok[(size_t)r * 5 + 4], key_p = tok[(size_t)r * 5 + 3] >> shift;
      start = r == 0 || tok[(size_t)(r - 1) * 5 + 4] != key_pt ||
              (tok[(size_t)(r - 1) * 5 + 3] >> shift) != key_p;
    }
    // inclusive scan of `start` over the block
    int v = start;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v += n;
    }
    if (lane == 31) warp_sums[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += n;
      }
      warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int before = (warp > 0 ? warp_sums[warp - 1] : 0) + v - start;
    if (start) tiles[base + before] = r;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base += before + start;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tiles[rows] = base;
    tiles[rows + 1] = 0;  // work counter of the tcgen05 kernel's dynamic item queue
  }
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&p);
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// B fragments of two 8x8 bf16 tiles stacked along k, from a row-major [k][n] smem tile:
// lanes 0-15 address rows k0..k0+15 (16-byte aligned), .trans hands thread (g, t) the pairs
// (k = 2t, 2t+1 | n = g) of each tile - the m16n8k16 "col" operand.
__device__ __forceinline__ void ldsm_x2_trans(uint32_t& b0, uint32_t& b1, const void* row) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(row));
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
               : "=r"(b0), "=r"(b1)
               : "r"(a));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 16 : 0));  // src-size 0: zero fill
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Four 8x8 bf16 tiles (no transpose): lane l addresses row (l & 7) of tile l >> 3.
__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        const void* row) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(row));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}

template <int HD>
__global__ void __launch_bounds__(128) attn_prefill_kernel(PrefillAttnParams P) {
  constexpr int BR = 64, BC = 64;
  constexpr int LD = HD + 8;  // padded smem row (bf16): conflict-free fragment loads
  constexpr int KS = HD / 16; // k-steps over the head dim
  // K/V tiles double-buffered: tile kt+1 streams in (cp.async) while tile kt is consumed
  extern __shared__ __align__(16) uint8_t smem_pf[];
  auto sKb = reinterpret_cast<__nv_bfloat16(*)[BC][LD]>(smem_pf);
  auto sVb = reinterpret_cast<__nv_bfloat16(*)[BC][LD]>(smem_pf + 2 * BC * LD * 2);
  __shared__ int sPos[BR];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n_tiles = P.tiles[P.rows];
  const size_t v_off = (size_t)P.H * 16 * HD;

  for (int item = blockIdx.x; item < n_tiles * P.H; item += gridDim.x) {
    const int tile = item / P.H, head = item - tile * P.H;
    const int r0 = P.tiles[tile];
    const int r1 = tile + 1 < n_tiles ? P.tiles[tile + 1] : P.rows;
    const int nr = r1 - r0;  // <= 64 rows of one request
    const int pt_row = P.tok[(size_t)r0 * 5 + 4];
    const int* pt = P.page_table + (size_t)pt_row * P.pt_stride;
    __syncthreads();  // previous item done with sPos / sK / sV
    if (threadIdx.x < BR) sPos[threadIdx.x] = threadIdx.x < nr ? P.tok[(size_t)(r0 + threadIdx.x) * 5 + 3] : -1;
    __syncthreads();
    int max_pos = 0;
    for (int i = 0; i < nr; ++i) max_pos = max(max_pos, sPos[i]);
    // this warp's rows: tile rows 16*warp + g and + 8
    const int ra = 16 * warp + g, rb = ra + 8;
    const int pa = sPos[ra], pb = sPos[rb];
    // Q fragments (prescaled into log2 units) for all k-steps
    uint32_t qf[KS][4];
    {
      const __nv_bfloat16* qa = P.q + (size_t)(r0 + (ra < nr ? ra : 0)) * P.H * HD + head * HD;
      const __nv_bfloat16* qb = P.q + (size_t)(r0 + (rb < nr ? rb : 0)) * P.H * HD + head * HD;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int c = ks * 16 + 2 * t;
        auto ld = [&](const __nv_bfloat16* base, int col) {
          const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(base + col);
          const float2 f = __bfloat1622float2(v);
          return pack2(f.x * P.scale_log2, f.y * P.scale_log2);
        };
        qf[ks][0] = ld(qa, c);
        qf[ks][1] = ld(qb, c);
        qf[ks][2] = ld(qa, c + 8);
        qf[ks][3] = ld(qb, c + 8);
      }
    }
    float o[HD / 8][4];
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float ma = -FLT_MAX, mb = -FLT_MAX, la = 0.f, lb = 0.f;

    const int n_kt = max_pos / BC + 1;
    // K/V of tokens [kt*64, kt*64+64): 4 pages, each head's 16 x HD run contiguous
    auto load_tile = [&](int kt, int buf) {
      constexpr int kChunks = BC * HD / 8;  // 16-byte chunks per tile
      for (int c = threadIdx.x; c < kChunks; c += blockDim.x) {
        const int tok = c / (HD / 8), col = (c % (HD / 8)) * 8;
        const int p = kt * BC + tok;
        const int page = p <= max_pos ? pt[p >> 4] : -1;
        const size_t off = page >= 0 ? (size_t)page * P.page_elems +
                                           (size_t)P.layer * P.layer_elems +
                                           ((size_t)head * 16 + (p & 15)) * HD + col
                                     : 0;
        cp_async16(&sKb[buf][tok][col], P.pool + off, page >= 0);
        cp_async16(&sVb[buf][tok][col], P.pool + off + v_off, page >= 0);
      }
      cp_async_commit();
    };
    __syncthreads();  // the previous item is done with both buffers
    load_tile(0, 0);
    for (int kt = 0; kt < n_kt; ++kt) {
      const int buf = kt & 1;
      if (kt + 1 < n_kt) {
        load_tile(kt + 1, buf ^ 1);
        cp_async_wait<1>();  // tile kt landed (kt + 1 may still be in flight)
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      auto& sK = sKb[buf];
      auto& sV = sVb[buf];
      // S = Q K^T: 16 rows x 64 keys per warp (8 n-tiles of 8 keys)
      float s[BC / 8][4];
#pragma unroll
      for (int j = 0; j < BC / 8; ++j) {
        s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < KS; ks += 2) {
          // K rows j*8.. as the B operand of k-steps ks and ks+1 in one ldmatrix
          uint32_t b0, b1, b2, b3;
          ldsm_x4(b0, b1, b2, b3, &sK[j * 8 + (lane & 7)][ks * 16 + (lane >> 3) * 8]);
          mma16816(s[j], qf[ks], b0, b1);
          mma16816(s[j], qf[ks + 1], b2, b3);
        }
      }
      // causal mask (key position <= query position), then online softmax in log2 units
      float mxa = ma, mxb = mb;
#pragma unroll
      for (int j = 0; j < BC / 8; ++j) {
        const int k0 = kt * BC + j * 8 + 2 * t;
        if (k0 > pa) s[j][0] = -FLT_MAX;
        if (k0 + 1 > pa) s[j][1] = -FLT_MAX;
        if (k0 > pb) s[j][2] = -FLT_MAX;
        if (k0 + 1 > pb) s[j][3] = -FLT_MAX;
        mxa = fmaxf(mxa, fmaxf(s[j][0], s[j][1]));
        mxb = fmaxf(mxb, fmaxf(s[j][2], s[j][3]));
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, off));
        mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, off));
      }
      const float ca = ma == -FLT_MAX ? 0.f : exp2f(ma - mxa);
      const float cb = mb == -FLT_MAX ? 0.f : exp2f(mb - mxb);
      float sa = 0.f, sb = 0.f;
      uint32_t pf[BC / 16][4];  // P as A fragments of the PV mma (two S n-tiles per k-step)
#pragma unroll
      for (int j = 0; j < BC / 8; ++j) {
        const float p0 = s[j][0] == -FLT_MAX ? 0.f : exp2f(s[j][0] - mxa);
        const float p1 = s[j][1] == -FLT_MAX ? 0.f : exp2f(s[j][1] - mxa);
        const float p2 = s[j][2] == -FLT_MAX ? 0.f : exp2f(s[j][2] - mxb);
        const float p3 = s[j][3] == -FLT_MAX ? 0.f : exp2f(s[j][3] - mxb);
        sa += p0 + p1;
        sb += p2 + p3;
        const int kk = j >> 1;
        if ((j & 1) == 0) {
          pf[kk][0] = pack2(p0, p1);
          pf[kk][1] = pack2(p2, p3);
        } else {
          pf[kk][2] = pack2(p0, p1);
          pf[kk][3] = pack2(p2, p3);
        }
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, off);
        sb += __shfl_xor_sync(0xffffffffu, sb, off);
      }
      la = la * ca + sa;
      lb = lb * cb + sb;
      ma = mxa;
      mb = mxb;
      // O = O * corr + P V: 16 rows x HD per warp (HD/8 n-tiles), k = 64 keys (4 k-steps)
#pragma unroll
      for (int j = 0; j < HD / 8; ++j) {
        o[j][0] *= ca;
        o[j][1] *= ca;
        o[j][2] *= cb;
        o[j][3] *= cb;
#pragma unroll
        for (int kk = 0; kk < BC / 16; ++kk) {
          uint32_t b0, b1;
          ldsm_x2_trans(b0, b1, &sV[kk * 16 + (lane & 15)][j * 8]);
          mma16816(o[j], pf[kk], b0, b1);
        }
      }
      __syncthreads();  // every warp is done with this buffer before it is refilled
    }
    // normalise and store this warp's rows
    const float ia = la > 0.f ? 1.f / la : 0.f, ib = lb > 0.f ? 1.f / lb : 0.f;
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      const int col = head * HD + j * 8 + 2 * t;
      if (ra < nr)
        *reinterpret_cast<uint32_t*>(P.out + (size_t)(r0 + ra) * P.H * HD + col) =
            pack2(o[j][0] * ia, o[j][1] * ia);
      if (rb < nr)
        *reinterpret_cast<uint32_t*>(P.out + (size_t)(r0 + rb) * P.H * HD + col) =
            pack2(o[j][2] * ib, o[j][3] * ib);
    }
  }
}

cudaError_t launch_tile_index(const int* tok, int rows, int* tiles, int shift, cudaStream_t stream) {
  tile_index_kernel<<<1, 1024, 0, stream>>>(tok, rows, tiles, shift);
  return cudaGetLastError();
}

cudaError_t launch_attention_prefill(const PrefillAttnParams& P, int head_dim, int num_sms,
                                     cudaStream_t stream) {
  if (P.rows <= 0) return cudaSuccess;
  tile_index_kernel<<<1, 1024, 0, stream>>>(P.tok, P.rows, P.tiles, 6);
  const int grid = num_sms * 4;
  auto run = [&](auto kern, int hd) {
    const int smem = 2 * 2 * 64 * (hd + 8) * 2;  // [K,V][2 buffers][64][hd + 8] bf16
    static int configured = 0;  // per head dim, per device (bit)
    int dev = 0;
    cudaGetDevice(&dev);
    const int bit = (hd == 128 ? 1 : 2) << (2 * dev);
    if (!(configured & bit)) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      configured |= bit;
    }
    kern<<<grid, 128, smem, stream>>>(P);
    return cudaGetLastError();
  };
  if (head_dim == 128) return run(attn_prefill_kernel<128>, 128);
  if (head_dim == 64) return run(attn_prefill_kernel<64>, 64);
  return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace bx
