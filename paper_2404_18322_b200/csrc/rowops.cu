// Row kernels of the per-block path:
//   K1 gather  : routing-table gather of per-request activation rows into the block batch
//   K2 scatter : batch rows back to their next-hop rows of the activation arena
//   K7 cosine  : predicted-vs-actual per-row cosine + accept verdict (speculation check)
//   synth_init : counter-mode splitmix64 synthetic weights/inputs (identical bits to oracle/)
// All HBM-bound: 16-byte vector accesses, one warp (or CTA) per row, grid >= 148 * k.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "ptx.cuh"
#include "gemm_tc.cuh"

namespace bx {

// ---------------------------------------------------------------- K1 gather
// X[i] = float(arena[src[i]]), Xb[i] = arena[src[i]]; optional fp32 copy for the residual stream
// and the per-(row, 32-feature group) sums of squares the first fused RMSNorm reads (ss[r][g]).
// Four consecutive threads cover one group (8 features each); d % 32 == 0 keeps them in a warp.
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ arena,
                                   const int* __restrict__ src, int src_stride, int rows, int d,
                                   __nv_bfloat16* __restrict__ xb, float* __restrict__ x,
                                   float* __restrict__ ss, unsigned long long* tl, int tl_cap) {
  if (threadIdx.x == 0) {
    tl_start(tl, tl_cap);
    tl_go(tl, tl_cap);
  }
  // 32-bit index math (rows * d / 8 < 2^31, checked by the launcher): no 64-bit division
  const unsigned vec_per_row = (unsigned)d / 8u;
  const unsigned total = (unsigned)rows * vec_per_row;
  const unsigned stride = gridDim.x * blockDim.x;
  // every thread runs the same trip count so the group shuffles below see full warps
  const unsigned trips = (total + stride - 1) / stride;
  const unsigned v0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (unsigned k = 0; k < trips; ++k) {
    const unsigned v = v0 + k * stride;
    const bool live = v < total;
    const int r = live ? (int)(v / vec_per_row) : 0;
    const int c = live ? (int)(v - (unsigned)r * vec_per_row) : 0;
    float sq = 0.f;
    if (live) {
      const uint4 val = __ldg(reinterpret_cast<const uint4*>(arena + (size_t)src[(size_t)r * src_stride] * d) + c);
      reinterpret_cast<uint4*>(xb + (size_t)r * d)[c] = val;
      if (x != nullptr) {
        const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&val);
        float f[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(b[i]);
        float4* px = reinterpret_cast<float4*>(x + (size_t)r * d) + 2 * c;
        px[0] = make_float4(f[0], f[1], f[2], f[3]);
        px[1] = make_float4(f[4], f[5], f[6], f[7]);
        // pairwise (x0^2 + x1^2) like the GEMM epilogue, then left to right
#pragma unroll
        for (int i = 0; i < 8; i += 2) sq += f[i] * f[i] + f[i + 1] * f[i + 1];
      }
    }
    if (ss != nullptr) {
      sq += __shfl_xor_sync(0xffffffffu, sq, 1);
      sq += __shfl_xor_sync(0xffffffffu, sq, 2);
      if (live && (c & 3) == 0) ss[(size_t)r * (d / 32) + (c >> 2)] = sq;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) tl_end(tl, tl_cap);
}

// ---------------------------------------------------------------- K2 scatter
__global__ void scatter_rows_kernel(const __nv_bfloat16* __restrict__ xb,
                                    const int* __restrict__ dst, int dst_stride, int rows, int d,
                                    __nv_bfloat16* __restrict__ arena, unsigned long long* tl,
                                    int tl_cap) {
  if (threadIdx.x == 0) {
    tl_start(tl, tl_cap);
    tl_go(tl, tl_cap);
  }
  const unsigned vec_per_row = (unsigned)d / 8u;
  const unsigned total = (unsigned)rows * vec_per_row;
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < total; v += gridDim.x * blockDim.x) {
    const int r = (int)(v / vec_per_row);
    const int c = (int)(v - (unsigned)r * vec_per_row);
    const int drow = dst[(size_t)r * dst_stride];
    if (drow < 0) continue;  // token output not needed downstream
    const uint4 val = reinterpret_cast<const uint4*>(xb + (size_t)r * d)[c];
    reinterpret_cast<uint4*>(arena + (size_t)drow * d)[c] = val;
  }
  __syncthreads();
  if (threadIdx.x == 0) tl_end(tl, tl_cap);
}

// ---------------------------------------------------------------- K7 cosine
// cos[r] = <a_r, b_r> / (|a_r| |b_r|) in fp32; accept[r] = cos[r] >= thr. One warp per row.
__global__ void cosine_rows_kernel(const __nv_bfloat16* __restrict__ a,
                                   const __nv_bfloat16* __restrict__ b, int rows, int d,
                                   float thr, float* __restrict__ cos_out,
                                   int* __restrict__ accept) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const uint4* pa = reinterpret_cast<const uint4*>(a + (size_t)warp * d);
  const uint4* pb = reinterpret_cast<const uint4*>(b + (size_t)warp * d);
  float dot = 0.f, na = 0.f, nb = 0.f;
  for (int c = lane; c < d / 8; c += 32) {
    const uint4 va = __ldcs(pa + c), vb = __ldcs(pb + c);
    const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&va);
    const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&vb);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 fa = __bfloat1622float2(ha[i]);
      const float2 fb = __bfloat1622float2(hb[i]);
      dot = fmaf(fa.x, fb.x, fmaf(fa.y, fb.y, dot));
      na = fmaf(fa.x, fa.x, fmaf(fa.y, fa.y, na));
      nb = fmaf(fb.x, fb.x, fmaf(fb.y, fb.y, nb));
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    dot += __shfl_xor_sync(0xffffffffu, dot, off);
    na += __shfl_xor_sync(0xffffffffu, na, off);
    nb += __shfl_xor_sync(0xffffffffu, nb, off);
  }
  if (lane == 0) {
    // zero-norm rows have no defined cosine (the reference throws): report NaN, reject
    const float c = (na > 0.f && nb > 0.f) ? dot / (sqrtf(na) * sqrtf(nb)) : __int_as_float(0x7fc00000);
    cos_out[warp] = c;
    if (accept != nullptr) accept[warp] = (c >= thr) ? 1 : 0;
  }
}

// ---------------------------------------------------------------- synthetic init
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// value of logical element i of the tensor whose stream key is `key` (see oracle/synth.h)
__device__ __forceinline__ float synth_value(uint64_t key, uint64_t i, float scale) {
  const uint64_t z = mix64(key + (i + 1) * 0x9e3779b97f4a7c15ull);
  const float u = (float)(z >> 40) * (1.0f / 16777216.0f);
  return (2.0f * u - 1.0f) * scale;
}

// Physical row layouts (see gemm QKV/SwiGLU epilogues):
//   perm 0: identity
//   perm 1: q/k rotate_half pair interleave inside each head (phys 2j <- j, 2j+1 <- j + hd/2)
//   perm 2: gate/up interleave (phys 2j <- gate j, 2j+1 <- up j), two keys
// dst holds `rows` physical rows of `cols`; gamma (optional, length cols) is folded in.
// src_cols: logical row stride of the generated stream (>= cols: a column prefix of a wider
// matrix, the pruned FFN of a speculation surrogate)
__global__ void synth_weight_kernel(__nv_bfloat16* __restrict__ dst, int rows, int cols,
                                    uint64_t key0, uint64_t key1, float scale, int perm,
                                    int head_dim, const float* __restrict__ gamma, int src_cols) {
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int pr = (int)(idx / cols);
    const int c = (int)(idx - (long long)pr * cols);
    int lr = pr;
    uint64_t key = key0;
    if (perm == 1) {
      const int h = pr / head_dim, e = pr - h * head_dim;
      lr = h * head_dim + ((e & 1) ? (e >> 1) + head_dim / 2 : (e >> 1));
    } else if (perm == 2) {
      lr = pr >> 1;
      key = (pr & 1) ? key1 : key0;
    }
    float v = synth_value(key, (uint64_t)lr * src_cols + c, scale);
    v = __bfloat162float(__float2bfloat16_rn(v));  // logical bf16 weight
    if (gamma != nullptr) v *= gamma[c];
    dst[packed_index(pr, c, cols)] = __float2bfloat16_rn(v);  // GEMM-ready tile layout
  }
}

// LoRA adapter factors in plain row-major layout: rows of the logical stream, perm 1 = the q/k
// rotate_half pair interleave of the GEMM rows they feed (same row map as synth_weight_kernel)
__global__ void synth_plain_kernel(__nv_bfloat16* __restrict__ dst, int rows, int cols,
                                   uint64_t key, float scale, int perm, int head_dim) {
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int pr = (int)(idx / cols);
    const int c = (int)(idx - (long long)pr * cols);
    int lr = pr;
    if (perm == 1) {
      const int h = pr / head_dim, e = pr - h * head_dim;
      lr = h * head_dim + ((e & 1) ? (e >> 1) + head_dim / 2 : (e >> 1));
    }
    dst[idx] = __float2bfloat16_rn(synth_value(key, (uint64_t)lr * cols + c, scale));
  }
}

// LoRA shrink (segmented by adapter): u[t][j] = scale_t * <A_{a(t)}[j], x[t]> for j < r3, where
// a(t) = idx[t] (-1: no adapter, u = 0) and scale_t = rstd of the token's fused RMSNorm (from the
// residual producer's sums of squares, as the GEMM computes it) or 1 without a norm. One CTA per
// (token, 8 rows of A): the token's row is staged in shared memory as fp32, each warp takes one
// A row with 16-byte loads, all of them in flight (d <= 8192: at most 32 per lane).
__global__ void __launch_bounds__(256) lora_shrink_kernel(
    const __nv_bfloat16* __restrict__ x, int ldx, int d, const float* __restrict__ ss,
    int ss_groups, float eps, const __grid_constant__ LoraTable A, int r3,
    const int* __restrict__ idx,
    float* __restrict__ u) {
  extern __shared__ float xs[];
  const int t = blockIdx.x;
  const int a = idx[t];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (a < 0) {
    const int j = blockIdx.y * 8 + (int)threadIdx.x;
    if (threadIdx.x < 8 && j < r3) u[(size_t)t * r3 + j] = 0.f;
    return;
  }
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t)t * ldx);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) {
    const uint4 w = xr[c];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(h[q]);
      xs[8 * c + 2 * q] = f.x;
      xs[8 * c + 2 * q + 1] = f.y;
    }
  }
  __shared__ float s_scale;
  if (warp == 0) {
    float sc = 1.f;
    if (ss != nullptr) {
      float sum = 0.f;
      for (int g = lane; g < ss_groups; g += 32) sum += ss[(size_t)t * ss_groups + g];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      sc = rsqrtf(sum / (float)d + eps);
    }
    if (lane == 0) s_scale = sc;
  }
  __syncthreads();
  const int nv = d / 8 / 32;  // uint4 loads per lane per row
  // blockIdx.y picks this CTA's 8 rows of A (one per warp)
  for (int j = blockIdx.y * 8 + warp; j < r3 && j < blockIdx.y * 8 + 8; j += 8) {
    const uint4* row = reinterpret_cast<const uint4*>(A.p[a] + (size_t)j * d);
    float acc = 0.f;
#pragma unroll 16
    for (int i = 0; i < nv; ++i) {
      const int c = lane + 32 * i;
      const uint4 w = __ldg(row + c);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
      const float* xv = xs + 8 * c;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h[q]);
        acc += f.x * xv[2 * q] + f.y * xv[2 * q + 1];
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) u[(size_t)t * r3 + j] = acc * s_scale;
  }
}

// row-major [rows][cols] -> packed tile layout (ptx.cuh packed_index)
__global__ void pack_weight_kernel(const __nv_bfloat16* __restrict__ src,
                                   __nv_bfloat16* __restrict__ dst, int rows, int cols) {
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / cols), c = (int)(idx - (long long)r * cols);
    dst[packed_index(r, c, cols)] = src[idx];
  }
}

__global__ void synth_rows_kernel(__nv_bfloat16* __restrict__ dst, long long n, uint64_t key,
                                  float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(synth_value(key, (uint64_t)i, scale));
}

// rope[pos][j] = (cos, sin)(pos * theta^(-2j/hd)), computed in double for both sides
__global__ void rope_table_kernel(float2* __restrict__ rope, int max_pos, int head_dim,
                                  double theta) {
  const int half = head_dim / 2;
  const long long total = (long long)max_pos * half;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int pos = (int)(i / half), j = (int)(i - (long long)pos * half);
    const double inv = pow(theta, -2.0 * j / head_dim);
    const double ang = (double)pos * inv;
    rope[i] = make_float2((float)cos(ang), (float)sin(ang));
  }
}

// ---------------------------------------------------------------- launchers
static inline int grid_for(long long work, int threads, int cap) {
  long long g = (work + threads - 1) / threads;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_gather(const __nv_bfloat16* arena, const int* src, int src_stride, int rows,
                          int d, __nv_bfloat16* xb, float* x, float* ss, cudaStream_t st,
                          unsigned long long* tl, int tl_cap) {
  if (rows <= 0) return cudaSuccess;
  if ((long long)rows * d / 8 >= (1ll << 31)) return cudaErrorInvalidValue;  // 32-bit indexing
  gather_rows_kernel<<<grid_for((long long)rows * d / 8, 256, 148 * 16), 256, 0, st>>>(
      arena, src, src_stride, rows, d, xb, x, ss, tl, tl_cap);
  return cudaGetLastError();
}
cudaError_t launch_scatter(const __nv_bfloat16* xb, const int* dst, int dst_stride, int rows,
                           int d, __nv_bfloat16* arena, cudaStream_t st, unsigned long long* tl,
                           int tl_cap) {
  if (rows <= 0) return cudaSuccess;
  if ((long long)rows * d / 8 >= (1ll << 31)) return cudaErrorInvalidValue;  // 32-bit indexing
  scatter_rows_kernel<<<grid_for((long long)rows * d / 8, 256, 148 * 16), 256, 0, st>>>(
      xb, dst, dst_stride, rows, d, arena, tl, tl_cap);
  return cudaGetLastError();
}
cudaError_t launch_cosine(const __nv_bfloat16* a, const __nv_bfloat16* b, int rows, int d,
                          float thr, float* cos_out, int* accept, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  cosine_rows_kernel<<<(rows + 7) / 8, 256, 0, st>>>(a, b, rows, d, thr, cos_out, accept);
  return cudaGetLastError();
}
cudaError_t launch_synth_weight(__nv_bfloat16* dst, int rows, int cols, uint64_t key0,
                                uint64_t key1, float scale, int perm, int head_dim,
                                const float* gamma, cudaStream_t st, int src_cols) {
  synth_weight_kernel<<<grid_for((long long)rows * cols, 256, 148 * 32), 256, 0, st>>>(
      dst, rows, cols, key0, key1, scale, perm, head_dim, gamma, src_cols > 0 ? src_cols : cols);
  return cudaGetLastError();
}
cudaError_t launch_synth_plain(__nv_bfloat16* dst, int rows, int cols, uint64_t key, float scale,
                               int perm, int head_dim, cudaStream_t st) {
  synth_plain_kernel<<<grid_for((long long)rows * cols, 256, 148 * 32), 256, 0, st>>>(
      dst, rows, cols, key, scale, perm, head_dim);
  return cudaGetLastError();
}
cudaError_t launch_lora_shrink(const __nv_bfloat16* x, int ldx, int d, const float* ss,
                               int ss_groups, float eps, const LoraTable& A, int r3,
                               const int* idx, float* u, int ntok, cudaStream_t st) {
  if (ntok <= 0) return cudaSuccess;
  if (d % 256 != 0 || d > 8192) return cudaErrorInvalidValue;  // whole uint4 sweeps per lane
  lora_shrink_kernel<<<dim3(ntok, (r3 + 7) / 8), 256, d * sizeof(float), st>>>(x, ldx, d, ss, ss_groups, eps, A, r3,
                                                            idx, u);
  return cudaGetLastError();
}
cudaError_t launch_pack_weight(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int cols,
                               cudaStream_t st) {
  pack_weight_kernel<<<grid_for((long long)rows * cols, 256, 148 * 32), 256, 0, st>>>(src, dst, rows, cols);
  return cudaGetLastError();
}
cudaError_t launch_synth_rows(__nv_bfloat16* dst, long long n, uint64_t key, float scale,
                              cudaStream_t st) {
  synth_rows_kernel<<<grid_for(n, 256, 148 * 32), 256, 0, st>>>(dst, n, key, scale);
  return cudaGetLastError();
}
cudaError_t launch_rope_table(float2* rope, int max_pos, int head_dim, double theta,
                              cudaStream_t st) {
  rope_table_kernel<<<grid_for((long long)max_pos * head_dim / 2, 256, 148 * 8), 256, 0, st>>>(
      rope, max_pos, head_dim, theta);
  return cudaGetLastError();
}

}  // namespace bx
