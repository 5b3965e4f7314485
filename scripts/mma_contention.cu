// Does the tensor pipe slow the incoming weight stream? One CTA per SM streams a share of a
// 2 GB buffer through a 6-stage x 16 KB bulk-copy ring (the GEMM producer's scheme) while an
// independent warp issues back-to-back tcgen05.mma (M=128, N=64, K=16, SS) on a separate
// resident tile: stream rate with 0 / 1 / 2 MMA per 16 KB received.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/mma_contention.cu -o scripts/mma_contention
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2404_18322_b200/csrc/ptx.cuh"

using namespace bx;
constexpr int CH = 16384, ST = 6;

__global__ void __launch_bounds__(96, 1) stream_mma(const uint8_t* buf, size_t per_cta, int mma_per_chunk,
                                                    int* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = sm;                      // ST x 16 KB
  uint8_t* sA = sm + ST * CH;              // 16 KB resident A
  uint8_t* sB = sA + CH;                   // 8 KB resident B
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + 8192);
  uint64_t* empty = full + ST;
  uint64_t* mbar = empty + ST;
  uint32_t* holder = reinterpret_cast<uint32_t*>(mbar + 2);
  volatile int* done = reinterpret_cast<volatile int*>(holder + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(mbar, 1);
    *done = 0;
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<64>(holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  const uint8_t* base = buf + (size_t)blockIdx.x * per_cta;
  const long long n = per_cta / CH;
  if (warp == 0 && lane == 0) {
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % ST);
      mbar_wait(&empty[s], (uint32_t)((i / ST) & 1) ^ 1u);
      mbar_arrive_expect_tx(&full[s], CH);
      bulk_load(ring + s * CH, base + i * CH, CH, &full[s], kEvictFirst);
    }
  } else if (warp == 1) {
    int acc = 0;
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % ST);
      mbar_wait(&full[s], (uint32_t)((i / ST) & 1));
      acc += ring[s * CH + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (lane == 0) *done = 1;
    if (acc == 12345678) *sink = acc;
  } else if (warp == 2 && lane == 0 && mma_per_chunk > 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, 64);
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    long long k = 0;
    while (*done == 0) {
      umma_bf16(tmem, make_sdesc_k128(a + (k & 3) * 32), make_sdesc_k128(b + (k & 3) * 32), idesc, 1u);
      ++k;
      if ((k & 63) == 0) {  // bounded queue: wait for the issued MMAs now and then
        umma_commit(mbar);
        mbar_wait(mbar, (uint32_t)(((k >> 6) - 1) & 1));
      }
    }
    if (k == 1234567) *sink = (int)k;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_free<64>(tmem);
}

int main() {
  const size_t bytes = (size_t)2 << 30;
  uint8_t* buf;
  int* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = ST * CH + CH + 8192 + 256 + 1024;
  cudaFuncSetAttribute(stream_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const size_t per = (bytes / sms) / CH * CH;
  for (int m : {0, 1, 0, 1}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    stream_mma<<<sms, 96, smem>>>(buf, per, m, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) stream_mma<<<sms, 96, smem>>>(buf, per, m, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("stream with %s MMAs beside it: %.0f GB/s (%s)\n", m ? "continuous" : "no",
           (double)per * sms * 3 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
