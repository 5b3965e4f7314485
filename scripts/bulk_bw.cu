// Microbenchmark: HBM read bandwidth of per-SM streaming schemes on B200 (design evidence for
// the GEMM producer). Each persistent CTA streams a contiguous 1/grid share of a buffer into a
// shared-memory ring; a consumer warp releases slots as they land.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/bulk_bw.cu -o bulk_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2404_18322_b200/csrc/ptx.cuh"

using namespace bx;

template <int CHUNK, int STAGES, int SPLIT>
__global__ void __launch_bounds__(64, 1) stream_bulk(const uint8_t* buf, size_t per_cta, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* base = buf + (size_t)blockIdx.x * per_cta;
  const long long n = per_cta / CHUNK;
  if (warp == 0 && lane == 0) {
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % STAGES);
      mbar_wait(&empty[s], (uint32_t)((i / STAGES) & 1) ^ 1u);
      mbar_arrive_expect_tx(&full[s], CHUNK);
#pragma unroll
      for (int k = 0; k < SPLIT; ++k)
        bulk_load(sm + s * CHUNK + k * (CHUNK / SPLIT), base + i * CHUNK + k * (CHUNK / SPLIT),
                  CHUNK / SPLIT, &full[s], kEvictFirst);
    }
  } else if (warp == 1) {
    int acc = 0;
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % STAGES);
      mbar_wait(&full[s], (uint32_t)((i / STAGES) & 1));
      acc += sm[s * CHUNK + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 12345678) *sink = acc;
  }
}

__global__ void stream_ldg(const uint4* buf, size_t n_vec, int* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_vec;
       i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(buf + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = (int)acc;
}

template <int CHUNK, int STAGES, int SPLIT>
float run(const uint8_t* buf, size_t bytes, int grid, int* sink) {
  const size_t per = (bytes / grid) / CHUNK * CHUNK;
  const int smem = STAGES * CHUNK + 2 * STAGES * 8 + 64;
  cudaFuncSetAttribute(stream_bulk<CHUNK, STAGES, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  stream_bulk<CHUNK, STAGES, SPLIT><<<grid, 64, smem>>>(buf, per, sink);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) stream_bulk<CHUNK, STAGES, SPLIT><<<grid, 64, smem>>>(buf, per, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double gbs = (double)per * grid * reps / (ms / 1e3) / 1e9;
  printf("bulk chunk=%6d stages=%2d split=%d grid=%d: %.0f GB/s  (%s)\n", CHUNK, STAGES, SPLIT, grid,
         gbs, cudaGetErrorString(cudaGetLastError()));
  return (float)gbs;
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
  run<16384, 8, 1>(buf, bytes, sms, sink);
  run<16384, 12, 1>(buf, bytes, sms, sink);
  run<16384, 8, 4>(buf, bytes, sms, sink);
  run<32768, 6, 1>(buf, bytes, sms, sink);
  run<32768, 6, 8>(buf, bytes, sms, sink);
  run<8192, 24, 1>(buf, bytes, sms, sink);
  run<4096, 48, 1>(buf, bytes, sms, sink);
  run<16384, 8, 1>(buf, bytes, 2 * sms, sink);
  run<16384, 12, 1>(buf, bytes, sms / 2, sink);
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    stream_ldg<<<sms * 8, 512>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) stream_ldg<<<sms * 8, 512>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg grid=%d x 512: %.0f GB/s\n", sms * 8, (double)bytes * 5 / (ms / 1e3) / 1e9);
  }
  return 0;
}
