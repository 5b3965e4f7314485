// Microbenchmark: per-launch time of a pure weight stream of GEMM-sized buffers (33.5 MB = the
// 7B O projection, 100 MB QKV, 180 MB gate/up, 90 MB down) by the GEMM's producer scheme
// (persistent CTA per SM, 16 KB bulk copies into an 8-stage ring): the floor a decode GEMM of
// that size can reach per launch. Buffers rotate over 2 GB so nothing is served from L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/bulk_small.cu -o scripts/bulk_small
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2404_18322_b200/csrc/ptx.cuh"

using namespace bx;

template <int CHUNK, int STAGES>
__global__ void __launch_bounds__(64, 1) stream_bulk(const uint8_t* buf, size_t total, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const long long nch = total / CHUNK;
  const long long b = nch * blockIdx.x / gridDim.x, e = nch * (blockIdx.x + 1) / gridDim.x;
  if (warp == 0 && lane == 0) {
    for (long long i = b; i < e; ++i) {
      const long long k = i - b;
      const int s = (int)(k % STAGES);
      mbar_wait(&empty[s], (uint32_t)((k / STAGES) & 1) ^ 1u);
      mbar_arrive_expect_tx(&full[s], CHUNK);
      bulk_load(sm + s * CHUNK, buf + i * CHUNK, CHUNK, &full[s], kEvictFirst);
    }
  } else if (warp == 1) {
    int acc = 0;
    for (long long i = b; i < e; ++i) {
      const long long k = i - b;
      const int s = (int)(k % STAGES);
      mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
      acc += sm[s * CHUNK + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 12345678) *sink = acc;
  }
}

int main() {
  const size_t span = (size_t)2 << 30;
  uint8_t* buf;
  int* sink;
  cudaMalloc(&buf, span);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, span);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  constexpr int CH = 16384, ST = 8;
  const int smem = ST * CH + 2 * ST * 8 + 64;
  cudaFuncSetAttribute(stream_bulk<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const size_t sizes[] = {33554432, 100663296, 134217728, 180355072, 90177536, 721420288};
  for (size_t sz : sizes) {
    const int n = (int)(span / sz);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int r = 0; r < n; ++r) stream_bulk<CH, ST><<<sms, 64, smem>>>(buf + r * sz, sz, sink);
    cudaEventRecord(a);
    const int reps = 3 * n;
    for (int r = 0; r < reps; ++r) stream_bulk<CH, ST><<<sms, 64, smem>>>(buf + (r % n) * sz, sz, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / reps;
    printf("bulk stream %7.1f MB: %7.2f us per launch = %6.0f GB/s (%s)\n", sz / 1048576.0, us,
           sz / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
