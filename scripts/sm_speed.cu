// Per-SM HBM streaming speed under full load: is the ~20% spread between SMs a stable property
// of the SM (so a static split could weight it) or launch-to-launch noise?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/sm_speed.cu -o sm_speed
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_2404_18322_b200/csrc/ptx.cuh"

using namespace bx;

constexpr int CHUNK = 16384, STAGES = 8;

__global__ void __launch_bounds__(64, 1) stream_timed(const uint8_t* buf, size_t per_cta,
                                                      unsigned long long* rec, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long t0 = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  }
  __syncthreads();
  const uint8_t* base = buf + (size_t)blockIdx.x * per_cta;
  const long long n = per_cta / CHUNK;
  if (warp == 0 && lane == 0) {
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % STAGES);
      mbar_wait(&empty[s], (uint32_t)((i / STAGES) & 1) ^ 1u);
      mbar_arrive_expect_tx(&full[s], CHUNK);
      bulk_load(sm + s * CHUNK, base + i * CHUNK, CHUNK, &full[s], kEvictFirst);
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
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t1, smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    unsigned int s32;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s32));
    smid = s32;
    rec[blockIdx.x * 3 + 0] = smid;
    rec[blockIdx.x * 3 + 1] = t0;
    rec[blockIdx.x * 3 + 2] = t1;
  }
}

int main() {
  const int grid = 148;
  const size_t per = (size_t)4 << 20;  // 4 MB per CTA: 592 MB total (> L2)
  uint8_t* buf;
  cudaMalloc(&buf, per * grid);
  cudaMemset(buf, 1, per * grid);
  unsigned long long* rec;
  cudaMalloc(&rec, grid * 3 * sizeof(unsigned long long));
  int* sink;
  cudaMalloc(&sink, 4);
  const int smem = STAGES * CHUNK + 2 * STAGES * 8 + 64;
  cudaFuncSetAttribute(stream_timed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int runs = 8;
  std::vector<std::vector<double>> t(runs, std::vector<double>(grid, 0));  // by smid
  for (int r = 0; r < runs + 1; ++r) {
    stream_timed<<<grid, 64, smem>>>(buf, per, rec, sink);
    cudaDeviceSynchronize();
    if (r == 0) continue;  // warm-up
    std::vector<unsigned long long> h(grid * 3);
    cudaMemcpy(h.data(), rec, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[c * 3 + 1]);
    for (int c = 0; c < grid; ++c) {
      const int smid = (int)h[c * 3];
      if (smid < grid) t[r - 1][smid] = (h[c * 3 + 2] - h[c * 3 + 1]) / 1e3;  // us
    }
  }
  // per-SM mean, spread, and run-to-run correlation of per-SM times
  std::vector<double> mean(grid, 0);
  for (int s = 0; s < grid; ++s) {
    for (int r = 0; r < runs; ++r) mean[s] += t[r][s];
    mean[s] /= runs;
  }
  auto corr = [&](const std::vector<double>& a, const std::vector<double>& b) {
    double ma = 0, mb = 0;
    for (int i = 0; i < grid; ++i) { ma += a[i]; mb += b[i]; }
    ma /= grid; mb /= grid;
    double sab = 0, saa = 0, sbb = 0;
    for (int i = 0; i < grid; ++i) {
      sab += (a[i] - ma) * (b[i] - mb); saa += (a[i] - ma) * (a[i] - ma); sbb += (b[i] - mb) * (b[i] - mb);
    }
    return sab / std::sqrt(saa * sbb);
  };
  double cavg = 0;
  int nc = 0;
  for (int r = 0; r < runs; ++r)
    for (int q = r + 1; q < runs; ++q) { cavg += corr(t[r], t[q]); ++nc; }
  const auto mm = std::minmax_element(mean.begin(), mean.end());
  double avg = 0;
  for (double v : mean) avg += v;
  avg /= grid;
  printf("per-SM time for 4 MB under full load: mean %.1f us, min %.1f, max %.1f (max/mean %.3f)\n",
         avg, *mm.first, *mm.second, *mm.second / avg);
  printf("run-to-run correlation of per-SM times (avg over %d pairs): %.3f\n", nc, cavg / nc);
  for (int r = 0; r < runs; ++r) {
    const auto m2 = std::minmax_element(t[r].begin(), t[r].end());
    printf("run %d: min %.1f max %.1f\n", r, *m2.first, *m2.second);
  }
  printf("smid:mean_us ");
  for (int s = 0; s < grid; ++s) printf("%d:%.1f ", s, mean[s]);
  printf("\n");
  return 0;
}
