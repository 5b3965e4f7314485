// Microbenchmark: tcgen05.mma throughput and issue->commit latency for the decode GEMM's stage
// (M=128 weight rows x N tokens x K=64, four K=16 instructions, SS operands with 128B swizzle),
// one CTA per SM, operands resident in shared memory (no loads): is the MMA pipe a limit when a
// 16 KB weight stage arrives every ~0.37 us per SM at the HBM rate?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/mma_probe.cu -o scripts/mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2404_18322_b200/csrc/ptx.cuh"

using namespace bx;

template <int N, int NACC = 1>
__global__ void __launch_bounds__(128, 1) mma_loop(int stages, int wait_each, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                 // 16 KB
  uint8_t* sB = sm + 16384;         // N*128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + N * 128);
  uint32_t* holder = reinterpret_cast<uint32_t*>(bar + 2);
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<256>(holder);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N);
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    uint32_t ph = 0;
    unsigned long long lat = 0;
    const unsigned long long t0 = gtimer();
    for (int s = 0; s < stages; ++s) {
      const unsigned long long ti = gtimer();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // NACC accumulators side by side in TMEM, consecutive instructions alternating
        const int acc = (s * 4 + k) % NACC;
        umma_bf16(tmem + acc * N, make_sdesc_k128(a + k * 32), make_sdesc_k128(b + k * 32), idesc,
                  (s * 4 + k >= NACC) ? 1u : 0u);
      }
      if (wait_each || s == stages - 1) umma_commit(bar);
      if (wait_each) {
        mbar_wait(bar, ph);
        ph ^= 1u;
        lat += gtimer() - ti;
      }
    }
    if (!wait_each) mbar_wait(bar, 0);  // one commit after the last stage (MMAs run in order)
    const unsigned long long t1 = gtimer();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = wait_each ? lat / stages : 0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<256>(tmem);
}

template <int N, int NACC = 1>
void run(int sms, unsigned long long* d, unsigned long long* h) {
  const int smem = 16384 + N * 128 + 64 + 1024;
  cudaFuncSetAttribute(mma_loop<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("accumulators %d\n", NACC);
  for (int wait_each = 0; wait_each < 2; ++wait_each) {
    const int stages = 2000;
    mma_loop<N, NACC><<<sms, 128, smem>>>(stages, wait_each, d);
    mma_loop<N, NACC><<<sms, 128, smem>>>(stages, wait_each, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sms * 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double tot = 0, lat = 0;
    for (int i = 0; i < sms; ++i) {
      tot += h[2 * i];
      lat += h[2 * i + 1];
    }
    tot /= sms;
    lat /= sms;
    printf("N=%3d %s: %.1f ns per stage (4 x K=16 MMAs%s)%s\n", N,
           wait_each ? "commit-waited" : "pipelined   ", tot / stages,
           wait_each ? ", issue->commit latency" : "",
           cudaGetErrorString(cudaGetLastError()));
    if (wait_each) printf("       latency per stage %.1f ns\n", lat);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *d, *h = new unsigned long long[2 * sms];
  cudaMalloc(&d, 2 * sms * sizeof(unsigned long long));
  run<16>(sms, d, h);
  run<64>(sms, d, h);
  run<128>(sms, d, h);
  run<256>(sms, d, h);
  run<16, 2>(sms, d, h);
  run<64, 2>(sms, d, h);
  run<64, 4>(sms, d, h);
  run<16, 4>(sms, d, h);
  return 0;
}
