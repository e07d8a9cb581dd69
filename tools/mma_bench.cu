// mma_bench.cu — cycles per tile of each tcgen05 MMA group used by the fused
// kernel (issue + completion, one CTA, operands resident in smem/TMEM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/mma_bench.cu -o tools/mma_bench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace spcp::tc;

__global__ void __launch_bounds__(128) bench(int variant, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (warp == 0) {
    const uint32_t u0 = smem_u32(sm), v0 = smem_u32(sm + 32768), g0 = smem_u32(sm + 65536);
    constexpr uint32_t RB = 64;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (variant == 0 || variant == 9) {  // residual: 12 x SS M128 N64 K16
        for (int q = 0; q < 6; ++q)
          for (int ks = 0; ks < 2; ++ks)
            mma_ss_w(tm, umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                   umma_desc(v0 + q * 4096 + ks * 32, 16, 8 * RB, SW_64),
                   idesc_f16(128, 64, false, false), (q | ks) != 0);
      }
      if (variant == 1 || variant == 9) {  // GV: 12 x TS M128 N32
        for (int ks = 0; ks < 4; ++ks)
          for (int q = 0; q < 3; ++q)
            mma_ts_w(tm + 256, tm + 128 + 8 * ks + (q == 2 ? 32 : 0),
                   umma_desc(v0 + (q == 1 ? 4096 : 0) + ks * 16 * RB, 8192, 8 * RB, SW_64),
                   idesc_f16(128, 32, false, true), 1);
      }
      if (variant == 2 || variant == 9) {  // GtU: 24 x SS M64 N32 (MN-major A)
        for (int ks = 0; ks < 8; ++ks)
          for (int q = 0; q < 3; ++q)
            mma_ss_w(tm + 320, umma_desc(g0 + (q == 2 ? 16384 : 0) + 2048 * ks, 16384, 1024, SW_128),
                   umma_desc(u0 + (q == 1 ? 8192 : 0) + ks * 16 * RB, 8192, 8 * RB, SW_64),
                   idesc_f16(64, 32, true, true), 1);
      }
      if (variant == 3) {  // GtU alt: 16 x SS M128 N32, A = [gh; gl] stacked along M
        for (int ks = 0; ks < 8; ++ks)
          for (int q = 0; q < 2; ++q)
            mma_ss_w(tm + 320, umma_desc(g0 + 2048 * ks, 16384, 1024, SW_128),
                   umma_desc(u0 + (q == 1 ? 8192 : 0) + ks * 16 * RB, 8192, 8 * RB, SW_64),
                   idesc_f16(128, 32, true, true), 1);
      }
      if (variant == 4) {  // residual with N = 128 (two tiles): 12 x SS M128 N128
        for (int q = 0; q < 6; ++q)
          for (int ks = 0; ks < 2; ++ks)
            mma_ss_w(tm, umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                   umma_desc(v0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                   idesc_f16(128, 128, false, false), (q | ks) != 0);
      }
      if (variant == 5) {  // 12 x SS M128 N256
        for (int q = 0; q < 6; ++q)
          for (int ks = 0; ks < 2; ++ks)
            mma_ss_w(tm, umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                   umma_desc(v0 + ks * 32, 16, 8 * RB, SW_64),
                   idesc_f16(128, 256, false, false), (q | ks) != 0);
      }
      if (variant == 6 || variant == 7) {  // residual, interleaved over 2 / 4 accumulators
        const int nacc = variant == 6 ? 2 : 4;
        for (int q = 0; q < 6; ++q)
          for (int ks = 0; ks < 2; ++ks) {
            const int i = q * 2 + ks;
            mma_ss_w(tm + 64 * (i % nacc), umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                   umma_desc(v0 + q * 4096 + ks * 32, 16, 8 * RB, SW_64),
                   idesc_f16(128, 64, false, false), i >= nacc);
          }
      }
      if (variant == 8) {  // 48 x SS M128 N64 (4 groups) with one commit
        for (int r = 0; r < 4; ++r)
          for (int q = 0; q < 6; ++q)
            for (int ks = 0; ks < 2; ++ks)
              mma_ss_w(tm + 64 * r, umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                     umma_desc(v0 + q * 4096 + ks * 32, 16, 8 * RB, SW_64),
                     idesc_f16(128, 64, false, false), (q | ks) != 0);
      }
      mma_commit_w(&bar);
      mbar_wait(&bar, it & 1);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[variant] = (t1 - t0) / iters;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaMemset(d, 0, 16 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"residual 12x SS M128 N64", "GV 12x TS M128 N32", "GtU 24x SS M64 N32",
                         "GtU-alt 16x SS M128 N32", "residual 12x SS M128 N128",
                         "12x SS M128 N256", "res 12x, 2 accumulators", "res 12x, 4 accumulators",
                         "48x SS M128 N64 one commit", "all (res+GV+GtU)"};
  int vars[] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9};
  for (int v : vars) {
    bench<<<1, 128, 200 * 1024>>>(v, 2000, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  }
  long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int v : vars) printf("%-28s %6lld cycles per group (incl. commit+wait)\n", names[v], h[v]);
  return 0;
}
