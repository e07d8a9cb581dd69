// mma_cost.cu — tensor-pipe cost of one 128 x 64 tile's MMA set (k = 20,
// KP16 = 32) for the candidate operand placements of the fused kernel, issued
// back to back from one thread (throughput, not latency), with and without
// background shared-memory traffic from 16 LSU warps (the epilogue's X reads
// and G image writes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/mma_cost.cu -o tools/mma_cost
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace spcp::tc;

// part bits: 1 residual, 2 GT, 4 GV.  mode: 0 = v3 (all SS), 1 = residual/GV A
// in TMEM (TS), GT SS M64; 2 = TS + GT stacked M128; 3 = TS + GT as U^T G (TS, M64 N128)
__global__ void __launch_bounds__(544) cost(int mode, int parts, int iters, int bg, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    stop = 0;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t u0 = smem_u32(sm), v0 = smem_u32(sm + 16384), g0 = smem_u32(sm + 32768);
  if (warp == 0) {
    if (threadIdx.x == 0) {
      const uint32_t ID_RES = idesc_f16(128, 64, false, false);
      const uint32_t ID_GT64 = idesc_f16(64, 64, true, true);
      const uint32_t ID_GT128 = idesc_f16(128, 64, true, true);
      const uint32_t ID_GTT = idesc_f16(64, 128, false, true);
      const uint32_t ID_GV = idesc_f16(128, 64, false, true);
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        if (parts & 1) {
          for (int q = 0; q < 3; ++q)
            for (int ks = 0; ks < 2; ++ks) {
              const int sa = q == 2, sb = q == 1;
              const uint64_t db = umma_desc(v0 + sb * 4096 + ks * 32, 16, 512, SW_64);
              if (mode == 0)
                mma_ss(tm + 0, umma_desc(u0 + sa * 8192 + ks * 32, 16, 512, SW_64), db, ID_RES, q | ks);
              else
                mma_ts(tm + 0, tm + 256 + sa * 16 + ks * 8, db, ID_RES, q | ks);
            }
        }
        if (parts & 2) {
          for (int ks = 0; ks < 8; ++ks) {
            const uint64_t dbu = umma_desc(u0 + ks * 1024, 8192, 512, SW_64);
            if (mode <= 1) {
              for (int s = 0; s < 2; ++s)
                mma_ss(tm + 128, umma_desc(g0 + s * 16384 + 2048 * ks, 16384, 1024, SW_128), dbu,
                       ID_GT64, 1);
            } else if (mode == 2) {
              mma_ss(tm + 128, umma_desc(g0 + 2048 * ks, 16384, 1024, SW_128), dbu, ID_GT128, 1);
            } else {
              mma_ts(tm + 128, tm + 384 + ks * 8, umma_desc(g0 + 2048 * ks, 16384, 1024, SW_128),
                     ID_GTT, 1);
            }
          }
        }
        if (parts & 4) {
          for (int ks = 0; ks < 4; ++ks)
            for (int s = 0; s < 2; ++s) {
              const uint64_t dbv = umma_desc(v0 + ks * 1024, 4096, 512, SW_64);
              if (mode == 0)
                mma_ss(tm + 64, umma_desc(g0 + s * 16384 + 32 * ks, 16, 1024, SW_128), dbv, ID_GV, 1);
              else
                mma_ts(tm + 64, tm + 320 + s * 32 + ks * 8, dbv, ID_GV, 1);
            }
        }
        mma_commit(&bar);
      }
      mbar_wait(&bar, (iters - 1) & 1);
      long long t1 = clock64();
      out[0] = (t1 - t0) / iters;
      stop = 1;
    }
  } else if (bg) {
    // background LSU traffic: LDS.128 + STS.128 over a private 64 KB region
    const int t = threadIdx.x - 32;
    unsigned char* reg = sm + 98304 + (t % 256) * 16;
    float4 acc = make_float4(0, 0, 0, 0);
    int n = 0;
    while (!*(volatile int*)&stop) {
      for (int r = 0; r < 16; ++r) {
        float4 v = lds128(reg + r * 4096);
        acc.x += v.x;
        *reinterpret_cast<float4*>(reg + ((r + 8) & 15) * 4096) = make_float4(acc.x, v.y, v.z, acc.w);
      }
      ++n;
    }
    if (acc.x == 12345.f) out[1] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  const int smem = 98304 + 65536 + 1024;
  cudaFuncSetAttribute(cost, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* mn[4] = {"v3 all-SS", "TS res/GV, GT SS M64", "TS res/GV, GT stacked M128", "TS res/GV, GT=U^T G TS"};
  const char* pn[8] = {"", "residual", "GT", "res+GT", "GV", "res+GV", "GT+GV", "all"};
  for (int bg = 0; bg < 2; ++bg)
    for (int mode = 0; mode < 4; ++mode)
      for (int parts : {1, 2, 4, 7}) {
        if (mode > 0 && parts == 1 && mode != 1) continue;
        long long h[2] = {0, 0};
        cost<<<1, bg ? 544 : 32, smem>>>(mode, parts, 2000, bg, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("bg=%d %-28s %-9s %6lld cycles per tile\n", bg, mn[mode], pn[parts], h[0]);
      }
  return 0;
}
