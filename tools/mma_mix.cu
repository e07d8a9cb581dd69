// mma_mix.cu — does mixing MMA shapes / majorness / A-source in one tensor
// pipe cost more than the sum of the parts?  Tile-sized MMA sets (k = 20):
//   R  residual  6 x SS M128 N64 (K-major)          (R' = TS)
//   T  G^T U    16 x SS M64 N64 (A MN-major)
//   V  G.V       8 x SS M128 N64 (B MN-major)       (V' = TS)
// issued per iteration by 1 or 2 warps; cycles per iteration (= per tile).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/mma_mix.cu -o tools/mma_mix
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace spcp::tc;

// which: bit0 R, bit1 T, bit2 V, bit3 R as TS, bit4 V as TS
__device__ __forceinline__ void issue_set(int which, uint32_t tm, uint32_t u0, uint32_t v0, uint32_t g0) {
  constexpr uint32_t ID_RES = idesc_f16(128, 64, false, false);
  constexpr uint32_t ID_GT = idesc_f16(64, 64, true, true);
  constexpr uint32_t ID_GV = idesc_f16(128, 64, false, true);
  const uint64_t dUk = umma_desc(u0, 16, 512, SW_64), dVk = umma_desc(v0, 16, 512, SW_64);
  const uint64_t dGm = umma_desc(g0, 16384, 1024, SW_128), dUn = umma_desc(u0, 8192, 512, SW_64);
  const uint64_t dGk = umma_desc(g0, 16, 1024, SW_128), dVn = umma_desc(v0, 4096, 512, SW_64);
  if (which & 1) {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      if (which & 8)
        mma_ts(tm + 0, tm + 448 + 8 * (i & 1), dVk + 2 * (i & 1), ID_RES, 1);
      else
        mma_ss(tm + 0, dUk + 2 * (i & 1), dVk + 2 * (i & 1), ID_RES, 1);
    }
  }
  if (which & 2) {
#pragma unroll
    for (int i = 0; i < 16; ++i) mma_ss(tm + 64, dGm + 128 * (i >> 1), dUn + 64 * (i >> 1), ID_GT, 1);
  }
  if (which & 4) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (which & 16)
        mma_ts(tm + 128, tm + 384 + 8 * (i & 3), dVn + 64 * (i & 3), ID_GV, 1);
      else
        mma_ss(tm + 128, dGk + 2 * (i & 3), dVn + 64 * (i & 3), ID_GV, 1);
    }
  }
}

__global__ void __launch_bounds__(64) mix(int w0, int w1, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t u0 = smem_u32(sm), v0 = smem_u32(sm + 16384), g0 = smem_u32(sm + 32768);
  const int which = warp == 0 ? w0 : w1;
  long long t0 = 0;
  if (which) {
    for (int it = 0; it < iters + 1; ++it) {
      if (it == 1) t0 = clock64();
      if ((threadIdx.x & 31) == 0) {
        issue_set(which, tm + warp * 192, u0, v0, g0);
        mma_commit(&bar[warp]);
      }
      __syncwarp();
      mbar_wait(&bar[warp], it & 1);
    }
  }
  if ((threadIdx.x & 31) == 0) out[warp] = which ? (clock64() - t0) / iters : 0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct Case { int w0, w1; const char* name; } cases[] = {
      {1, 0, "R alone"}, {2, 0, "T alone"}, {4, 0, "V alone"}, {9, 0, "R' (TS) alone"},
      {20, 0, "V' (TS) alone"}, {7, 0, "R+T+V one warp"}, {1, 6, "R | T+V two warps"},
      {1, 1, "R | R two warps"}, {2, 2, "T | T two warps"}, {4, 4, "V | V two warps"},
      {9, 22, "R' | T+V' two warps"}, {9 + 2 + 4 + 16, 0, "R'+T+V' one warp"},
      {9, 20, "R' | V' two warps"}, {1, 4, "R | V two warps"}, {1, 2, "R | T two warps"}};
  for (auto& c : cases) {
    mix<<<1, 64, smem>>>(c.w0, c.w1, 300, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-22s %6lld %6lld cycles per iteration (warp 0, warp 1)\n", c.name, h[0], h[1]);
  }
  return 0;
}
