// mma_streams.cu — the fused kernel's two MMA streams (KC layout, SEG = 20)
// replayed without any data dependency: warp 0 issues the residual (4 SS MMAs
// + commit per tile), warp 1 the reductions (8 G^T U + 8 G.V + commits per
// tile).  Cycles per tile per stream, alone and together; plus a variant in
// which one warp issues everything in tile order.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/mma_streams.cu -o tools/mma_streams
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"
#include <utility>

using namespace spcp::tc;

template <int N, typename F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void sfor(F&& f) {
  sfor_impl<N>(f, std::make_integer_sequence<int, N>{});
}

// smem: U image @0 (16 KB, RB 128), V image @16K (8 KB), G images @32K (2 x 16 KB)
__device__ __forceinline__ void res_tile(uint32_t tm, uint32_t base, int t, uint64_t* bar) {
  constexpr uint32_t ID = idesc_f16(128, 64, false, false);
  const uint64_t da = umma_desc(base, 16, 1024, SW_128), db = umma_desc(base + 16384, 16, 1024, SW_128);
  const uint32_t dt = tm + (t & 1) * 64;
  sfor<4>([&](auto I) { mma_ss_1<(I * 2), (I * 2)>(dt, da, db, ID, I != 0); });
  mma_commit(bar);
}
__device__ __forceinline__ void red_tile(uint32_t tm, uint32_t base, int t, uint64_t* bar) {
  constexpr uint32_t ID_GT = idesc_f16(128, 64, true, true);
  constexpr uint32_t ID_GV = idesc_f16(128, 64, false, true);
  const uint64_t dGm = umma_desc(base + 32768, 16384, 1024, SW_128);
  const uint64_t dUn = umma_desc(base, 8192, 1024, SW_128);
  const uint64_t dGk = umma_desc(base + 32768, 16, 1024, SW_128);
  const uint64_t dVn = umma_desc(base + 16384, 8192, 1024, SW_128);
  const uint32_t gt = tm + 256 + (t & 3) * 64, gv = tm + 128 + 0;
  sfor<8>([&](auto I) { mma_ss_1<((2048 * I) >> 4), ((I * 16 * 128) >> 4)>(gt, dGm, dUn, ID_GT, I > 0); });
  mma_commit(bar);
  sfor<4>([&](auto I) {
    mma_ss_1<((32 * I) >> 4), ((I * 16 * 128) >> 4)>(gv, dGk, dVn, ID_GV, 1);
    mma_ss_1<(((32 * I) >> 4) + (16384 >> 4)), ((I * 16 * 128) >> 4)>(gv, dGk, dVn, ID_GV, 1);
  });
  mma_commit(bar + 1);
  mma_commit(bar + 2);
}

__global__ void __launch_bounds__(64) streams(int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2], dummy[8];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&dummy[i], 1 << 19);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase, base = smem_u32(sm);
  // mode 0: residual only (warp 0); 1: reductions only (warp 1); 2: both warps; 3: one warp, tile order
  const bool active = (mode == 0 && warp == 0) || (mode == 1 && warp == 1) || mode == 2 || (mode == 3 && warp == 0);
  if (active && (threadIdx.x & 31) == 0) {
    long long t0 = clock64();
    for (int t = 0; t < iters; ++t) {
      if (mode == 3) {
        res_tile(tm, base, t, &dummy[0]);
        red_tile(tm, base, t, &dummy[2]);
      } else if (warp == 0) {
        res_tile(tm, base, t, &dummy[0]);
      } else {
        red_tile(tm, base, t, &dummy[2]);
      }
    }
    mma_commit(&bar[warp]);
    mbar_wait(&bar[warp], 0);
    out[warp] = (clock64() - t0) / iters;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(streams, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* nm[4] = {"residual stream alone", "reduction stream alone", "both streams (2 warps)",
                       "one warp, tile order"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(d, 0, 64);
    streams<<<1, 64, smem>>>(mode, 300, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-26s warp0 %6lld  warp1 %6lld cycles per tile\n", nm[mode], h[0], h[1]);
  }
  return 0;
}
