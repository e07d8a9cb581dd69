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

__global__ void __launch_bounds__(640) streams(int mode, int iters, int bg, const float* gsrc, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2], dummy[8], ring_full[3];
  __shared__ volatile int stop;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&dummy[i], 1 << 19);
    for (int i = 0; i < 3; ++i) mbar_init(&ring_full[i], 1);
    stop = 0;
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
  if (warp < 2) {
    __syncwarp();
    named_bar_sync(1, 64);
    if (threadIdx.x == 0) stop = 1;
  } else if (warp == 2 && (bg & 1)) {
    // bulk copies global -> smem (HBM stream like the X producer): 3 x 32 KB ring
    if ((threadIdx.x & 31) == 0) {
      size_t off = size_t(blockIdx.x) * 32768;
      int i = 0;
      for (; !stop; ++i) {
        const int s2 = i % 3;
        if (i >= 3) mbar_wait(&ring_full[s2], ((i / 3) - 1) & 1);
        mbar_arrive_expect_tx(&ring_full[s2], 32768);
        bulk_load(sm + 65536 + s2 * 32768, gsrc + off / 4, 32768, &ring_full[s2]);
        off = (off + 148 * 32768) % (size_t(1) << 30);
      }
      for (int j = i - 3 < 0 ? 0 : i - 3; j < i; ++j) mbar_wait(&ring_full[j % 3], (j / 3) & 1);
    }
  } else if (warp >= 4 && (bg & 2)) {
    // epilogue-like TMEM reads (tcgen05.ld 32x32b.x16, columns 448..511)
    uint32_t acc = 0;
    const uint32_t la = uint32_t(32 * (warp & 3)) << 16;
    while (!stop) {
      uint32_t r[16];
      tmem_ld16(tm + la + 448 + 16 * (warp & 3), r);
      tmem_wait_ld();
      acc += r[0] ^ r[15];
    }
    if (acc == 12345) out[7] = acc;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  const int smem = 64 * 1024 + 3 * 32768 + 1024;
  cudaFuncSetAttribute(streams, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float* gsrc;
  cudaMalloc(&gsrc, size_t(1) << 30);
  cudaMemset(gsrc, 0, size_t(1) << 30);
  const char* nm[4] = {"residual stream alone", "reduction stream alone", "both streams (2 warps)",
                       "one warp, tile order"};
  for (int bg = 0; bg < 4; ++bg)
  for (int mode = 2; mode < 4; ++mode) {
    cudaMemset(d, 0, 64);
    streams<<<148, 640, smem>>>(mode, 300, bg, gsrc, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("bg=%d (1 bulk HBM, 2 tcgen05.ld) %-26s warp0 %6lld  warp1 %6lld cycles per tile\n", bg, nm[mode], h[0], h[1]);
  }
  return 0;
}
