// mma_commit.cu — cost of tcgen05.commit inside an MMA stream: one warp
// issues tiles of 20 SS M128 N64 MMAs with C commits per tile (to mbarriers
// nobody waits on), straight-line code; cycles per tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/mma_commit.cu -o tools/mma_commit
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace spcp::tc;

template <int C, int NW>
__global__ void __launch_bounds__(640) commit_cost(int iters, int poll, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[4], dummy[8], never;
  __shared__ volatile int stop;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&dummy[i], 1 << 19);
    mbar_init(&never, 1);
    stop = 0;
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (warp < NW && (threadIdx.x & 31) == 0) {
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
    constexpr uint32_t ID = idesc_f16(128, 64, false, false);
    const uint64_t da = umma_desc(a0, 16, 1024, SW_128);
    const uint64_t db = umma_desc(b0, 16, 1024, SW_128);
    const uint32_t d = tm + warp * 128;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 20; ++i) {
        mma_ss(d + (i & 1) * 64, da + 2 * (i & 3), db + 2 * (i & 3), ID, 1);
        if (C > 0 && (i % (20 / (C > 0 ? C : 1))) == (20 / (C > 0 ? C : 1)) - 1)
          mma_commit(&dummy[(i / 4) & 7]);
      }
    }
    mma_commit(&bar[warp]);
    mbar_wait(&bar[warp], 0);
    out[warp] = (clock64() - t0) / iters;
    stop = 1;
  } else if (warp >= 4 && poll) {
    // warps polling an mbarrier phase that never completes (as epilogue warps
    // waiting on the tensor pipe do), with or without the suspend-time hint
    uint32_t ok = 0;
    while (!stop) {
      if (poll == 1)
        asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\nselp.b32 %0, 1, 0, P1;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(&never)), "r"(0u), "r"(0x989680u) : "memory");
      else
        asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.b32 %0, 1, 0, P1;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(&never)), "r"(0u) : "memory");
    }
    if (ok == 77) out[7] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

template <int C, int NW>
void run(long long* d, int poll = 0) {
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(commit_cost<C, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  commit_cost<C, NW><<<1, poll ? 640 : 128, smem>>>(200, poll, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < NW; ++w) mx = h[w] > mx ? h[w] : mx;
  printf("poll=%d warps=%d commits/tile=%d  %6lld cycles per 20-MMA tile per warp (%5.1f per MMA overall)\n", poll, NW, C,
         mx, mx / (20.0 * NW));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  run<0, 1>(d); run<1, 1>(d); run<2, 1>(d); run<4, 1>(d); run<5, 1>(d); run<10, 1>(d);
  run<0, 2>(d); run<2, 2>(d); run<5, 2>(d);
  run<0, 1>(d, 1); run<0, 1>(d, 2); run<0, 2>(d, 1); run<0, 2>(d, 2);
  return 0;
}
