// mma_issue.cu — throughput of a stream of small tcgen05 MMAs when issue is
// not the limit (4 issuing warps, each into its own accumulator), per operand
// placement, with and without background LSU shared-memory traffic (16 warps
// of LDS.128 + STS.128, like the fused kernel's epilogue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/mma_issue.cu -o tools/mma_issue
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace spcp::tc;

template <int M, int N, bool TS, bool AMN>
__global__ void __launch_bounds__(640) issue(int nw, int iters, int bg, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  __shared__ int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
    stop = 0;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  long long t0 = 0;
  if (warp < 4) {
    if (warp < nw) {
      const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
      constexpr uint32_t ID = idesc_f16(M, N, AMN, false);
      const uint64_t da = AMN ? umma_desc(a0, 16384, 1024, SW_128) : umma_desc(a0, 16, 1024, SW_128);
      const uint64_t db = umma_desc(b0, 16, 1024, SW_128);
      const uint32_t d = tm + warp * (N <= 64 ? 64 : 96);
      const uint32_t ta = tm + 384 + warp * 16;
      for (int it = 0; it < iters + 1; ++it) {
        if (it == 1) t0 = clock64();
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
          for (int i = 0; i < 24; ++i) {
            if (TS)
              mma_ts(d, ta + 8 * (i & 1), db + 2 * (i & 1), ID, 1);
            else
              mma_ss(d, da + (AMN ? 128 : 2) * (i & 1), db + 2 * (i & 1), ID, 1);
          }
          mma_commit(&bar[warp]);
        }
        __syncwarp();
        mbar_wait(&bar[warp], it & 1);
      }
      if ((threadIdx.x & 31) == 0) out[warp] = (clock64() - t0) / iters;
    }
    __syncwarp();
    if (threadIdx.x == 0) {
      // wait for the other issuers by polling their outputs being set via a barrier-free spin
    }
  } else if (bg) {
    const int t = threadIdx.x - 128;
    unsigned char* reg = sm + 65536 + (t % 256) * 16;
    float4 acc = make_float4(0, 0, 0, 0);
    int n = 0;
    while (!*(volatile int*)&stop) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        float4 v = lds128(reg + r * 4096);
        acc.x += v.x;
        *reinterpret_cast<float4*>(reg + ((r + 8) & 15) * 4096) = make_float4(acc.x, v.y, v.z, acc.w);
      }
      ++n;
    }
    if (acc.x == 12345.f) out[5] = n;
    out[4 + (t == 0)] = n;
  }
  if (warp < 4) {
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) *(volatile int*)&stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

template <int M, int N, bool TS, bool AMN>
void run(const char* name, long long* d) {
  const int smem = 64 * 1024 + 65536 + 1024;
  cudaFuncSetAttribute(issue<M, N, TS, AMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int bg = 0; bg < 2; ++bg) {
    const int nw = 4;
    issue<M, N, TS, AMN><<<1, 640, smem>>>(nw, 200, bg, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
    long long h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
    printf("%-30s bg=%d  %6.1f cycles per MMA (floor %d)\n", name, bg, mx / (24.0 * nw),
           (M < 128 ? 128 : M) * N / 256);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  run<128, 64, false, false>("SS M128 N64", d);
  run<128, 64, true, false>("TS M128 N64", d);
  run<128, 32, true, false>("TS M128 N32", d);
  run<128, 96, true, false>("TS M128 N96", d);
  run<128, 32, false, false>("SS M128 N32", d);
  run<64, 64, false, true>("SS M64 N64 (A MN-major)", d);
  run<128, 64, false, true>("SS M128 N64 (A MN-major)", d);
  run<64, 96, true, false>("TS M64 N96", d);
  run<128, 96, false, false>("SS M128 N96", d);
  return 0;
}
