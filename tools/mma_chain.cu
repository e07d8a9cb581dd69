// mma_chain.cu — dependent-accumulator chains vs interleaved independent
// accumulators, in ONE issue stream (one lane), throughput over many
// iterations (single wait at the end): does the tensor pipe overlap MMAs into
// different accumulators, and what does a chain cost per MMA?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/mma_chain.cu -o tools/mma_chain
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace spcp::tc;

template <int M, int N, int KIND, int NACC>
__global__ void __launch_bounds__(32) chain(int iters, long long* out) {
  // KIND 0: SS K-major, 1: TS, 2: SS A MN-major
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 32) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncwarp();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
    constexpr uint32_t ID = idesc_f16(M, N, KIND == 2, false);
    const uint64_t da = KIND == 2 ? umma_desc(a0, 16384, 1024, SW_128) : umma_desc(a0, 16, 1024, SW_128);
    const uint64_t db = umma_desc(b0, 16, 1024, SW_128);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        const uint32_t d = tm + (i % NACC) * 64;
        if (KIND == 1)
          mma_ts(d, tm + 448 + 8 * (i & 1), db + 2 * (i & 1), ID, 1);
        else
          mma_ss(d, da + (KIND == 2 ? 128 : 2) * (i & 1), db + 2 * (i & 1), ID, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = (clock64() - t0) / iters;
  }
  tc_fence_before();
  __syncwarp();
  tmem_dealloc(tm, 512);
}

template <int M, int N, int KIND, int NACC>
void run(const char* name, long long* d) {
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(chain<M, N, KIND, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  chain<M, N, KIND, NACC><<<1, 32, smem>>>(400, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  long long h;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-24s nacc=%d  %6.1f cycles per MMA (floor %d)\n", name, NACC, h / 24.0,
         (M < 128 ? 128 : M) * N / 256);
}

#define RUN4(M, N, K, name) run<M, N, K, 1>(name, d); run<M, N, K, 2>(name, d); \
  run<M, N, K, 3>(name, d); run<M, N, K, 4>(name, d);

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  RUN4(128, 64, 0, "SS M128 N64");
  RUN4(128, 64, 1, "TS M128 N64");
  RUN4(128, 32, 1, "TS M128 N32");
  RUN4(64, 64, 2, "SS M64 N64 A-MN");
  RUN4(128, 64, 2, "SS M128 N64 A-MN");
  return 0;
}
