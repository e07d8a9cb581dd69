// mma_ops.cu — throughput (cycles per MMA, no waits inside the stream) of the
// exact operand configurations of the fused kernel, issued by 1 or 4 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/mma_ops.cu -o tools/mma_ops
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace spcp::tc;

struct Op {
  const char* name;
  int M, N;
  bool amn, bmn;
  uint32_t a_off, a_lbo, a_sbo, a_sw;  // A (smem) descriptor; a_sw = 99: A from TMEM
  uint32_t b_off, b_lbo, b_sbo, b_sw;
  uint32_t a_step, b_step;  // per-MMA start-address step (bytes), alternating 2 values
};

__global__ void __launch_bounds__(128) ops(Op op, int nw, int iters, int rnd, int cmt, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[4], dummy[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t(i) * 2654435761u) ^ (uint32_t(blockIdx.x) * 40503u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    // random fp16 pairs with exponents in [-8, 7] (finite, no overflow in fp32 sums)
    const uint32_t r = (h & 0x83ff83ffu) | 0x20002000u | ((h >> 3) & 0x1c001c00u);
    reinterpret_cast<uint32_t*>(sm)[i] = rnd ? r : 0x3c003c00u;
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&dummy[i], 1 << 20);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (warp < nw && (threadIdx.x & 31) == 0) {
    const uint32_t base = smem_u32(sm);
    const uint32_t id = idesc_f16(op.M, op.N, op.amn, op.bmn);
    const uint64_t da0 = umma_desc(base + op.a_off, op.a_lbo, op.a_sbo, op.a_sw == 99 ? 0 : op.a_sw);
    const uint64_t da1 = umma_desc(base + op.a_off + op.a_step, op.a_lbo, op.a_sbo, op.a_sw == 99 ? 0 : op.a_sw);
    const uint64_t db0 = umma_desc(base + op.b_off, op.b_lbo, op.b_sbo, op.b_sw);
    const uint64_t db1 = umma_desc(base + op.b_off + op.b_step, op.b_lbo, op.b_sbo, op.b_sw);
    const uint32_t d = tm + warp * 64;
    const uint32_t ta = tm + 256 + warp * 64;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (op.a_sw == 99)
          mma_ts(d, ta + 8 * (i & 1), (i & 1) ? db1 : db0, id, 1);
        else
          mma_ss(d, (i & 1) ? da1 : da0, (i & 1) ? db1 : db0, id, 1);
        if (cmt && (i % cmt) == cmt - 1) mma_commit(&dummy[warp]);
      }
    }
    mma_commit(&bar[warp]);
    mbar_wait(&bar[warp], 0);
    if (blockIdx.x == 0) out[warp] = (clock64() - t0) / iters;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  const int smem = 128 * 1024 + 1024;
  cudaFuncSetAttribute(ops, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // smem map: U image @0 (16 KB), V image @16K (8 KB), G images @32K (2 x 16 KB)
  Op list[] = {
      // legacy (KP16 = 32: RB = 64, SW64, two splits)
      {"res legacy SS SW64 K/K", 128, 64, false, false, 0, 16, 512, SW_64, 16384, 16, 512, SW_64, 32, 32},
      {"GT legacy SS M64 A-MN SW128 B-MN SW64x2", 64, 64, true, true, 32768, 16384, 1024, SW_128, 0, 8192, 512, SW_64, 2048, 1024},
      {"GV legacy SS A-K SW128 B-MN SW64x2", 128, 64, false, true, 32768, 16, 1024, SW_128, 16384, 4096, 512, SW_64, 32, 1024},
      // KC (SEG = 20: RB = 128, SW128, one image)
      {"res KC SS SW128 K/K", 128, 64, false, false, 0, 16, 1024, SW_128, 16384, 16, 1024, SW_128, 32, 32},
      {"GT KC SS M128 A-MN SW128 B-MN SW128", 128, 64, true, true, 32768, 16384, 1024, SW_128, 0, 8192, 1024, SW_128, 2048, 2048},
      {"GV KC SS A-K SW128 B-MN SW128", 128, 64, false, true, 32768, 16, 1024, SW_128, 16384, 8192, 1024, SW_128, 32, 2048},
      // TS candidates
      {"res KC TS B-K SW128", 128, 64, false, false, 0, 16, 1024, 99, 16384, 16, 1024, SW_128, 0, 32},
      {"GV KC TS B-MN SW128", 128, 64, false, true, 0, 16, 1024, 99, 16384, 8192, 1024, SW_128, 0, 2048},
      {"GT KC SS M128 N48", 128, 48, true, true, 32768, 16384, 1024, SW_128, 0, 8192, 1024, SW_128, 2048, 2048},
      {"GV KC SS N32 B-MN SW128", 128, 32, false, true, 32768, 16, 1024, SW_128, 16384, 8192, 1024, SW_128, 32, 2048},
  };
  for (int cmt : {0, 8, 4, 2, 1})
  for (int li = 0; li < 8; li += (cmt ? 3 : 1))
    for (int nw : {1, 4}) {
      auto& op = list[li];
      const int cfg = 1;
      ops<<<1, 128, smem>>>(op, nw, 100, 1, cmt, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: error %s\n", op.name, cudaGetErrorString(e)); return 1; }
      long long h[4];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
      printf("%-42s commit/%d warps=%d %6.1f cycles per MMA\n", op.name, cmt, nw, mx / (8.0 * nw));
    }
  return 0;
}
