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
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
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
      if (variant == 10 || variant == 11) {  // residual TS: A = U from TMEM, B = V (6 or 3 products)
        const int nq = variant == 10 ? 6 : 3;
        for (int q = 0; q < nq; ++q)
          for (int ks = 0; ks < 2; ++ks)
            mma_ts_w(tm, tm + 448 + 16 * (q % 3) + 8 * ks,
                     umma_desc(v0 + q * 4096 + ks * 32, 16, 8 * RB, SW_64),
                     idesc_f16(128, 64, false, false), (q | ks) != 0);
      }
      if (variant == 12) {  // GtU stacked [gh; gl] M128, B = [uh | um] N64
        for (int ks = 0; ks < 8; ++ks)
          mma_ss_w(tm + 320, umma_desc(g0 + 2048 * ks, 16384, 1024, SW_128),
                   umma_desc(u0 + ks * 16 * RB, 8192, 8 * RB, SW_64),
                   idesc_f16(128, 64, true, true), 1);
      }
      if (variant == 13) {  // residual 3 products SS
        for (int q = 0; q < 3; ++q)
          for (int ks = 0; ks < 2; ++ks)
            mma_ss_w(tm, umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                   umma_desc(v0 + q * 4096 + ks * 32, 16, 8 * RB, SW_64),
                   idesc_f16(128, 64, false, false), (q | ks) != 0);
      }
      if (variant == 14 || variant == 15 || variant == 16) {  // the v2 per-tile set
        // residual: 3 products x 2 ks, SS M128 N64 (KP16 = 32, SW64)
        if (variant != 16)
          for (int q = 0; q < 3; ++q)
            for (int ks = 0; ks < 2; ++ks)
              mma_ss_w(tm, umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                       umma_desc(v0 + q * 4096 + ks * 32, 16, 8 * RB, SW_64),
                       idesc_f16(128, 64, false, false), (q | ks) != 0);
        // GtU: 16 x SS M64 N64 (B = [uh|um])
        if (variant != 15)
          for (int ks = 0; ks < 8; ++ks)
            for (int q = 0; q < 2; ++q)
              mma_ss_w(tm + 384, umma_desc(g0 + q * 16384 + 2048 * ks, 16384, 1024, SW_128),
                       umma_desc(u0 + ks * 16 * RB, 8192, 8 * RB, SW_64),
                       idesc_f16(64, 64, true, true), 1);
        // GV: 8 x TS M128 N64 (B = [vh|vm])
        if (variant != 16)
          for (int ks = 0; ks < 4; ++ks)
            for (int q = 0; q < 2; ++q)
              mma_ts_w(tm + 256, tm + 128 + 32 * q + 8 * ks,
                       umma_desc(v0 + ks * 16 * RB, 4096, 8 * RB, SW_64),
                       idesc_f16(128, 64, false, true), 1);
      }
      if (variant >= 17 && variant <= 19) {  // v2 tile with the kernel's intermediate commits
        __shared__ uint64_t xb[8];
        if (it == 0 && lane == 0)
          for (int i = 0; i < 8; ++i) mbar_init(&xb[i], 1);
        __syncwarp();
        for (int q = 0; q < 3; ++q)
          for (int ks = 0; ks < 2; ++ks)
            mma_ss_w(tm, umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                     umma_desc(v0 + q * 4096 + ks * 32, 16, 8 * RB, SW_64),
                     idesc_f16(128, 64, false, false), (q | ks) != 0);
        if (variant >= 18) mma_commit_w(&xb[0]);
        for (int ks = 0; ks < 8; ++ks)
          for (int q = 0; q < 2; ++q)
            mma_ss_w(tm + 384, umma_desc(g0 + q * 16384 + 2048 * ks, 16384, 1024, SW_128),
                     umma_desc(u0 + ks * 16 * RB, 8192, 8 * RB, SW_64),
                     idesc_f16(64, 64, true, true), 1);
        if (variant >= 18) { mma_commit_w(&xb[1]); mma_commit_w(&xb[2]); }
        for (int ks = 0; ks < 4; ++ks)
          for (int q = 0; q < 2; ++q)
            mma_ts_w(tm + 256, tm + 128 + 32 * q + 8 * ks,
                     umma_desc(v0 + ks * 16 * RB, 4096, 8 * RB, SW_64),
                     idesc_f16(128, 64, false, true), 1);
        if (variant >= 18) { mma_commit_w(&xb[3]); mma_commit_w(&xb[4]); }
        if (variant == 19) { mma_commit_w(&xb[5]); mma_commit_w(&xb[6]); }
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


// v2 tile MMA set on warp 0 while warps 1..NW do background traffic:
// mode 0 none, 1 LDS.128 stream, 2 STS.128 stream, 3 LDS+STS, 4 tcgen05.ld (32 cols),
// 5 tcgen05.st (32 cols), 6 ld+st TMEM
__device__ const unsigned char* g_src;
__global__ void __launch_bounds__(512) bench_bg(int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
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
      for (int q = 0; q < 3; ++q)
        for (int ks = 0; ks < 2; ++ks)
          mma_ss_w(tm, umma_desc(u0 + q * 8192 + ks * 32, 16, 8 * RB, SW_64),
                   umma_desc(v0 + q * 4096 + ks * 32, 16, 8 * RB, SW_64),
                   idesc_f16(128, 64, false, false), (q | ks) != 0);
      for (int ks = 0; ks < 8; ++ks)
        for (int q = 0; q < 2; ++q)
          mma_ss_w(tm + 384, umma_desc(g0 + q * 16384 + 2048 * ks, 16384, 1024, SW_128),
                   umma_desc(u0 + ks * 16 * RB, 8192, 8 * RB, SW_64),
                   idesc_f16(64, 64, true, true), 1);
      for (int ks = 0; ks < 4; ++ks)
        for (int q = 0; q < 2; ++q)
          mma_ts_w(tm + 256, tm + 128 + 32 * q + 8 * ks,
                   umma_desc(v0 + ks * 16 * RB, 4096, 8 * RB, SW_64),
                   idesc_f16(128, 64, false, true), 1);
      mma_commit_w(&bar);
      mbar_wait(&bar, it & 1);
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = (t1 - t0) / iters; stop = 1; }
  } else {
    // background: region 128 KB .. 200 KB of smem; TMEM columns 448..479
    unsigned char* b = sm + 131072;
    uint4 acc = make_uint4(0, 0, 0, 0);
    long long n = 0;
    const uint32_t lane_addr = uint32_t(32 * (warp & 3)) << 16;
    while (!stop) {
      for (int r = 0; r < 16; ++r) {
        const uint32_t o = ((threadIdx.x * 16) + r * 8192) % 65536;
        if (mode == 1 || mode == 3) {
          uint4 v;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(b + o)));
          acc.x ^= v.x; acc.y += v.y;
        }
        if (mode == 2 || mode == 3)
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(smem_u32(b + o)), "r"(acc.x), "r"(acc.y), "r"(acc.z), "r"(acc.w) : "memory");
        if (mode == 4 || mode == 6) {
          uint32_t v[16];
          tmem_ldn<16>(tm + lane_addr + 448, v);
          tmem_wait_ld();
          acc.x ^= v[0] + v[15];
        }
        if (mode == 5 || mode == 6) {
          uint32_t v[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = acc.x + c;
          tmem_st16(tm + lane_addr + 448 + 16 * ((warp >> 2) & 1), v);
          tmem_wait_st();
        }
        if (mode == 8) {  // STS + proxy fence (the epilogue's G-image handoff)
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(smem_u32(b + o)), "r"(acc.x), "r"(acc.y), "r"(acc.z), "r"(acc.w) : "memory");
          fence_proxy_async_smem();
        }
        if (mode == 9) {  // tcgen05 fences only
          tc_fence_before();
          tc_fence_after();
        }
        if (mode == 10) {  // mbarrier polling (never completes)
          __shared__ uint64_t pb;
          if (threadIdx.x == 32 && n == 0) mbar_init(&pb, 1000);
          uint32_t ok;
          asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.b32 %0,1,0,P;\n}\n" : "=r"(ok) : "r"(smem_u32(&pb)) : "memory");
          acc.x += ok;
        }
        if (mode == 11 && (threadIdx.x & 31) == 0 && warp == 1) {  // TMA-engine bulk copies from HBM
          __shared__ uint64_t cb;
          if (n == 0) { mbar_init(&cb, 1); fence_barrier_init(); }
          mbar_arrive_expect_tx(&cb, 32768);
          bulk_load(sm + 131072 + (n & 1) * 32768, g_src + ((n * 32768) % (512u << 20)), 32768, &cb);
          mbar_wait(&cb, n & 1);
        }
        if (mode == 12 && (threadIdx.x & 31) == 0 && warp <= 4) {  // TMA bulk writes, 2 in flight/warp
          __shared__ uint64_t cb2[8];
          const int w = warp - 1;
          if (n == 0) { mbar_init(&cb2[2 * w], 1); mbar_init(&cb2[2 * w + 1], 1); fence_barrier_init(); }
          const int slot = n & 1;
          if (n >= 2) mbar_wait(&cb2[2 * w + slot], ((n >> 1) - 1) & 1);
          mbar_arrive_expect_tx(&cb2[2 * w + slot], 8192);
          bulk_load(sm + 131072 + (w * 2 + slot) * 8192, g_src + ((n * 8192 + w * 65536) % (2u << 20)), 8192,
                    &cb2[2 * w + slot]);
        }
        if (mode == 7) {
          float f0 = __uint_as_float(acc.x), f1 = f0 + 1.f, f2 = f0 + 2.f, f3 = f0 + 3.f;
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            f0 = fmaf(f0, 1.0001f, f1); f1 = fmaf(f1, 0.9999f, f2);
            f2 = fmaf(f2, 1.0001f, f3); f3 = fmaf(f3, 0.9999f, f0);
          }
          acc.x = __float_as_uint(f0 + f1 + f2 + f3);
        }
        ++n;
      }
    }
    if (acc.x == 0x1234567u) out[15] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 32 * sizeof(long long));
  cudaMemset(d, 0, 32 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"residual 12x SS M128 N64", "GV 12x TS M128 N32", "GtU 24x SS M64 N32",
                         "GtU-alt 16x SS M128 N32", "residual 12x SS M128 N128",
                         "12x SS M128 N256", "res 12x, 2 accumulators", "res 12x, 4 accumulators",
                         "48x SS M128 N64 one commit", "all (res+GV+GtU)",
                         "residual 12x TS (A=U TMEM)", "residual 6x TS (3 products)",
                         "GtU stacked 8x SS M128 N64", "residual 6x SS (3 products)",
                         "v2 tile: res6 + GtU16 + GV8", "v2 tile without GtU", "v2 GtU16 only",
                         "v2 tile, 1 commit", "v2 tile, 5 commits", "v2 tile, 7 commits"};
  int vars[] = {13, 14, 15, 17, 18, 19};
  for (int v : vars) {
    bench<<<1, 128, 200 * 1024>>>(v, 2000, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  }
  long long h[32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int v : vars) printf("%-28s %6lld cycles per group (incl. commit+wait)\n", names[v], h[v]);
  { unsigned char* src; cudaMalloc(&src, 512u << 20); cudaMemset(src, 0, 512u << 20); cudaMemcpyToSymbol(g_src, &src, sizeof(src)); }
  cudaFuncSetAttribute(bench_bg, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* bgn[] = {"none", "LDS.128", "STS.128", "LDS+STS", "tcgen05.ld x16", "tcgen05.st x16", "TMEM ld+st", "FFMA issue", "STS+proxy fence", "tcgen05 fences", "mbar polling", "bulk copy HBM", "TMA bulk L2 x8"};
  for (int nw : {4, 8, 16})
    for (int mode = 0; mode < 13; ++mode) {
      bench_bg<<<1, 32 * (1 + nw), 200 * 1024>>>(mode, 500, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof(long long), cudaMemcpyDeviceToHost);
      printf("v2 tile with %2d bg warps %-16s %6lld cycles\n", nw, bgn[mode], h[0]);
    }
  return 0;
}
