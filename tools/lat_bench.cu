// lat_bench.cu — latency of one bulk copy (global -> smem, mbarrier completion)
// for L2-resident sources, by size.  nvcc -gencode arch=compute_100a,code=sm_100a
//   -O2 -std=c++17 -I paper_1702_02241_b200/csrc tools/lat_bench.cu -o tools/lat_bench
#include <cuda_runtime.h>
#include <cstdio>
#include "tc_common.cuh"
using namespace spcp::tc;
__global__ void lat(const unsigned char* src, int bytes, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int it = 0; it < iters; ++it) {
      long long t0 = clock64();
      mbar_arrive_expect_tx(&bar, bytes);
      bulk_load(sm, src + (size_t)(it % 16) * bytes, bytes, &bar);
      mbar_wait(&bar, it & 1);
      tot += clock64() - t0;
    }
    out[blockIdx.x] = tot / iters;
  }
}
int main() {
  unsigned char* src; long long* d; cudaMalloc(&src, 64 << 20); cudaMalloc(&d, 1024 * 8);
  cudaMemset(src, 1, 64 << 20);
  cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int sizes[] = {1024, 4096, 8192, 16384, 32768};
  for (int grid : {1, 148}) for (int b : sizes) {
    lat<<<grid, 32, 64 * 1024>>>(src, b, 200, d);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
    long long s = 0; for (int i = 0; i < grid; ++i) s += h[i];
    printf("grid %3d bytes %6d  latency %lld cycles\n", grid, b, s / grid);
  }
  return 0;
}
