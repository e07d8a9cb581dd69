// hbm_probe.cu — the achievable read-only HBM stream on this B200: the
// ceiling a kernel that reads X once can reach (MEASURED_PEAKS.json's hbm_gbs
// is a copy, read + write).  Reads 1.6 GB (the C2 X) with 128-bit loads, a
// persistent grid of 148 x occupancy CTAs, and reports GB/s for a burst (20
// launches) and a sustained run (~2 s, past the power-cap transition).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_probe tools/hbm_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_sum(const float4* __restrict__ x, long long n4, float* out) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
#pragma unroll 4
  for (; i < n4; i += stride) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(x + i));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const long long bytes = 20096LL * 20032 * 4;
  const long long n4 = bytes / 16;
  float4* x;
  float* o;
  cudaMalloc(&x, bytes);
  cudaMalloc(&o, 4);
  cudaMemset(x, 0, bytes);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, read_sum, 512, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocks_per_sm : {1, 2, occ}) {
    const int grid = 148 * blocks_per_sm;
    for (int i = 0; i < 5; ++i) read_sum<<<grid, 512>>>(x, n4, o);
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) read_sum<<<grid, 512>>>(x, n4, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("burst grid=%d: %.4f ms/read  %.1f GB/s\n", grid, ms / 20, bytes / (ms / 20 * 1e-3) / 1e9);
  }
  const int grid = 148 * occ;
  cudaEventRecord(a);
  for (int i = 0; i < 6000; ++i) read_sum<<<grid, 512>>>(x, n4, o);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("sustained (6000 reads, %.2f s): %.4f ms/read  %.1f GB/s\n", ms * 1e-3, ms / 6000,
         bytes / (ms / 6000 * 1e-3) / 1e9);
  return 0;
}
