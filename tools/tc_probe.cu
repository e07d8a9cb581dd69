// tc_probe.cu — verifies the tcgen05 / TMEM / TMA building blocks the fused
// tensor-core kernel relies on, against exact CPU results (small integers,
// so every product and sum is exact in fp32).
//
//   P1  D = A B^T, A (128x32) and B (64x32) K-major SW64 images in smem
//   P2  same with A written to TMEM (2 fp16 per 32-bit column)
//   P3  D = G^T U: A = G MN-major SW128 (K = 128 rows, M = 128 = 2 atoms),
//       B = U MN-major SW64 (the same image as P1's A)
//   P4  D = G V: A = G from TMEM (K = 64), B = V MN-major SW64 (P1's B image)
//   P5  TMA 2-D tile load fp32 box {32, 128} SWIZZLE_128B + swizzled reads
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1702_02241_b200/csrc tools/tc_probe.cu -o tools/tc_probe
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace spcp::tc;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      exit(2);                                                                     \
    }                                                                              \
  } while (0)

struct Out {
  float d1[128 * 64], d2[128 * 64], d3[128 * 32], d4[128 * 32], x5[128 * 32];
  float d6[128 * 32];
  float d7[128 * 64];
  uint32_t cp_raw[128 * 16], st_raw[128 * 16];
};

__global__ void __launch_bounds__(128) probe(const __half* U, const __half* V, const __half* G,
                                             const __grid_constant__ CUtensorMap xmap, Out* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* a_img = sm;                 // 8 KB  U: 128 rows x 64 B (SW64)
  unsigned char* b_img = sm + 8192;          // 4 KB  V: 64 rows x 64 B (SW64)
  unsigned char* g_img = sm + 16384;         // 32 KB G: 2 MN atoms x 16 K-groups x 1 KB
  float* x_img = reinterpret_cast<float*>(sm + 65536);  // 16 KB TMA box
  __shared__ uint64_t bar_mma, bar_tma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;

  // ---- operand images (generic-proxy stores)
  for (int q = tid; q < 128 * 32; q += 128) {
    const int r = q / 32, k = q % 32;
    *reinterpret_cast<__half*>(a_img + Swz<64>::offset(r, k * 2)) = U[q];
  }
  for (int q = tid; q < 64 * 32; q += 128) {
    const int r = q / 32, k = q % 32;
    *reinterpret_cast<__half*>(b_img + Swz<64>::offset(r, k * 2)) = V[q];
  }
  for (int q = tid; q < 128 * 128; q += 128) {  // G[i][j], K = i, MN = j
    const int i = q / 128, j = q % 128;
    const int atom = j / 64, jj = j % 64;
    *reinterpret_cast<__half*>(g_img + atom * 16384 + Swz<128>::offset(i, jj * 2)) = G[q];
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  if (tid == 0) {
    mbar_init(&bar_mma, 1);
    mbar_init(&bar_tma, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;

  // ---- TMEM A operands: U (cols 128..143) and G[:, 0:64] (cols 192..223)
  {
    const int row = warp * 32 + (tid % 32);
    uint32_t r[16];
    for (int c = 0; c < 16; ++c) {
      __half lo = U[row * 32 + 2 * c], hi = U[row * 32 + 2 * c + 1];
      r[c] = uint32_t(__half_as_ushort(lo)) | (uint32_t(__half_as_ushort(hi)) << 16);
    }
    tmem_st16(tm + lane_base + 128, r);
    for (int h = 0; h < 2; ++h) {
      for (int c = 0; c < 16; ++c) {
        __half lo = G[row * 128 + h * 32 + 2 * c], hi = G[row * 128 + h * 32 + 2 * c + 1];
        r[c] = uint32_t(__half_as_ushort(lo)) | (uint32_t(__half_as_ushort(hi)) << 16);
      }
      tmem_st16(tm + lane_base + 192 + h * 16, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (tid == 0) {
    const uint32_t a0 = smem_u32(a_img), b0 = smem_u32(b_img), g0 = smem_u32(g_img);
    // P1
    for (int s = 0; s < 2; ++s)
      mma_ss(tm + 0, umma_desc(a0 + 32 * s, 16, 512, SW_64), umma_desc(b0 + 32 * s, 16, 512, SW_64),
             idesc_f16(128, 64, false, false), s > 0);
    // P2
    for (int s = 0; s < 2; ++s)
      mma_ts(tm + 64, tm + 128 + 8 * s, umma_desc(b0 + 32 * s, 16, 512, SW_64),
             idesc_f16(128, 64, false, false), s > 0);
    // P3: K = 128 rows of G / U, 16 per step = 2 K-groups
    for (int s = 0; s < 8; ++s)
      mma_ss(tm + 160, umma_desc(g0 + 2048 * s, 16384, 1024, SW_128),
             umma_desc(a0 + 1024 * s, 8192, 512, SW_64), idesc_f16(128, 32, true, true), s > 0);
    // P4: K = 64 columns of G / rows of V
    for (int s = 0; s < 4; ++s)
      mma_ts(tm + 224, tm + 192 + 8 * s, umma_desc(b0 + 1024 * s, 8192, 512, SW_64),
             idesc_f16(128, 32, false, true), s > 0);
    // P6: M = 64 accumulator, D = G[:, 0:64]^T U (64 x 32), read all lanes
    for (int s = 0; s < 8; ++s)
      mma_ss(tm + 256, umma_desc(g0 + 2048 * s, 16384, 1024, SW_128),
             umma_desc(a0 + 1024 * s, 8192, 512, SW_64), idesc_f16(64, 32, true, true), s > 0);
    // P7: tcgen05.cp of the K-major SW64 U image (one K-step of 16 fp16 = 8
    // TMEM columns per copy) into cols 320.., then a TS MMA from the copy
    for (int s = 0; s < 2; ++s)
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 320 + 8 * s),
                   "l"(umma_desc(a0 + 32 * s, 16, 512, SW_64))
                   : "memory");
    for (int s = 0; s < 2; ++s)
      mma_ts(tm + 352, tm + 320 + 8 * s, umma_desc(b0 + 32 * s, 16, 512, SW_64),
             idesc_f16(128, 64, false, false), s > 0);
    mma_commit(&bar_mma);
    // P5: TMA
    mbar_arrive_expect_tx(&bar_tma, 128 * 32 * 4);
    tma_load_2d(x_img, &xmap, 32, 128, &bar_tma);
  }
  mbar_wait(&bar_mma, 0);
  mbar_wait(&bar_tma, 0);
  tc_fence_after();
  const int row = warp * 32 + (tid % 32);
  uint32_t r[16];
  for (int c0 = 0; c0 < 64; c0 += 16) {
    tmem_ld16(tm + lane_base + c0, r);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out->d1[row * 64 + c0 + c] = __uint_as_float(r[c]);
    tmem_ld16(tm + lane_base + 64 + c0, r);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out->d2[row * 64 + c0 + c] = __uint_as_float(r[c]);
  }
  for (int c0 = 0; c0 < 32; c0 += 16) {
    tmem_ld16(tm + lane_base + 160 + c0, r);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out->d3[row * 32 + c0 + c] = __uint_as_float(r[c]);
    tmem_ld16(tm + lane_base + 224 + c0, r);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out->d4[row * 32 + c0 + c] = __uint_as_float(r[c]);
    tmem_ld16(tm + lane_base + 256 + c0, r);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out->d6[row * 32 + c0 + c] = __uint_as_float(r[c]);
  }
  for (int c0 = 0; c0 < 64; c0 += 16) {
    tmem_ld16(tm + lane_base + 352 + c0, r);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out->d7[row * 64 + c0 + c] = __uint_as_float(r[c]);
  }
  tmem_ld16(tm + lane_base + 320, r);
  tmem_wait_ld();
  for (int c = 0; c < 16; ++c) out->cp_raw[row * 16 + c] = r[c];
  tmem_ld16(tm + lane_base + 128, r);
  tmem_wait_ld();
  for (int c = 0; c < 16; ++c) out->st_raw[row * 16 + c] = r[c];
  for (int c = 0; c < 32; ++c) {
    const uint32_t o = Swz<128>::offset(row, c * 4);
    out->x5[row * 32 + c] = *reinterpret_cast<const float*>(reinterpret_cast<unsigned char*>(x_img) + o);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  std::vector<__half> U(128 * 32), V(64 * 32), G(128 * 128);
  std::vector<float> Uf(U.size()), Vf(V.size()), Gf(G.size());
  srand(1);
  for (size_t i = 0; i < U.size(); ++i) { Uf[i] = float(rand() % 7 - 3); U[i] = __float2half(Uf[i]); }
  for (size_t i = 0; i < V.size(); ++i) { Vf[i] = float(rand() % 7 - 3); V[i] = __float2half(Vf[i]); }
  for (size_t i = 0; i < G.size(); ++i) { Gf[i] = float(rand() % 5 - 2); G[i] = __float2half(Gf[i]); }
  const int XR = 256, XC = 128;
  std::vector<float> X(XR * XC);
  for (int i = 0; i < XR * XC; ++i) X[i] = float(i);
  __half *dU, *dV, *dG;
  float* dX;
  Out* dO;
  CK(cudaMalloc(&dU, U.size() * 2));
  CK(cudaMalloc(&dV, V.size() * 2));
  CK(cudaMalloc(&dG, G.size() * 2));
  CK(cudaMalloc(&dX, X.size() * 4));
  CK(cudaMalloc(&dO, sizeof(Out)));
  CK(cudaMemcpy(dU, U.data(), U.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dG, G.data(), G.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice));
  EncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                             cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t dims[2] = {XC, XR};
  cuuint64_t strides[1] = {XC * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", int(cr)); return 2; }
  const int smem = 65536 + 16384;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<<<1, 128, smem>>>(dU, dV, dG, map, dO);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  Out* h = new Out;
  CK(cudaMemcpy(h, dO, sizeof(Out), cudaMemcpyDeviceToHost));
  int bad1 = 0, bad2 = 0, bad3 = 0, bad4 = 0, bad5 = 0, bad7 = 0, bad7r = 0;
  for (int i = 0; i < 128 * 16; ++i) bad7r += h->cp_raw[i] != h->st_raw[i];
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 64; ++j) {
      float e = 0;
      for (int k = 0; k < 32; ++k) e += Uf[i * 32 + k] * Vf[j * 32 + k];
      bad1 += h->d1[i * 64 + j] != e;
      bad2 += h->d2[i * 64 + j] != e;
      bad7 += h->d7[i * 64 + j] != e;
    }
  for (int j = 0; j < 128; ++j)
    for (int c = 0; c < 32; ++c) {
      float e = 0;
      for (int i = 0; i < 128; ++i) e += Gf[i * 128 + j] * Uf[i * 32 + c];
      bad3 += h->d3[j * 32 + c] != e;
    }
  for (int i = 0; i < 128; ++i)
    for (int c = 0; c < 32; ++c) {
      float e = 0;
      for (int j = 0; j < 64; ++j) e += Gf[i * 128 + j] * Vf[j * 32 + c];
      bad4 += h->d4[i * 32 + c] != e;
    }
  for (int i = 0; i < 128; ++i)
    for (int c = 0; c < 32; ++c) bad5 += h->x5[i * 32 + c] != X[(128 + i) * XC + 32 + c];
  // P6: locate each expected row j (0..63) among the 128 lanes (first 16 cols)
  int found = 0, identity = 0;
  for (int j = 0; j < 64; ++j) {
    float e[32];
    for (int c = 0; c < 32; ++c) {
      e[c] = 0;
      for (int i = 0; i < 128; ++i) e[c] += Gf[i * 128 + j] * Uf[i * 32 + c];
    }
    for (int ln = 0; ln < 128; ++ln) {
      bool ok = true;
      for (int c = 0; c < 32 && ok; ++c) ok = h->d6[ln * 32 + c] == e[c];
      if (ok) { ++found; identity += (ln == j); if (j < 4 || j > 60) printf("P6 row %d -> lane %d\n", j, ln); break; }
    }
  }
  printf("P6 M=64 accumulator rows found %d / 64 (lane == row for %d)\n", found, identity);
  printf("P1 ss K-major SW64          mismatches %d / %d  (d1[0]=%g)\n", bad1, 128 * 64, h->d1[0]);
  printf("P2 ts A-in-TMEM             mismatches %d / %d\n", bad2, 128 * 64);
  printf("P3 ss MN-major SW128 x SW64 mismatches %d / %d\n", bad3, 128 * 32);
  printf("P4 ts A-TMEM x MN-major B   mismatches %d / %d\n", bad4, 128 * 32);
  printf("P5 TMA SW128 fp32 tile      mismatches %d / %d\n", bad5, 128 * 32);
  printf("P7 tcgen05.cp U -> TMEM     raw mismatches vs tcgen05.st %d / %d, TS MMA mismatches %d / %d\n",
         bad7r, 128 * 16, bad7, 128 * 64);
  return (bad1 + bad2 + bad3 + bad4 + bad5 + bad7) ? 1 : 0;
}
