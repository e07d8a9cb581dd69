// common.cuh — shared device helpers for the Split-SPCP sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/spcp_b200.h"

#define SPCP_DEV __device__ __forceinline__

namespace spcp {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define SPCP_CUDA(call)                                     \
  do {                                                      \
    cudaError_t _e = (call);                                \
    if (_e != cudaSuccess) return ::spcp::cuda_fail(_e, #call); \
  } while (0)

bool debug_sync();  // SPCP_DEBUG_SYNC=1: synchronise after every launch

#define SPCP_CHECK_LAUNCH(where)                                \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e == cudaSuccess && ::spcp::debug_sync()) _e = cudaDeviceSynchronize(); \
    if (_e != cudaSuccess) return ::spcp::cuda_fail(_e, where); \
  } while (0)

// ---------------------------------------------------------------- vectors
template <typename T, int N>
struct alignas(sizeof(T) * N) VecT {
  T v[N];
};

// 16-byte vector of T
template <typename T>
struct V16 {
  static constexpr int N = 16 / sizeof(T);
  using type = VecT<T, N>;
};

SPCP_DEV void cp_async16(void* smem, const void* gmem) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
SPCP_DEV void cp_async8(void* smem, const void* gmem) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
SPCP_DEV void cp_async4(void* smem, const void* gmem) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
SPCP_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
SPCP_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <typename T>
SPCP_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree), result valid in thread 0.
// `scratch` must hold blockDim.x/32 doubles.
SPCP_DEV double block_sum(double v, double* scratch) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

template <typename T>
SPCP_DEV T tcopysign(T a, T b);
template <>
SPCP_DEV float tcopysign<float>(float a, float b) { return copysignf(a, b); }
template <>
SPCP_DEV double tcopysign<double>(double a, double b) { return copysign(a, b); }

// Huber / clip epilogue of objective.py:108-116 for one residual r = x - l on
// an observed entry: returns g = -clip(r, +-tau) and adds huber(r) to h.
// huber(r) = c (|r| - c/2) with c = min(|r|, tau): for |r| <= tau this is the
// quadratic branch rounded exactly as 0.5*r*r; otherwise tau|r| - tau^2/2.
template <typename T>
SPCP_DEV T huber_clip(T r, T tau, T& h) {
  const T a = r < T(0) ? -r : r;
  const T c = a < tau ? a : tau;
  h += c * (a - T(0.5) * c);
  return -tcopysign<T>(c, r);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace spcp
