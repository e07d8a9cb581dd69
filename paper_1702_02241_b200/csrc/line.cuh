// Line-restricted evaluation for the fp64 line searches (lbfgs.py:64-99 probes
// f and f' along one ray per search).  On the ray z + a dz the residual is a
// quadratic in a:
//   R(a) = X - (U + a dU)(V + a dV)^T = R0 - a D1 - a^2 D2   on Omega,
//   R0 = X - U V^T,  D1 = dU V^T + U dV^T,  D2 = dU dV^T,
// so after one setup pass that stores R0, D1, D2 (float64, 24 bytes per
// entry) every further probe is a single HBM stream with no rank-k products:
//   phi(a)  = sum huber(R(a)),
//   phi'(a) = sum g(R(a)) (D1 + 2 a D2),  g = -clip(R, +-tau)  (dphi/dL).
// Off-Omega entries are stored as zeros (huber(0) = 0, g(0) = 0).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace spcp {

// R0, D1, D2 of rows [0, m) (row-major, ld = n): 64 x 64 tiles, 4 x 4 entries
// per thread, the three rank-k sums accumulated together from one staging of
// U, dU, V, dV; the next K-chunk is loaded into registers while the current
// one is multiplied (one CTA per SM at this register count, so the loads
// would otherwise sit exposed between the chunks).
template <typename TX>
__global__ void __launch_bounds__(256) line_setup_kernel(
    const double* __restrict__ z, const double* __restrict__ dz, int64_t m, int64_t n,
    int64_t k, const TX* __restrict__ x, int64_t ldx, const uint32_t* __restrict__ mbits,
    int64_t ldm, double* __restrict__ r0, double* __restrict__ d1, double* __restrict__ d2) {
  constexpr int TB = 64, KC = 8;
  __shared__ double st[4][KC][TB + 1];  // U, dU (tile rows), V, dV (tile columns)
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t i0 = int64_t(blockIdx.y) * TB, j0 = int64_t(blockIdx.x) * TB;
  const double* src[4] = {z, dz, z + m * k, dz + m * k};
  // this thread's 8 staging slots: array a = i / 2, (row, column) from q
  double pre[8];
  auto gload = [&](int64_t kc) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int q = int(threadIdx.x) + 256 * (i & 1);
      const int r = q / KC, c = q % KC;
      const int64_t row = (i < 4 ? i0 : j0) + r, lim = i < 4 ? m : n, gk = kc + c;
      pre[i] = (row < lim && gk < k) ? __ldg(src[i >> 1] + row * k + gk) : 0.0;
    }
  };
  double p1[4][4] = {}, q1[4][4] = {}, q2[4][4] = {};
  gload(0);
  for (int64_t kc = 0; kc < k; kc += KC) {
    __syncthreads();  // the previous chunk's reads are done
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int q = int(threadIdx.x) + 256 * (i & 1);
      st[i >> 1][q % KC][q / KC] = pre[i];
    }
    __syncthreads();
    if (kc + KC < k) gload(kc + KC);
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      double a[4], da[4], b[4], db[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = st[0][c][ty * 4 + e];
        da[e] = st[1][c][ty * 4 + e];
        b[e] = st[2][c][tx * 4 + e];
        db[e] = st[3][c][tx * 4 + e];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          p1[e][f] = fma(a[e], b[f], p1[e][f]);
          q1[e][f] = fma(a[e], db[f], fma(da[e], b[f], q1[e][f]));
          q2[e][f] = fma(da[e], db[f], q2[e][f]);
        }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t gi = i0 + ty * 4 + e;
    if (gi >= m) continue;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int64_t gj = j0 + tx * 4 + f;
      if (gj >= n) continue;
      const bool obs = mbits == nullptr || ((mbits[gi * ldm + (gj >> 5)] >> (gj & 31)) & 1u);
      const int64_t o = gi * n + gj;
      r0[o] = obs ? double(x[gi * ldx + gj]) - p1[e][f] : 0.0;
      d1[o] = obs ? q1[e][f] : 0.0;
      d2[o] = obs ? q2[e][f] : 0.0;
    }
  }
}

// One probe: block partials of phi(a) and phi'(a) over a fixed grid
// (grid-stride in a fixed order, so the sums are reproducible).
__global__ void __launch_bounds__(256) line_probe_kernel(
    const double* __restrict__ r0, const double* __restrict__ d1, const double* __restrict__ d2,
    int64_t total, double alpha, double tau, double* __restrict__ part) {
  __shared__ double scratch[32];
  double h = 0.0, s = 0.0;
  const double a2 = 2.0 * alpha;
  const int64_t pairs = total >> 1;
  const double2* r2 = reinterpret_cast<const double2*>(r0);
  const double2* p2 = reinterpret_cast<const double2*>(d1);
  const double2* q2 = reinterpret_cast<const double2*>(d2);
  auto one = [&](double r, double p, double q) {
    const double rr = fma(-alpha, fma(alpha, q, p), r);  // R0 - a (D1 + a D2)
    const double g = huber_clip<double>(rr, tau, h);
    s = fma(g, fma(a2, q, p), s);
  };
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < pairs;
       t += int64_t(gridDim.x) * blockDim.x) {
    const double2 r = __ldcs(r2 + t), p = __ldcs(p2 + t), q = __ldcs(q2 + t);
    one(r.x, p.x, q.x);
    one(r.y, p.y, q.y);
  }
  if ((total & 1) && blockIdx.x == 0 && threadIdx.x == 0)
    one(r0[total - 1], d1[total - 1], d2[total - 1]);
  h = block_sum(h, scratch);
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = h;
    part[2 * blockIdx.x + 1] = s;
  }
}

// fixed-order fold of the probe partials -> out[0] = phi, out[1] = phi'
__global__ void line_fold_kernel(const double* __restrict__ part, int nb,
                                 double* __restrict__ out) {
  __shared__ double scratch[32];
  double h = 0.0, s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    h += part[2 * b];
    s += part[2 * b + 1];
  }
  h = block_sum(h, scratch);
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) {
    out[0] = h;
    out[1] = s;
  }
}

}  // namespace spcp
