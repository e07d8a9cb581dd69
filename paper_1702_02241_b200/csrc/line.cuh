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
#include "stream_f64mma.cuh"

namespace spcp {

// R0, D1, D2 of rows [0, m) (row-major, ld = n_pad, zero pads): 64 x 64 tiles, 4 x 4 entries
// per thread, the three rank-k sums accumulated together from one staging of
// U, dU, V, dV; the next K-chunk is loaded into registers while the current
// one is multiplied (one CTA per SM at this register count, so the loads
// would otherwise sit exposed between the chunks).
template <typename TX>
__global__ void __launch_bounds__(256) line_setup_kernel(
    const double* __restrict__ z, const double* __restrict__ dz, int64_t m, int64_t n,
    int64_t n_pad, int64_t k, const TX* __restrict__ x, int64_t ldx,
    const uint32_t* __restrict__ mbits, int64_t ldm, double* __restrict__ r0,
    double* __restrict__ d1, double* __restrict__ d2) {
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
      if (gj >= n_pad) continue;
      const bool obs = gj < n && (mbits == nullptr ||
                                  ((mbits[gi * ldm + (gj >> 5)] >> (gj & 31)) & 1u));
      const int64_t o = gi * n_pad + gj;
      r0[o] = obs ? double(x[gi * ldx + gj]) - p1[e][f] : 0.0;
      d1[o] = obs ? q1[e][f] : 0.0;
      d2[o] = obs ? q2[e][f] : 0.0;
    }
  }
}

// The same three products on the FP64 tensor cores (DMMA m8n8k4, k <= 64):
// a CTA owns a 128-row band and a chunk of 64-column tiles; U, dU of the band
// are staged once, V, dV per tile; per tile three warp-tiled GEMMs (warp tile
// 32 x 32, as the evaluation's phase 1) with the accumulator reused:
// P1 = U V^T -> R0 = x - P1, then D1 = dU V^T + U dV^T, then D2 = dU dV^T.
// Output rows are n_pad long (pads hold zeros), so the probe streams aligned
// double2 pairs.
template <int KP, bool MASK>
struct LineGeom {
  static constexpr int BM = 128, BN = 64, KS = ((KP + 15) / 16) * 16 + 4;
  static constexpr size_t U_B = size_t(BM) * KS * 8, V_B = size_t(BN) * KS * 8;
  static constexpr size_t OFF_U = 0, OFF_DU = U_B, OFF_V = 2 * U_B, OFF_DV = 2 * U_B + V_B,
                          SMEM = 2 * U_B + 2 * V_B;
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <int KP, bool MASK>
__global__ void __launch_bounds__(256, 1) line_setup_mma_kernel(
    const double* __restrict__ z, const double* __restrict__ dz, int64_t m, int64_t n,
    int64_t n_pad, int64_t k, const float* __restrict__ x, int64_t ldx,
    const uint32_t* __restrict__ mbits, int64_t ldm, int64_t chunk_cols,
    double* __restrict__ r0, double* __restrict__ d1, double* __restrict__ d2) {
  using G = LineGeom<KP, MASK>;
  constexpr int BM = G::BM, BN = G::BN, KS = G::KS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Us = reinterpret_cast<double*>(smem_raw + G::OFF_U);
  double* dUs = reinterpret_cast<double*>(smem_raw + G::OFF_DU);
  double* Vs = reinterpret_cast<double*>(smem_raw + G::OFF_V);
  double* dVs = reinterpret_cast<double*>(smem_raw + G::OFF_DV);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t rb0 = int64_t(blockIdx.y) * BM;
  const int64_t c_begin = int64_t(blockIdx.x) * chunk_cols;
  const int64_t c_end = c_begin + chunk_cols < n_pad ? c_begin + chunk_cols : n_pad;
  const double *U = z, *V = z + m * k, *dU = dz, *dV = dz + m * k;
  for (int q = tid; q < BM * KP; q += 256) {
    const int r = q / KP, c = q % KP;
    const int64_t gi = rb0 + r;
    const bool ok = gi < m && c < k;
    Us[r * KS + c] = ok ? U[gi * k + c] : 0.0;
    dUs[r * KS + c] = ok ? dU[gi * k + c] : 0.0;
  }
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
  for (int64_t c0 = c_begin; c0 < c_end; c0 += BN) {
    __syncthreads();  // previous tile's V reads done
    for (int q = tid; q < BN * KP; q += 256) {
      const int r = q / KP, c = q % KP;
      const int64_t gj = c0 + r;
      const bool ok = gj < n && c < k;
      Vs[r * KS + c] = ok ? V[gj * k + c] : 0.0;
      dVs[r * KS + c] = ok ? dV[gj * k + c] : 0.0;
    }
    __syncthreads();
    double acc[4][4][2];
    auto zero = [&] {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    };
    // pass 0: P1 -> R0, 1: D1, 2: D2
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
      zero();
      const double* A0 = pass == 2 ? dUs : Us;   // first product: U V, dU V (D1), dU dV
      const double* B0 = pass == 2 ? dVs : Vs;
      const double* A1 = pass == 1 ? dUs : nullptr;  // D1 = dU V + U dV: two products
#pragma unroll 2
      for (int k0 = 0; k0 < KP; k0 += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) af[a] = (A1 ? A1 : A0)[(wr + 8 * a + gq) * KS + k0 + tq];
#pragma unroll
        for (int b = 0; b < 4; ++b) bf[b] = B0[(wc + 8 * b + gq) * KS + k0 + tq];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        if (pass == 1) {  // + U dV
#pragma unroll
          for (int a = 0; a < 4; ++a) af[a] = Us[(wr + 8 * a + gq) * KS + k0 + tq];
#pragma unroll
          for (int b = 0; b < 4; ++b) bf[b] = dVs[(wc + 8 * b + gq) * KS + k0 + tq];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
      }
      double* out = pass == 0 ? r0 : (pass == 1 ? d1 : d2);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int64_t gi = rb0 + wr + 8 * a + gq;
        if (gi >= m) continue;
        uint32_t mw0 = 0xffffffffu, mw1 = 0xffffffffu;
        if constexpr (MASK) {
          mw0 = mbits[gi * ldm + (c0 >> 5)];
          mw1 = mbits[gi * ldm + (c0 >> 5) + 1];
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = wc + 8 * b + 2 * tq;  // tile column (even)
          double v0 = acc[a][b][0], v1 = acc[a][b][1];
          if (pass == 0) {
            const float2 xv = __ldg(reinterpret_cast<const float2*>(x + gi * ldx + c0 + c));
            v0 = double(xv.x) - v0;
            v1 = double(xv.y) - v1;
          }
          if constexpr (MASK) {
            const uint32_t w = c < 32 ? mw0 : mw1;
            v0 = ((w >> (c & 31)) & 1u) ? v0 : 0.0;
            v1 = ((w >> ((c + 1) & 31)) & 1u) ? v1 : 0.0;
          }
          *reinterpret_cast<double2*>(out + gi * n_pad + c0 + c) = make_double2(v0, v1);
        }
      }
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
