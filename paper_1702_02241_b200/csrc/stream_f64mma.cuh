// stream_f64mma.cuh — the fp64 evaluation pass on the FP64 tensor cores
// (DMMA, mma.sync m8n8k4 f64): the L-BFGS polish of the mixed solver and every
// fp64-mode evaluation of fp32-exact data (X read as fp32, all arithmetic fp64).
//
// Per 128 x 64 tile of X (read once), three warp-level fp64 GEMM phases:
//   1  S = U_t V_t^T          m8n8k4 DMMAs, warp tile 32 x 32 (16 accumulators),
//      epilogue on the accumulator fragments: r = x - S (mask: select),
//      g = -clip(r, +-tau), phi += huber(r); G tile -> shared memory
//   2  Lacc += G V_t          (128 x KP) accumulated over the CTA's column chunk
//                              in registers (warp: 16 rows x KP)
//   3  R_t = G^T U_t          (64 x KP) per tile (warp: 8 columns x KP, K = 128)
// Each DMMA is 256 fp64 FMAs for two 8-byte shared-memory operand loads per
// thread, so the FP64 pipe, not shared memory or issue, bounds the pass (the
// SIMT kernels load 1 operand per 2-4 FMAs).  Partials use the SIMT kernels'
// layout (pleft[chunk][m_pad][KP], pright[band][n_pad][KP]) and are folded by
// reduce_kernel<double> in a fixed order: bitwise reproducible.
// (ncu at C2, k = 20: DMMA pipe 68% busy, top stalls "wait" and math-pipe
// throttle; splitting phases 2 / 3 over warp pairs for twice the independent
// accumulators measured 3.35 vs 3.25 ms, so the single-warp K loops stay.)
#pragma once

#include <type_traits>

#include "common.cuh"
#include "stream_simt.cuh"

namespace spcp {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int KP>
struct MmaGeom {
  static constexpr int NT = 256, BM = 128, BN = 64;
  // pitches (doubles): 2 * pitch = 8 (mod 32) banks, so the 8 rows x 4
  // consecutive values of an A / B fragment load hit distinct bank quads
  static constexpr int KS = ((KP + 15) / 16) * 16 + 4;
  static constexpr int GS = BN + 4;
  static constexpr int XS = BN + 4;  // floats
  static constexpr int NN = KP / 8;  // n-tiles of the rank dimension
  static constexpr size_t U_B = size_t(BM) * KS * 8, V_B = size_t(BN) * KS * 8;
  static constexpr size_t X_B = size_t(BM) * XS * 4, G_B = size_t(BM) * GS * 8;
  static constexpr size_t M_B = size_t(BM) * 2 * 4;
  static constexpr size_t OFF_U = 0, OFF_V = U_B, OFF_X = OFF_V + V_B, OFF_G = OFF_X + X_B,
                          OFF_M = OFF_G + G_B, SMEM = OFF_M + M_B + 64;
  static_assert(KP % 8 == 0 && KP <= 64, "rank width");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// RAW0: the k = 0 products of the randomized SVD (linalg.py:77-106 sketches
// X W and X^T Q): phase 1 only stages the observed X tile as G (fp64), and
// phases 2 / 3 run when p.do_left / p.do_right ask for them, with uc / vc
// holding the staged W_left / W_right (KP columns).
// GOUT (4 / 8): phase 1 only, the G tile written to p.pleft as float / double
// [m_pad][ldx] (spcp_grad_store: the certificate's stored gradient).
template <int KP, bool MASK, bool RAW0 = false, int GOUT = 0>
__global__ void __launch_bounds__(256, 1) f64_mma_kernel(const StreamParams p) {
  using G = MmaGeom<KP>;
  constexpr int BM = G::BM, BN = G::BN, KS = G::KS, GS = G::GS, XS = G::XS, NN = G::NN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Us = reinterpret_cast<double*>(smem_raw + G::OFF_U);
  double* Vs = reinterpret_cast<double*>(smem_raw + G::OFF_V);
  float* Xs = reinterpret_cast<float*>(smem_raw + G::OFF_X);
  double* Gs = reinterpret_cast<double*>(smem_raw + G::OFF_G);
  uint32_t* Ms = reinterpret_cast<uint32_t*>(smem_raw + G::OFF_M);
  __shared__ double red_scratch[8];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;  // fragment row group / thread in group
  const int chunk = blockIdx.x, rb = blockIdx.y;
  const int64_t r0 = int64_t(rb) * BM;
  const int64_t c_begin = int64_t(chunk) * p.chunk_cols;
  int64_t c_end = c_begin + p.chunk_cols;
  if (c_end > p.n_pad) c_end = p.n_pad;
  const int ntiles = int((c_end - c_begin) / BN);
  const double tau = p.tau;
  const float* __restrict__ X = reinterpret_cast<const float*>(p.x);
  const double* __restrict__ Uc = reinterpret_cast<const double*>(p.uc);
  const double* __restrict__ Vc = reinterpret_cast<const double*>(p.vc);

  const bool need_u = !RAW0 || p.do_right, need_v = !RAW0 || p.do_left;
  const bool do_left = GOUT == 0 && need_v, do_right = GOUT == 0 && need_u;
  if (need_u) {  // the row band's U (once)
    constexpr int CPR = KP / 2;
    for (int q = tid; q < BM * CPR; q += 256) {
      const int r = q / CPR, c = q % CPR;
      cp_async16(Us + r * KS + 2 * c, Uc + (r0 + r) * KP + 2 * c);
    }
  }
  // X / mask of a tile (land once phase 1 is done); V of a tile (after phase 2)
  auto load_x = [&](int t) {
    const int64_t c0 = c_begin + int64_t(t) * BN;
    constexpr int CPR = BN / 4;
    for (int q = tid; q < BM * CPR; q += 256) {
      const int r = q / CPR, c = q % CPR;
      cp_async16(Xs + r * XS + 4 * c, X + (r0 + r) * p.ldx + c0 + 4 * c);
    }
    if constexpr (MASK) {
      if (tid < BM) cp_async8(Ms + tid * 2, p.mbits + (r0 + tid) * p.ldm + (c0 >> 5));
    }
    cp_async_commit();
  };
  auto load_v = [&](int t) {
    const int64_t c0 = c_begin + int64_t(t) * BN;
    constexpr int CPR = KP / 2;
    for (int q = tid; q < (need_v ? BN * CPR : 0); q += 256) {
      const int r = q / CPR, c = q % CPR;
      cp_async16(Vs + r * KS + 2 * c, Vc + (c0 + r) * KP + 2 * c);
    }
    cp_async_commit();
  };
  if (ntiles > 0) {
    load_x(0);
    load_v(0);
  }

  // phase 1 warp tile: rows wr1 .. +32 (4 m-tiles), columns wc1 .. +32 (4 n-tiles)
  const int wr1 = (warp >> 1) * 32, wc1 = (warp & 1) * 32;
  // phase 2: rows 16 w .. +16 (2 m-tiles) x NN n-tiles, accumulated over tiles
  double lacc[2][NN][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NN; ++b) lacc[a][b][0] = lacc[a][b][1] = 0.0;
  double phi_acc = 0.0;

  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<0>();
    __syncthreads();  // X, V of tile t (and U) resident

    // ---------------- phase 1: S = U V^T, epilogue, G tile
    if constexpr (RAW0) {  // G = the observed X tile
      for (int q = tid; q < BM * (BN / 2); q += 256) {
        const int r = q / (BN / 2), c = 2 * (q % (BN / 2));
        const float2 xv = *reinterpret_cast<const float2*>(Xs + r * XS + c);
        double2 g = make_double2(double(xv.x), double(xv.y));
        if constexpr (MASK) {
          const uint32_t w = Ms[r * 2 + (c >> 5)];
          g.x = ((w >> (c & 31)) & 1u) ? g.x : 0.0;
          g.y = ((w >> ((c + 1) & 31)) & 1u) ? g.y : 0.0;
        }
        *reinterpret_cast<double2*>(Gs + r * GS + c) = g;
      }
    } else {
      double acc[4][4][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 2
      for (int k0 = 0; k0 < KP; k0 += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) af[a] = Us[(wr1 + 8 * a + gq) * KS + k0 + tq];
#pragma unroll
        for (int b = 0; b < 4; ++b) bf[b] = Vs[(wc1 + 8 * b + gq) * KS + k0 + tq];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      }
      double hs = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int r = wr1 + 8 * a + gq;
        uint32_t mw0 = 0xffffffffu, mw1 = 0xffffffffu;
        if constexpr (MASK) {
          mw0 = Ms[r * 2];
          mw1 = Ms[r * 2 + 1];
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = wc1 + 8 * b + 2 * tq;
          const float2 xv = *reinterpret_cast<const float2*>(Xs + r * XS + c);
          double r0v = double(xv.x) - acc[a][b][0];
          double r1v = double(xv.y) - acc[a][b][1];
          if constexpr (MASK) {
            const uint32_t w = c < 32 ? mw0 : mw1;  // select: off-mask X may be garbage
            r0v = ((w >> (c & 31)) & 1u) ? r0v : 0.0;
            r1v = ((w >> ((c + 1) & 31)) & 1u) ? r1v : 0.0;
          }
          double2 g;
          g.x = huber_clip<double>(r0v, tau, hs);
          g.y = huber_clip<double>(r1v, tau, hs);
          *reinterpret_cast<double2*>(Gs + r * GS + c) = g;
        }
      }
      phi_acc += hs;
    }
    __syncthreads();  // G tile complete; X and the mask free
    if (t + 1 < ntiles) load_x(t + 1);
    if constexpr (GOUT != 0) {
      using TO = typename std::conditional<GOUT == 4, float, double>::type;
      if (t + 1 < ntiles) load_v(t + 1);  // V_t consumed by phase 1
      const int64_t c0 = c_begin + int64_t(t) * BN;
      TO* dst = reinterpret_cast<TO*>(p.pleft);
      for (int q = tid; q < BM * (BN / 2); q += 256) {
        const int r = q / (BN / 2), c = 2 * (q % (BN / 2));
        const double2 g = *reinterpret_cast<const double2*>(Gs + r * GS + c);
        TO* o = dst + (r0 + r) * p.ldx + c0 + c;
        o[0] = TO(g.x);
        o[1] = TO(g.y);
      }
      continue;
    }

    // ---------------- phase 2: Lacc += G V_t   (A = G rows, B = V_t)
    if (do_left) {
      const int wr2 = warp * 16;
#pragma unroll 4
      for (int j0 = 0; j0 < BN; j0 += 4) {
        double af[2], bf[NN];
#pragma unroll
        for (int a = 0; a < 2; ++a) af[a] = Gs[(wr2 + 8 * a + gq) * GS + j0 + tq];
#pragma unroll
        for (int b = 0; b < NN; ++b) bf[b] = Vs[(j0 + tq) * KS + 8 * b + gq];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < NN; ++b) dmma_8x8x4(lacc[a][b][0], lacc[a][b][1], af[a], bf[b]);
      }
    }
    if (t + 1 < ntiles) {
      __syncthreads();  // V_t consumed
      load_v(t + 1);
    }
    // ---------------- phase 3: R_t = G^T U   (A = G^T: columns 8 w .., K = rows)
    if (do_right) {
      double racc[NN][2];
#pragma unroll
      for (int b = 0; b < NN; ++b) racc[b][0] = racc[b][1] = 0.0;
      const int wc3 = warp * 8;
#pragma unroll 4
      for (int i0 = 0; i0 < BM; i0 += 4) {
        const double af = Gs[(i0 + tq) * GS + wc3 + gq];
        double bf[NN];
#pragma unroll
        for (int b = 0; b < NN; ++b) bf[b] = Us[(i0 + tq) * KS + 8 * b + gq];
#pragma unroll
        for (int b = 0; b < NN; ++b) dmma_8x8x4(racc[b][0], racc[b][1], af, bf[b]);
      }
      const int64_t c0 = c_begin + int64_t(t) * BN;
      double* dst = reinterpret_cast<double*>(p.pright) +
                    (int64_t(rb) * p.n_pad + c0 + wc3 + gq) * KP + 2 * tq;
#pragma unroll
      for (int b = 0; b < NN; ++b)
        *reinterpret_cast<double2*>(dst + 8 * b) = make_double2(racc[b][0], racc[b][1]);
    }
  }

  // ---- flush the band's left product: pleft[chunk][r0 + row][p]
  if (do_left) {
    const int wr2 = warp * 16;
    double* dst = reinterpret_cast<double*>(p.pleft) + (int64_t(chunk) * p.m_pad + r0) * KP;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < NN; ++b)
        *reinterpret_cast<double2*>(dst + (wr2 + 8 * a + gq) * KP + 8 * b + 2 * tq) =
            make_double2(lacc[a][b][0], lacc[a][b][1]);
  }
  const double tot = block_sum(phi_acc, red_scratch);
  if (tid == 0) p.pphi[int64_t(rb) * p.nchunks + chunk] = tot;
}

}  // namespace spcp
