// stream_f64.cuh — the fp64 streaming pass (fp64 mode: the L-BFGS polish,
// the certificate's and growth step's fp64 products, the rSVD sketches),
// register-blocked for the FP64 pipe.
//
// Per 128 x BN tile of X (one read of X, and of its mask bits):
//   phase 1  R = X - U_t V_t^T          thread micro-tile TR x 4, k loop over
//            g = -clip(R, +-tau), phi     Un / Vn in shared memory (rows
//                                         strided by lane so a warp's loads hit
//                                         distinct banks), 32 independent
//                                         accumulators per thread
//   phase 2  Lacc += G W_r               (128 x PW) in registers across the
//                                         CTA's column chunk (W_r = V_t in EVAL)
//   phase 3  R_t = G^T W_l               (BN x PW) written once per tile as the
//                                         row band's partial (W_l = U_band in EVAL)
// Partials have the layout of stream_kernel's (pleft[chunk][m_pad][PW],
// pright[band][n_pad][PW]) and are folded by reduce_kernel<double> in a fixed
// order, so results are bitwise reproducible.  KP (rank, padded to 8) and PW
// (product width) go up to 64; the previous per-row register design capped
// fp64 at k = 32 (a row of U and the left accumulators lived in registers).
//
// Work per element: 3 K DFMA (EVAL).  Shared-memory loads per DFMA stay below
// the FP64 issue rate: phase 1 loads TR + 4 values per 4 TR DFMA, phase 2
// 4 + PW/8 per 4 PW/8, phase 3 BN/32 + PW/8 per (BN/32) PW/8.
#pragma once

#include "common.cuh"
#include "stream_simt.cuh"

namespace spcp {

template <int KP, int PW, int MODE, typename TX>
struct F64Geom {
  static constexpr int NT = 256, BM = 128;
  static constexpr int BN = (MODE == MODE_EVAL && sizeof(TX) == 4) ? 64 : 32;
  static constexpr int KS = KP + 2;   // Un / Vn row pitch (doubles): 16-B rows, KS = 2 mod 8
  static constexpr int WS = PW + 2;   // W tile pitch (APPLY / RAW)
  static constexpr int GS = BN + 1;   // G tile pitch (odd: column reads are conflict-free)
  static constexpr int XS = BN + 16 / int(sizeof(TX));  // X tile pitch (elements)
  // phase 1 lane grid: LC lanes across columns (4 each), LR across rows (TR each)
  static constexpr int LC = BN / 8, LR = 32 / LC, TR = 32 / LR, TC = 4;
  static constexpr int TP = PW / 8;   // products: p = pg + 8 q
  static constexpr int TJ = BN / 32;  // phase 3 columns per thread
  static constexpr size_t UN_B = KP > 0 ? size_t(BM) * KS * 8 : 0;
  static constexpr size_t VN_B = KP > 0 ? size_t(BN) * KS * 8 : 0;
  static constexpr size_t WL_B = MODE != MODE_EVAL ? size_t(BM) * WS * 8 : 0;
  static constexpr size_t WR_B = MODE != MODE_EVAL ? size_t(BN) * WS * 8 : 0;
  static constexpr size_t X_B = size_t(BM) * XS * sizeof(TX);
  static constexpr size_t G_B = size_t(BM) * GS * 8;
  static constexpr size_t M_B = size_t(BM) * ((BN + 31) / 32) * 4;
  static constexpr size_t OFF_UN = 0, OFF_VN = OFF_UN + UN_B, OFF_WL = OFF_VN + VN_B,
                          OFF_WR = OFF_WL + WL_B, OFF_X = OFF_WR + WR_B, OFF_G = OFF_X + X_B,
                          OFF_M = OFF_G + G_B, SMEM = OFF_M + M_B + 64;
  static_assert(PW % 8 == 0 && PW >= 8 && PW <= 64, "product width");
  static_assert(KP % 8 == 0 && KP <= 64, "rank width");
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <int KP, int PW, int MODE, bool MASK, typename TX>
__global__ void __launch_bounds__(256, 1) f64_stream_kernel(const StreamParams p) {
  using G = F64Geom<KP, PW, MODE, TX>;
  constexpr int BM = G::BM, BN = G::BN, KS = G::KS, WS = G::WS, GS = G::GS, XS = G::XS;
  constexpr int LC = G::LC, LR = G::LR, TR = G::TR, TC = G::TC, TP = G::TP, TJ = G::TJ;
  constexpr bool EVAL = MODE == MODE_EVAL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Un = reinterpret_cast<double*>(smem_raw + G::OFF_UN);
  double* Vn = reinterpret_cast<double*>(smem_raw + G::OFF_VN);
  double* Wl = EVAL ? Un : reinterpret_cast<double*>(smem_raw + G::OFF_WL);
  double* Wr = EVAL ? Vn : reinterpret_cast<double*>(smem_raw + G::OFF_WR);
  constexpr int WLS = EVAL ? KS : WS;  // pitch of the product operands
  TX* Xs = reinterpret_cast<TX*>(smem_raw + G::OFF_X);
  double* Gs = reinterpret_cast<double*>(smem_raw + G::OFF_G);
  uint32_t* Ms = reinterpret_cast<uint32_t*>(smem_raw + G::OFF_M);
  __shared__ double red_scratch[8];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = blockIdx.x, rb = blockIdx.y;
  const int64_t r0 = int64_t(rb) * BM;
  const int64_t c_begin = int64_t(chunk) * p.chunk_cols;
  int64_t c_end = c_begin + p.chunk_cols;
  if (c_end > p.n_pad) c_end = p.n_pad;
  const int ntiles = int((c_end - c_begin) / BN);
  const double tau = p.tau;
  const TX* __restrict__ X = reinterpret_cast<const TX*>(p.x);
  const double* __restrict__ Uc = reinterpret_cast<const double*>(p.uc);
  const double* __restrict__ Vc = reinterpret_cast<const double*>(p.vc);

  // row-band operands (once): U band for the residual (and G^T U), W_l band
  if constexpr (KP > 0) {
    constexpr int CPR = KP / 2;  // 16-B chunks per row
    for (int q = tid; q < BM * CPR; q += 256) {
      const int r = q / CPR, c = q % CPR;
      cp_async16(Un + r * KS + 2 * c, Uc + (r0 + r) * KP + 2 * c);
    }
  }
  if constexpr (!EVAL) {
    if (p.do_right) {
      constexpr int CPR = PW / 2;
      const double* wl = reinterpret_cast<const double*>(p.wl);
      for (int q = tid; q < BM * CPR; q += 256) {
        const int r = q / CPR, c = q % CPR;
        cp_async16(Wl + r * WS + 2 * c, wl + (r0 + r) * PW + 2 * c);
      }
    }
  }
  // tile operands in two groups: X / mask (and V in APPLY: phase 1 only) land
  // as soon as phase 1 is done; V (EVAL: phase 2's W_r) and W_r (APPLY) after
  // phase 2.  Phases 2 and 3 hide the loads.
  auto load_x = [&](int t) {
    const int64_t c0 = c_begin + int64_t(t) * BN;
    constexpr int VX = 16 / int(sizeof(TX)), CPRX = BN / VX;
    for (int q = tid; q < BM * CPRX; q += 256) {
      const int r = q / CPRX, c = q % CPRX;
      cp_async16(Xs + r * XS + c * VX, X + (r0 + r) * p.ldx + c0 + c * VX);
    }
    if constexpr (KP > 0 && !EVAL) {
      constexpr int CPR = KP / 2;
      for (int q = tid; q < BN * CPR; q += 256) {
        const int r = q / CPR, c = q % CPR;
        cp_async16(Vn + r * KS + 2 * c, Vc + (c0 + r) * KP + 2 * c);
      }
    }
    if constexpr (MASK) {
      if (tid < BM) {
        const uint32_t* src = p.mbits + (r0 + tid) * p.ldm + (c0 >> 5);
        if constexpr (BN == 64)
          cp_async8(Ms + tid * 2, src);
        else
          cp_async4(Ms + tid, src);
      }
    }
    cp_async_commit();
  };
  auto load_w = [&](int t) {
    const int64_t c0 = c_begin + int64_t(t) * BN;
    if constexpr (KP > 0 && EVAL) {
      constexpr int CPR = KP / 2;
      for (int q = tid; q < BN * CPR; q += 256) {
        const int r = q / CPR, c = q % CPR;
        cp_async16(Vn + r * KS + 2 * c, Vc + (c0 + r) * KP + 2 * c);
      }
    }
    if constexpr (!EVAL) {
      if (p.do_left) {
        constexpr int CPR = PW / 2;
        const double* wr = reinterpret_cast<const double*>(p.wr);
        for (int q = tid; q < BN * CPR; q += 256) {
          const int r = q / CPR, c = q % CPR;
          cp_async16(Wr + r * WS + 2 * c, wr + (c0 + r) * PW + 2 * c);
        }
      }
    }
    cp_async_commit();
  };
  if (ntiles > 0) {
    load_x(0);
    load_w(0);
  }

  // phase-1 identity: rows pr0 + LR e, columns pc0 + LC c
  const int wr_ = warp >> 1, wc_ = warp & 1;
  const int pr0 = wr_ * 32 + lane / LC;
  const int pc0 = wc_ * (BN / 2) + lane % LC;
  // phase-2 identity: rows q2r + 4 e (16 rows per warp), p = pg + 8 q
  const int pg = lane & 7;
  const int q2r = warp * 16 + (lane >> 3);
  // phase-3 identity: columns cl + 32 t, p = pg + 8 q
  const int cl = tid >> 3;

  double lacc[4][TP];
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int q = 0; q < TP; ++q) lacc[e][q] = 0.0;
  double phi_acc = 0.0;

  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<0>();
    __syncthreads();  // tile t (and the band operands) resident

    // ---------------- phase 1: residual, clip / Huber, G tile
    {
      double acc[TR][TC];
#pragma unroll
      for (int e = 0; e < TR; ++e)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[e][c] = 0.0;
      if constexpr (KP > 0) {
#pragma unroll 2
        for (int k = 0; k < KP; ++k) {
          double u[TR], v[TC];
#pragma unroll
          for (int e = 0; e < TR; ++e) u[e] = Un[(pr0 + LR * e) * KS + k];
#pragma unroll
          for (int c = 0; c < TC; ++c) v[c] = Vn[(pc0 + LC * c) * KS + k];
#pragma unroll
          for (int e = 0; e < TR; ++e)
#pragma unroll
            for (int c = 0; c < TC; ++c) acc[e][c] = fma(u[e], v[c], acc[e][c]);
        }
      }
      double hsum = 0.0;
#pragma unroll
      for (int e = 0; e < TR; ++e) {
        const int r = pr0 + LR * e;
#pragma unroll
        for (int c = 0; c < TC; ++c) {
          const int col = pc0 + LC * c;
          double res = double(Xs[r * XS + col]);
          if constexpr (KP > 0) res -= acc[e][c];
          if constexpr (MASK) {
            const uint32_t mw = Ms[r * ((BN + 31) / 32) + (col >> 5)];
            res = ((mw >> (col & 31)) & 1u) ? res : 0.0;  // select: off-mask X may be garbage
          }
          double g;
          if constexpr (MODE == MODE_RAW)
            g = res;
          else
            g = huber_clip<double>(res, tau, hsum);
          Gs[r * GS + col] = g;
        }
      }
      phi_acc += hsum;
    }
    __syncthreads();  // G tile complete; X, mask (and V in APPLY) free
    if (t + 1 < ntiles) load_x(t + 1);

    // ---------------- phase 2: left product G W_r, accumulated over tiles
    if (p.do_left) {
#pragma unroll 4
      for (int j = 0; j < BN; ++j) {
        double g[4], w[TP];
#pragma unroll
        for (int e = 0; e < 4; ++e) g[e] = Gs[(q2r + 4 * e) * GS + j];
#pragma unroll
        for (int q = 0; q < TP; ++q) w[q] = Wr[j * WLS + pg + 8 * q];
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int q = 0; q < TP; ++q) lacc[e][q] = fma(g[e], w[q], lacc[e][q]);
      }
    }
    if (t + 1 < ntiles) {
      __syncthreads();  // W_r (V in EVAL) consumed
      load_w(t + 1);
    }
    // ---------------- phase 3: right product G^T W_l of this tile
    if (p.do_right) {
      double racc[TJ][TP];
#pragma unroll
      for (int s = 0; s < TJ; ++s)
#pragma unroll
        for (int q = 0; q < TP; ++q) racc[s][q] = 0.0;
#pragma unroll 4
      for (int i = 0; i < BM; ++i) {
        double g[TJ], u[TP];
#pragma unroll
        for (int s = 0; s < TJ; ++s) g[s] = Gs[i * GS + cl + 32 * s];
#pragma unroll
        for (int q = 0; q < TP; ++q) u[q] = Wl[i * WLS + pg + 8 * q];
#pragma unroll
        for (int s = 0; s < TJ; ++s)
#pragma unroll
          for (int q = 0; q < TP; ++q) racc[s][q] = fma(g[s], u[q], racc[s][q]);
      }
      const int64_t c0 = c_begin + int64_t(t) * BN;
      double* dst = reinterpret_cast<double*>(p.pright) + (int64_t(rb) * p.n_pad + c0) * PW;
#pragma unroll
      for (int s = 0; s < TJ; ++s)
#pragma unroll
        for (int q = 0; q < TP; ++q) dst[(cl + 32 * s) * PW + pg + 8 * q] = racc[s][q];
    }
  }

  // ---- flush the band's left product: pleft[chunk][r0 + row][p]
  if (p.do_left) {
    double* dst = reinterpret_cast<double*>(p.pleft) + (int64_t(chunk) * p.m_pad + r0) * PW;
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int q = 0; q < TP; ++q) dst[(q2r + 4 * e) * PW + pg + 8 * q] = lacc[e][q];
  }
  const double tot = block_sum(phi_acc, red_scratch);
  if (tid == 0) p.pphi[int64_t(rb) * p.nchunks + chunk] = tot;
}

}  // namespace spcp
