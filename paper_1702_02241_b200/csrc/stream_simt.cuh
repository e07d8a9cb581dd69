// stream_simt.cuh — the fused streaming pass over X (SIMT FP32 / FP64 path).
//
// One launch reads every X tile (and its mask bits) once and, per entry
//   r = x - <U_i, V_j>        (residual of the split iterate, solver.py:119)
//   r = 0 off the mask        (objective.py:109-110)
//   g = -clip(r, +-tau), huber(r) accumulated          (objective.py:112-116)
// accumulates the two rank-k reductions
//   left  = G  @ W_r  (m x PW)   -> grad_U block  (solver.py:121, W_r = V)
//   right = G^T @ W_l (n x PW)   -> grad_V block  (solver.py:122, W_l = U)
// without ever writing G.  Modes:
//   EVAL : W_r = V, W_l = U (the objective/gradient evaluation, K1)
//   APPLY: separate product operands (certificate D.V1 / U1^T D, growth)
//   RAW  : no residual, g = P_Omega(x) (rSVD sketches of the observed matrix)
//
// CTA = 256 threads, tile = 128 rows x BN columns (BN = 64 fp32 / 32 fp64).
// A CTA owns one 128-row band and a contiguous chunk of column tiles:
//  * phase A ("row owner"): thread (row, half) holds U_row in registers, walks
//    its BN/2 columns, forms r, g, huber and the left product in registers
//    and parks g in shared memory (broadcast LDS of V_j: all lanes of a warp
//    sit on the same column).
//  * phase B ("column owner"): thread (col, slice) sums g * W_l over a slice of
//    rows; slices are folded through shared memory in a fixed order and the
//    band's right-product partial is written once per tile.
// Partials are reduced by reduce kernels in a fixed order (no float atomics),
// so results are bitwise reproducible run to run.
#pragma once

#include "common.cuh"

namespace spcp {

enum StreamMode { MODE_EVAL = 0, MODE_APPLY = 1, MODE_RAW = 2 };

struct StreamParams {
  int64_t m_pad, n_pad;     // padded sizes: m_pad % 128 == 0, n_pad % 64 == 0
  int64_t ldx;              // X row stride in elements (multiple of 64)
  const void* x;            // TX[m_pad][ldx], zero pads
  const uint32_t* mbits;    // [m_pad][ldm] mask words or nullptr
  int64_t ldm;              // words per row (even)
  const void* uc;           // residual U operand T[m_pad][KP]
  const void* vc;           // residual V operand T[n_pad][KP]
  const void* wr;           // left-product operand  T[n_pad][PW]
  const void* wl;           // right-product operand T[m_pad][PW]
  void* pleft;              // T[nchunks][m_pad][PW]
  void* pright;             // T[nrb][n_pad][PW]
  double* pphi;             // [nrb*nchunks]
  double tau;
  int64_t chunk_cols;       // multiple of BN
  int nchunks;
  int do_left, do_right;
};

template <typename T>
struct StreamGeom {
  static constexpr int NT = 256;
  static constexpr int BM = 128;
  static constexpr int BN = sizeof(T) == 4 ? 64 : 32;
  static constexpr int HALF = BN / 2;
  static constexpr int NSL = NT / BN;   // phase-B row slices
  static constexpr int RPS = BM / NSL;  // rows per slice
  static constexpr int VG = 16 / int(sizeof(T));
  static constexpr int GS = BN + VG;    // g tile row stride (elements)
};

// shared-memory footprint (bytes) of one instantiation
template <typename T, typename TX, int KR, int PW, int MODE, bool MASK>
constexpr size_t stream_smem_bytes() {
  using G = StreamGeom<T>;
  constexpr int VX = 16 / int(sizeof(TX));
  constexpr size_t xs = size_t(G::BM) * (G::BN + VX) * sizeof(TX);
  constexpr size_t gs = size_t(G::BM) * G::GS * sizeof(T);
  constexpr size_t red = size_t(G::NSL) * PW * (G::BN + 1) * sizeof(T);
  constexpr size_t gsr = gs > red ? gs : red;
  constexpr size_t vs = size_t(G::BN) * KR * sizeof(T);
  constexpr size_t ws = MODE == MODE_EVAL ? 0 : size_t(G::BN) * PW * sizeof(T);
  constexpr size_t us = size_t(G::BM) * PW * sizeof(T);
  constexpr size_t ms = MASK ? size_t(G::BM) * (G::BN / 32) * 4 : 0;
  constexpr size_t lft = size_t(G::BM) * PW * sizeof(T);  // half-combine scratch
  constexpr size_t tail = lft > 0 ? lft : 0;
  (void)tail;
  return xs + gsr + vs + ws + us + ms + 64;
}

template <typename T, typename TX, int KR, int PW, int MODE, bool MASK>
__global__ void __launch_bounds__(256) stream_kernel(const StreamParams p) {
  using G = StreamGeom<T>;
  constexpr int NT = G::NT, BM = G::BM, BN = G::BN, HALF = G::HALF;
  constexpr int NSL = G::NSL, RPS = G::RPS, VG = G::VG, GS = G::GS;
  constexpr int VX = 16 / int(sizeof(TX));
  constexpr int XS = BN + VX;
  constexpr bool SHARE = (MODE == MODE_EVAL);
  static_assert(!SHARE || KR == PW, "EVAL mode shares operands");
  static_assert(KR % VG == 0 && PW % VG == 0, "operand widths must be 16B multiples");
  using XV = VecT<TX, VX>;
  using TV = VecT<T, VG>;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr size_t xs_b = size_t(BM) * XS * sizeof(TX);
  constexpr size_t gs_b = size_t(BM) * GS * sizeof(T);
  constexpr size_t red_b = size_t(NSL) * PW * (BN + 1) * sizeof(T);
  constexpr size_t gsr_b = gs_b > red_b ? gs_b : red_b;
  constexpr size_t vs_b = size_t(BN) * KR * sizeof(T);
  constexpr size_t ws_b = MODE == MODE_EVAL ? 0 : size_t(BN) * PW * sizeof(T);
  constexpr size_t us_b = size_t(BM) * PW * sizeof(T);
  TX* xs = reinterpret_cast<TX*>(smem_raw);
  T* gs = reinterpret_cast<T*>(smem_raw + xs_b);
  T* red = gs;  // aliases g tile once phase B has consumed it
  T* vs = reinterpret_cast<T*>(smem_raw + xs_b + gsr_b);
  T* ws = reinterpret_cast<T*>(smem_raw + xs_b + gsr_b + vs_b);
  T* us = reinterpret_cast<T*>(smem_raw + xs_b + gsr_b + vs_b + ws_b);
  uint32_t* ms = reinterpret_cast<uint32_t*>(smem_raw + xs_b + gsr_b + vs_b + ws_b + us_b);
  __shared__ double red_scratch[NT / 32];

  const int tid = threadIdx.x;
  const int chunk = blockIdx.x;
  const int rb = blockIdx.y;
  const int64_t r0 = int64_t(rb) * BM;
  const int64_t c_begin = int64_t(chunk) * p.chunk_cols;
  int64_t c_end = c_begin + p.chunk_cols;
  if (c_end > p.n_pad) c_end = p.n_pad;
  const int ntiles = int((c_end - c_begin) / BN);
  const T tau = T(p.tau);

  const TX* __restrict__ X = reinterpret_cast<const TX*>(p.x);
  const T* __restrict__ Uc = reinterpret_cast<const T*>(p.uc);
  const T* __restrict__ Vc = reinterpret_cast<const T*>(p.vc);
  const T* __restrict__ Wr = reinterpret_cast<const T*>(SHARE ? p.vc : p.wr);
  const T* __restrict__ Wl = reinterpret_cast<const T*>(SHARE ? p.uc : p.wl);

  auto load_tile = [&](int t) {
    const int64_t c0 = c_begin + int64_t(t) * BN;
    constexpr int CPR = BN * int(sizeof(TX)) / 16;  // 16B chunks per X row
#pragma unroll
    for (int q = tid; q < BM * CPR; q += NT) {
      const int row = q / CPR, cc = q % CPR;
      cp_async16(xs + row * XS + cc * VX, X + (r0 + row) * p.ldx + c0 + cc * VX);
    }
    if constexpr (KR > 0) {
      constexpr int NCH = BN * KR * int(sizeof(T)) / 16;
      const T* src = Vc + c0 * KR;
      for (int q = tid; q < NCH; q += NT) cp_async16(vs + q * VG, src + q * VG);
    }
    if constexpr (MODE != MODE_EVAL) {
      if (p.do_left) {
        constexpr int NCH = BN * PW * int(sizeof(T)) / 16;
        const T* src = Wr + c0 * PW;
        for (int q = tid; q < NCH; q += NT) cp_async16(ws + q * VG, src + q * VG);
      }
    }
    if constexpr (MASK) {
      if (tid < BM) {
        const uint32_t* src = p.mbits + (r0 + tid) * p.ldm + (c0 >> 5);
        if constexpr (BN == 64)
          cp_async8(ms + tid * 2, src);
        else
          cp_async4(ms + tid, src);
      }
    }
    cp_async_commit();
  };

  // ---- prologue: right-product operand rows of this band + first tile
  if (p.do_right) {
    constexpr int NCH = BM * PW * int(sizeof(T)) / 16;
    const T* src = Wl + r0 * PW;
    for (int q = tid; q < NCH; q += NT) cp_async16(us + q * VG, src + q * VG);
  }
  if (ntiles > 0) load_tile(0);

  // phase-A identity and its residual row of U (registers)
  const int arow = tid % BM;
  const int ahalf = tid / BM;
  T u[KR > 0 ? KR : 1];
  if constexpr (KR > 0) {
    const TV* src = reinterpret_cast<const TV*>(Uc + (r0 + arow) * KR);
#pragma unroll
    for (int q = 0; q < KR / VG; ++q) {
      TV t = src[q];
#pragma unroll
      for (int e = 0; e < VG; ++e) u[q * VG + e] = t.v[e];
    }
  }
  T gl[PW];
#pragma unroll
  for (int b = 0; b < PW; ++b) gl[b] = T(0);
  double phi_acc = 0.0;

  // phase-B identity
  const int bcol = tid % BN;
  const int bsl = tid / BN;

  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<0>();
    __syncthreads();  // tile t (and us) resident

    // ---------------- phase A: residual, epilogue, left product
    T hsum = T(0);
    {
      const TX* xrow = xs + arow * XS + ahalf * HALF;
      T* grow = gs + arow * GS + ahalf * HALF;
#pragma unroll 1
      for (int cg = 0; cg < HALF; cg += VX) {
        const XV xv = *reinterpret_cast<const XV*>(xrow + cg);
        uint32_t mw = 0u;
        if constexpr (MASK) mw = ms[arow * (BN / 32) + ((ahalf * HALF + cg) >> 5)];
        T gv[VX];
#pragma unroll
        for (int e = 0; e < VX; ++e) {
          const int c = ahalf * HALF + cg + e;
          T r = T(xv.v[e]);
          T vreg[KR > 0 ? KR : 1];
          if constexpr (KR > 0) {
            T a0 = T(0), a1 = T(0);
            const TV* vrow = reinterpret_cast<const TV*>(vs + c * KR);
#pragma unroll
            for (int q = 0; q < KR / VG; ++q) {
              const TV vv = vrow[q];
#pragma unroll
              for (int f = 0; f < VG; ++f) {
                vreg[q * VG + f] = vv.v[f];
                if (f & 1)
                  a1 = fma(u[q * VG + f], vv.v[f], a1);
                else
                  a0 = fma(u[q * VG + f], vv.v[f], a0);
              }
            }
            r -= (a0 + a1);
          }
          if constexpr (MASK) r = ((mw >> (c & 31)) & 1u) ? r : T(0);
          T g;
          if constexpr (MODE == MODE_RAW)
            g = r;
          else
            g = huber_clip<T>(r, tau, hsum);
          if constexpr (SHARE) {
#pragma unroll
            for (int b = 0; b < PW; ++b) gl[b] = fma(g, vreg[b], gl[b]);
          } else {
            if (p.do_left) {
              const TV* wrow = reinterpret_cast<const TV*>(ws + c * PW);
#pragma unroll
              for (int q = 0; q < PW / VG; ++q) {
                const TV ww = wrow[q];
#pragma unroll
                for (int f = 0; f < VG; ++f) gl[q * VG + f] = fma(g, ww.v[f], gl[q * VG + f]);
              }
            }
          }
          gv[e] = g;
        }
#pragma unroll
        for (int e = 0; e < VX; e += VG) {
          TV o;
#pragma unroll
          for (int f = 0; f < VG; ++f) o.v[f] = gv[e + f];
          *reinterpret_cast<TV*>(grow + cg + e) = o;
        }
      }
    }
    phi_acc += double(hsum);
    __syncthreads();  // g tile complete; xs / vs / ws / ms free

    if (t + 1 < ntiles) load_tile(t + 1);  // overlaps phase B + fold

    // ---------------- phase B: right product over this tile's columns
    if (p.do_right) {
      T gr[PW];
#pragma unroll
      for (int b = 0; b < PW; ++b) gr[b] = T(0);
#pragma unroll 2
      for (int i = bsl * RPS; i < (bsl + 1) * RPS; ++i) {
        const T g = gs[i * GS + bcol];
        const TV* wrow = reinterpret_cast<const TV*>(us + i * PW);
#pragma unroll
        for (int q = 0; q < PW / VG; ++q) {
          const TV ww = wrow[q];
#pragma unroll
          for (int f = 0; f < VG; ++f) gr[q * VG + f] = fma(g, ww.v[f], gr[q * VG + f]);
        }
      }
      __syncthreads();  // everyone done reading gs before it becomes `red`
#pragma unroll
      for (int b = 0; b < PW; ++b) red[(bsl * PW + b) * (BN + 1) + bcol] = gr[b];
      __syncthreads();
      const int64_t c0 = c_begin + int64_t(t) * BN;
      T* dst = reinterpret_cast<T*>(p.pright) + (int64_t(rb) * p.n_pad + c0) * PW;
      for (int o = tid; o < BN * PW; o += NT) {
        const int col = o / PW, b = o % PW;
        T s = T(0);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) s += red[(sl * PW + b) * (BN + 1) + col];
        dst[o] = s;
      }
    }
  }

  // ---- flush the band's left product (combine the two column halves)
  __syncthreads();
  if (p.do_left) {
    T* scr = gs;  // BM x PW scratch (fits: gs tile >= BM*PW for PW <= BN)
    if (ahalf == 1) {
#pragma unroll
      for (int b = 0; b < PW; ++b) scr[arow * PW + b] = gl[b];
    }
    __syncthreads();
    if (ahalf == 0) {
      T* dst = reinterpret_cast<T*>(p.pleft) + (int64_t(chunk) * p.m_pad + r0 + arow) * PW;
#pragma unroll
      for (int q = 0; q < PW / VG; ++q) {
        TV o;
#pragma unroll
        for (int f = 0; f < VG; ++f) o.v[f] = gl[q * VG + f] + scr[arow * PW + q * VG + f];
        reinterpret_cast<TV*>(dst)[q] = o;
      }
    }
  }
  const double tot = block_sum(phi_acc, red_scratch);
  if (tid == 0) p.pphi[int64_t(rb) * p.nchunks + chunk] = tot;
}

}  // namespace spcp
