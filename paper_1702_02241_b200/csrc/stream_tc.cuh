// stream_tc.cuh — the fused objective/gradient pass on the 5th-gen tensor
// cores (fp32 mode, k <= 64).  One launch streams X once (TMA, SWIZZLE_128B)
// and computes, per 128 x 64 tile (sub-band sb, column tile tc):
//
//   S   = U_sb V_tc^T                  tcgen05.mma, fp16 operands, fp32 in TMEM
//   r   = x - S  (mask), g = -clip(r, +-tau), phi += huber(r)   (epilogue warps)
//   GV += G V_tc      (A = G from TMEM, B = V image MN-major)   -> grad_U block
//   GT  = G^T U_sb    (A = G image in smem MN-major, M = 64)    -> grad_V block
//
// Precision: operands are power-of-two scaled and split into
// two fp16 pieces computed in fp64 on the device, U'' = uh + um, V'' = vh +
// vm (relative representation error ~2^-22); the residual uses the three
// products uh.vh + uh.vm + um.vh, G'' = gh + gl, and the reductions use
// [gh|gl] x [vh|vm] (all four products where the N-concatenated form makes
// the fourth free).  Every product is exact in the fp32 accumulator; scales
// are exact powers of two, undone in the reduce kernel.
//
// Roles (640 threads = 20 warps, 5 per SM sub-partition, one CTA per SM):
//   warp 0      X / mask TMA producer (L2 evict-first),
//   warp 1      residual MMA issuer (+ TMEM owner): runs ahead of the
//               epilogue, bounded only by the S / V / U buffers,
//   warp 2      U / V operand-image producer (L2-resident images, TMA bulk copies),
//   warp 3      reduction MMA issuer: G^T U then G.V of each tile once its G
//               is staged (two issuers keep the tensor pipe fed),
//   warps 4-19  epilogue, two groups of 8 warps that take alternate tiles
//               (group g = tile parity), so one group's math overlaps the
//               other group's wait on the reduction MMAs.  Group g owns buffer
//               set g of S, GA (G in TMEM), the G smem image and GT.
//               Warp (quarter q = warp % 4, half h) handles rows 32q..32q+31
//               and columns 32h..32h+31 of its group's tiles.
// Work: a static, exactly balanced range of tiles per CTA in 2-D super-block
// order; GV accumulates in TMEM over a run of tiles with the same sub-band
// and is drained once per run, GT is drained per tile into a CTA-private slot
// per column tile (store on first touch, then fp32x4 reductions in L2 by the
// thread that owns the address — program order, so deterministic).
// Partials are folded in a fixed order by the reduce kernel.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"

#include <utility>

// Bisection switches for tools/bisect_*.sh, compile-time only (the product
// library is built with 0): 1 skip G^T U stores, 2 skip G.V stores, 8 skip all
// MMAs (pipeline skeleton), 16 / 32 / 64 skip the G^T U / G.V / residual MMAs,
// 128 epilogue ignores MMA completion, 256 drop G^T U stores, 512 store only.
#ifndef SPCP_TC_DEBUG_BITS
#define SPCP_TC_DEBUG_BITS 0
#endif

// 1: the G^T U drain folds the gh / gl halves through shared memory (64-row
// slots, two named barriers per tile); 0: 128-row slots folded by the reduce.
// Measured same-box at C2: 0.372 vs 0.348 ms (the barriers cost more than the
// halved slot traffic saves), so 0.
// 1: the lo piece of the G split by mixed-precision FMAs (fma.rn.f32.f16,
// one per element) instead of fp16 -> fp32 conversions and a packed subtract
#ifndef SPCP_TC_FHFMA
#define SPCP_TC_FHFMA 1
#endif

#ifndef SPCP_TC_GT_FOLD
#define SPCP_TC_GT_FOLD 0
#endif

#ifndef SPCP_TC_GV_FIRST
#define SPCP_TC_GV_FIRST 1
#endif

#ifndef SPCP_TC_XPF
#define SPCP_TC_XPF 0  // X tiles prefetched into L2 ahead of the stage ring (measured: no gain)
#endif

namespace spcp {

struct TcUnit {
  uint16_t sb, tc;
  int32_t gt_slot;
  int32_t gv_slot;  // global run id (consecutive within a CTA)
  uint32_t flags;
};
enum : uint32_t { TCU_FIRST_OF_RUN = 1u, TCU_LAST_OF_RUN = 2u, TCU_FIRST_TOUCH = 4u };

struct TcScales {
  float sigma;       // s_u * s_v: S'' = sigma * L
  float tau_s;       // sigma * tau
  float kappa;       // G'' = kappa * (sigma g)
  float gv_unscale;  // -1 / (kappa sigma s_v)   (partials are gp.V'', gp = -G'')
  float gt_unscale;  // 1 / (kappa sigma s_u)    (gp^T (-U'') = G''^T U'')
  float pad0;
  double phi_unscale;  // 1 / sigma^2
  double su, sv;
  unsigned long long max_bits[2];  // |U|max, |V|max as double bit patterns
};

struct TcParams {
  const TcUnit* units;
  const int32_t* cta_begin;  // [grid + 1]
  const unsigned char* u_img;
  const unsigned char* v_img;
  const TcScales* scales;
  float* pleft;   // [gv_slots][128][kstore]
  float* pright;  // [gt_slots][64][kstore]
  double* pphi;   // [grid]
  int kstore;  // partial row stride (floats): k rounded up to 4
#ifdef SPCP_TC_TIMESTAMPS
  long long* dbg_ts;  // [64][32] per-tile timestamps of CTA 0 (tools/ts_run.sh builds only)
#endif
};

template <int KP16, bool MASK, int SEG = 0>
struct TcCfg {
  // SEG > 0: K-concatenated single images (rank k <= SEG, SEG = round_up(k, 4) <= 32):
  //   U row = [um | uh | uh] and V row = [vh | vm | vh], segments SEG entries
  //   apart, so the residual um.vh + uh.vm + uh.vh is ONE K-sum of 3 SEG
  //   entries (ceil(3 SEG / 16) MMAs), and both reductions read the first two
  //   segments of the same images as N = 2 SEG wide B operands: [um | uh] for
  //   G^T U, [vh | vm] for G.V (the drains add the two halves).  Rows longer
  //   than one 128-byte swizzle atom (3 SEG > 64 entries, k > 20) are stored
  //   as NA K-atoms, atom a of every row at a * rows * 128 bytes; the
  //   reductions only read atom 0.  SEG == 0: two split images [uh|um], [vh|vm].
  static constexpr bool KC = SEG > 0;
  static constexpr int KE = 3 * SEG;
  // REUSE (SEG = 32, k = 21..32): rows store only the first two segments,
  // U = [um | uh], V = [vh | vm] (one 128-byte atom); the residual's third
  // K-segment re-reads uh (TMEM copies) and vh (B descriptors) instead of a
  // stored duplicate, so these ranks keep the one-atom pipeline depths
  static constexpr bool REUSE = KC && SEG % 16 == 0 && 3 * SEG > 64 && 2 * SEG <= 64;
  static constexpr int NA = KC ? (REUSE ? 1 : (KE * 2 + 127) / 128) : 1;  // K-atoms per row
  // gh / gl parts of G^T U summed in the drain (64-row slots): measured a win
  // for the wide REUSE rows (C4: step 0.697 -> 0.661 ms), a loss for SEG <= 20
  // (C2 kernel 0.333 -> 0.365 ms)
  static constexpr bool GT_FOLD = KC && (SPCP_TC_GT_FOLD || REUSE);
  static constexpr int RB = KC ? (NA > 1 ? 128 : (KE <= 16 ? 32 : (KE <= 32 ? 64 : 128)))
                               : KP16 * 2;
  static constexpr uint32_t SWK = RB == 128 ? tc::SW_128 : (RB == 64 ? tc::SW_64 : tc::SW_32);
  static constexpr int NSPLIT = KC ? 1 : 2;
  static constexpr int RT = RB * NSPLIT * NA;  // image bytes per row over all splits / atoms
  static constexpr int NKS = KC ? (KE + 15) / 16 : 0;  // residual K-steps (KC)
  static_assert(!KC || 2 * SEG <= RB / 2, "the reductions' B operand lies in atom 0");
  // X ring (released by the epilogue as soon as it has read the tile), V ring
  // (released when the tile's G.V MMA has finished), U buffers (per run)
#ifndef SPCP_TC_GB
#define SPCP_TC_GB 2
#endif
  static constexpr int GB = SPCP_TC_GB;  // G staging images (1: shared by both groups)
  static constexpr int NST = GB == 1 ? ((RT == 128 && MASK) ? 3 : 4)
                                     : (RT <= 64 ? (MASK ? 3 : 4) : (RT == 128 ? 3 : (MASK ? 2 : 3)));
  static constexpr int NSV = RT == 256 ? 2 : (MASK ? 3 : 4);
  static constexpr int UB = RT == 256 ? 1 : 2;
  static constexpr int LOOKAHEAD = NSV - 1 < 2 ? NSV - 1 : 2;  // residual issue lead (tiles)
  static constexpr int X_BYTES = 128 * 64 * 4;
  static constexpr int V_SPLIT = 64 * RB * NA;  // V_ATOM * NA
  static constexpr int V_ATOM = 64 * RB;
  static constexpr int V_BYTES = NSPLIT * V_SPLIT;
  static constexpr int U_ATOM = 128 * RB;
  static constexpr int U_SPLIT = 128 * RB * NA;
  static constexpr int U_BYTES = NSPLIT * U_SPLIT;
  static constexpr int M_BYTES = MASK ? 128 * 4 * 4 : 0;  // box {4 words, 128 rows}
  static constexpr int G_SPLIT = 128 * 64 * 2;            // one fp16 G image (MN-major SW128)
  static constexpr int G_BYTES = 2 * G_SPLIT;             // gh, gl
  // smem carve (all offsets multiples of 1 KB)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_V = OFF_X + NST * X_BYTES;
  static constexpr int OFF_U = OFF_V + NSV * V_BYTES;
  static constexpr int OFF_G = OFF_U + UB * U_BYTES;
  static constexpr int OFF_M = OFF_G + GB * G_BYTES;
  static constexpr int OFF_BAR = OFF_M + (MASK ? NST * 2048 : 0);
  static constexpr int SMEM = OFF_BAR + 512;  // dynamic smem base is 1 KB aligned
  static_assert(SMEM <= 232448, "shared memory budget");
  // TMEM columns: S [2 x 64] | GV [2 x GVW] | GT [4 x GTW] (two per epilogue
  // group); legacy: the N-concatenated forms hold the [vh|vm] (resp. [uh|um])
  // halves side by side, summed at the drain; KC: the image segments
  static constexpr int GCAT = KP16 <= 32 ? 2 : 1;
  static constexpr int GVC = KP16 <= 32 ? 2 : 1;
  // KC: G.V needs output columns [0, 2 SEG) only ([vh|vm] segments)
  static constexpr int GVW = KC ? ((2 * SEG + 15) / 16) * 16 : GVC * KP16;
  static constexpr int GTW = KC ? GVW : GCAT * KP16;
  // KC: the epilogue overwrites its S columns with G (fp16 pairs: gh at +0,
  // gl at +16 of each warp's 32 columns) and G.V reads A from TMEM; three S
  // buffers (the next writer of a buffer is the other group's tile) and three
  // G^T U accumulators
#ifndef SPCP_TC_NSB
#define SPCP_TC_NSB 3  // measured: 3 (0.339 ms) beats 4 with two G^T U buffers (0.347 ms)
#endif
  static constexpr int NSB = KC ? ((2 * SEG + 15) / 16 * 16 > 48 ? 3 : SPCP_TC_NSB) : 2;
  static_assert(NSB <= 4, "TcBarriers holds four S buffers");
  static constexpr uint32_t T_S = 0, T_GV = 64 * NSB;
  static constexpr uint32_t T_GT = T_GV + 2 * GVW;
  // KC: the run's U image also lives in TMEM (tcgen05.cp, 8 columns per K-step),
  // so the residual is a TS MMA that reads only V from shared memory
  static constexpr int U_COLS = KC ? NKS * 8 : 0;
  // three G^T U accumulators when they fit next to U, else two
  static constexpr int NGT = KC ? ((SPCP_TC_NSB < 4 && T_GT + 3 * GTW + U_COLS <= 512) ? 3 : 2)
                                : 4;
  static constexpr uint32_t T_U = T_GT + NGT * GTW;
  static_assert(T_U + U_COLS <= 512, "TMEM budget");
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr int NEPI = 16;  // epilogue warps: 2 groups x 4 quarters x 2 halves
  static constexpr int NEG = NEPI / 2;
#ifndef SPCP_TC_SPLIT_RED
#define SPCP_TC_SPLIT_RED 0  // measured: no gain
#endif
  static constexpr bool SPLIT_RED = SPCP_TC_SPLIT_RED != 0;
  static constexpr int FIRST_EPI = SPLIT_RED ? 5 : 4;  // warps 0-3: X producer, residual MMA
                                                       // issuer, U/V producer, reduction MMA
                                                       // issuer (G^T U), [4: G.V issuer]
  static constexpr int NTHREADS = 32 * (FIRST_EPI + NEPI);
  // KC drains: output columns [0, SEG) split over the two column-half warps
  static constexpr int CW = KC ? ((SEG / 2 + 3) / 4) * 4 : 0;
};

struct TcBarriers {
  uint64_t stage_full[4], stage_empty[4];
  uint64_t v_full[4], v_empty[4];
  uint64_t u_full[2], u_empty[2];
  uint64_t s_full[4], s_empty[4];
  uint64_t g_full[2], gs_empty[2];  // G image staged (per group) / free (per image)
  uint64_t gt_full[4], gt_empty[4];
  uint64_t gv_full[2], gv_empty[2];
  uint32_t tmem_base;
  double phi[16];
};
static_assert(sizeof(TcBarriers) <= 512, "barrier block exceeds its shared-memory slot");

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int N, typename F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl<N>(f, std::make_integer_sequence<int, N>{});
}

// A warp's window of 32 consecutive schedule entries (one per lane, read back
// with shuffles) plus the next 32 already in flight: schedule reads leave the
// issue paths of the single-warp roles.  get() is warp-uniform and its
// argument never decreases.
struct UnitWindow {
  const uint4* u;
  int T, base;
  uint4 cur, nxt;
  __device__ __forceinline__ uint4 load(int i) const {
    // branch-free (clamped) so the warp stays provably converged for the MMA issue
    return __ldg(u + max(0, min(i, T - 1)));
  }
  __device__ __forceinline__ UnitWindow(const TcUnit* units, int t_count)
      : u(reinterpret_cast<const uint4*>(units)), T(t_count), base(0) {
    const int l = threadIdx.x & 31;
    cur = load(l);
    nxt = load(32 + l);
  }
  __device__ __forceinline__ TcUnit get(int t) {
    while (t >= base + 32) {
      base += 32;
      cur = nxt;
      nxt = load(base + 32 + (threadIdx.x & 31));
    }
    const int src = t - base;
    uint4 w;
    w.x = __shfl_sync(0xffffffffu, cur.x, src);
    w.y = __shfl_sync(0xffffffffu, cur.y, src);
    w.z = __shfl_sync(0xffffffffu, cur.z, src);
    w.w = __shfl_sync(0xffffffffu, cur.w, src);
    return *reinterpret_cast<const TcUnit*>(&w);
  }
};
static_assert(sizeof(TcUnit) == 16, "TcUnit is read as one uint4");

#ifdef SPCP_TC_TIMESTAMPS
#define TC_TS(t, slot)                                                                      \
  do {                                                                                      \
    if (p.dbg_ts && blockIdx.x == 0 && (t) < 64) p.dbg_ts[(t) * 32 + (slot)] = clock64();               \
  } while (0)
#else
#define TC_TS(t, slot) \
  do {                 \
  } while (0)
#endif

// tcgen05.commit from a single lane (legacy issuers) or elected from the whole
// warp (K-concatenated issuers, which run warp-wide)
template <bool WARP>
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  if constexpr (WARP)
    tc::mma_commit_w(bar);
  else
    tc::mma_commit(bar);
}

// Residual MMA issuer (one lane of warp 1): its own function, so ptxas
// allocates it apart from the epilogue and keeps the descriptors uniform.
template <int KP16, bool MASK, int SEG>
__device__ __noinline__ void tc_residual_issuer(unsigned char* sm, TcBarriers* bar,
                                                const TcUnit* units, int T, int run0,
                                                uint32_t tm, const TcParams& p) {
  using C = TcCfg<KP16, MASK, SEG>;
  using namespace tc;
  constexpr uint32_t ID_RES = idesc_f16(128, 64, false, false);
  constexpr int KS = KP16 / 16;
  const bool do_mma = !(SPCP_TC_DEBUG_BITS & 8);
  const uint32_t u0 = smem_u32(sm + C::OFF_U), v0 = smem_u32(sm + C::OFF_V);
  TcUnit un_next = T > 0 ? units[0] : TcUnit{};
  const uint64_t dU_k = umma_desc(u0, 16, 8 * C::RB, C::SWK);  // residual A (K-major)
  const uint64_t dV_k = umma_desc(v0, 16, 8 * C::RB, C::SWK);  // residual B (K-major)
  int prev_run = -1;
  for (int t = 0; t < T; ++t) {
    const TcUnit un = un_next;
    if (t + 1 < T) un_next = units[t + 1];
    const int run = un.gv_slot - run0;
    const int ubuf = run % C::UB;
    if (run != prev_run) {
      mbar_wait(&bar->u_full[ubuf], (run / C::UB) & 1);
      prev_run = run;
      if constexpr (C::KC) {
        // U image -> TMEM (one copy per K-step); in issue order after the
        // previous run's residual MMAs, which read the single TMEM copy
        tc_fence_after();
        const uint64_t du = dU_k + uint64_t(ubuf * (C::U_BYTES >> 4));
        if (do_mma && !(SPCP_TC_DEBUG_BITS & 64)) {
          if constexpr (C::REUSE) {
            static_for<C::NKS>([&](auto I) {  // K-steps 4, 5 repeat uh (steps 2, 3)
              constexpr int src = I < 4 ? int(I) : int(I) - 2;
              tmem_cp_128x256b_w(tm + C::T_U + 8 * I, du + uint64_t(2 * src));
            });
          } else {
            static_for<C::NKS>([&](auto I) {  // K-step I: atom I / 4, 32 B step I % 4
              tmem_cp_128x256b_w(tm + C::T_U + 8 * I,
                                 du + uint64_t((I / 4) * (C::U_ATOM >> 4) + 2 * (I % 4)));
            });
          }
        }
      }
    }
    TC_TS(t, 12);
    const int st = t % C::NSV, b = t % C::NSB;
    mbar_wait(&bar->v_full[st], (t / C::NSV) & 1);
    TC_TS(t, 13);
    mbar_wait(&bar->s_empty[b], ((t / C::NSB) & 1) ^ 1);
    TC_TS(t, 1);
    tc_fence_after();
    const uint64_t da = dU_k + uint64_t(ubuf * (C::U_BYTES >> 4));
    const uint64_t db = dV_k + uint64_t(st * (C::V_BYTES >> 4));
    if (do_mma && !(SPCP_TC_DEBUG_BITS & 64)) {
      // uh.vh + uh.vm + um.vh: product q uses U split (q == 2), V split (q == 1)
      const uint32_t dt = tm + C::T_S + b * 64;
      if constexpr (C::KC) {
        // one K-sum over the concatenated segments: [um|uh|uh] . [vh|vm|vh]
        // (warp-wide batch: one elect, descriptors stepped by 32 B; a second
        // batch for the K-steps in atom 1)
        if constexpr (C::NKS <= 4) {
          mma_ts_batch<C::NKS, 2>(dt, tm + C::T_U, db, ID_RES, 0u);
        } else {
          mma_ts_batch<4, 2>(dt, tm + C::T_U, db, ID_RES, 0u);
          // K-steps 4..: atom 1 of the rows, or (REUSE) vh again
          mma_ts_batch<C::NKS - 4, 2>(dt, tm + C::T_U + 32,
                                      db + uint64_t(C::REUSE ? 0 : (C::V_ATOM >> 4)), ID_RES, 1u);
        }
      } else {
        static_for<3 * KS>([&](auto I) {
          constexpr int q = I / KS, ks = I % KS;
          constexpr int oa = ((q == 2 ? C::U_SPLIT : 0) + ks * 32) >> 4;
          constexpr int ob = ((q == 1 ? C::V_SPLIT : 0) + ks * 32) >> 4;
          mma_ss_1<oa, ob>(dt, da, db, ID_RES, I != 0);
        });
      }
    }
    tc_commit<C::KC>(&bar->s_full[b]);
    tc_commit<C::KC>(&bar->v_empty[st]);
    if (un.flags & TCU_LAST_OF_RUN) tc_commit<C::KC>(&bar->u_empty[ubuf]);
    TC_TS(t, 24);
  }
}

// Reduction MMA issuer (one lane of warp 3): G^T U first (it releases the
// group's G staging image), then G.V.
// ROLE 0: G^T U and G.V of each tile (one issuer); 1: G^T U only; 2: G.V only
// (two reduction issuers, SPCP_TC_SPLIT_RED: each warp blocks on its own MMA
// issue, so the two streams feed the tensor pipe in parallel)
template <int KP16, bool MASK, int SEG, int ROLE>
__device__ __noinline__ void tc_reduction_issuer(unsigned char* sm, TcBarriers* bar,
                                                 const TcUnit* units, int T, int run0,
                                                 uint32_t tm, const TcParams& p) {
  using C = TcCfg<KP16, MASK, SEG>;
  using namespace tc;
  // KC: G^T U stacked to M = 128 (A = [gh; gl], the two G images one N-atom
  // apart), so each K-step is ONE MMA; the accumulator's lanes 64..127 hold the
  // gl part, kept as separate partial rows and summed by the reduce kernel
  constexpr uint32_t ID_GV = idesc_f16(128, C::GVW, false, true);
  constexpr uint32_t ID_GT = idesc_f16(C::KC ? 128 : 64, C::GTW, true, true);
  const bool do_mma = !(SPCP_TC_DEBUG_BITS & 8);
  const uint32_t u0 = smem_u32(sm + C::OFF_U), v0 = smem_u32(sm + C::OFF_V);
  const uint32_t g0 = smem_u32(sm + C::OFF_G);
  TcUnit un_next = T > 0 ? units[0] : TcUnit{};
  // G^T U: A = G image read MN-major (M = 64 tile columns), B = [uh|um]
  const uint64_t dUn0 = umma_desc(u0, (C::GCAT == 2 && !C::KC) ? C::U_SPLIT : 8192, 8 * C::RB, C::SWK);
  const uint64_t dGm = umma_desc(g0, 16384, 1024, SW_128);
  // G.V: the same G image read K-major (M = 128 tile rows, K = tile columns),
  // B = [vh|vm] MN-major
  const uint64_t dGk = umma_desc(g0, 16, 1024, SW_128);
  const uint64_t dVn0 = umma_desc(v0, (C::GVC == 2 && !C::KC) ? C::V_SPLIT : 8192, 8 * C::RB, C::SWK);
  for (int t = 0; t < T; ++t) {
    const TcUnit un = un_next;
    if (t + 1 < T) un_next = units[t + 1];
    const int run = un.gv_slot - run0;
    const int ubuf = run % C::UB, b = t & 1, st = t % C::NSV, gvb = run & 1, gtb = t % C::NGT;
    const bool first = (un.flags & TCU_FIRST_OF_RUN) != 0;
    TC_TS(t, ROLE == 2 ? 26 : 14);
    mbar_wait(&bar->g_full[b], (t >> 1) & 1);
    TC_TS(t, ROLE == 2 ? 27 : 2);
    if (ROLE != 2 && !(SPCP_TC_DEBUG_BITS & 128)) mbar_wait(&bar->gt_empty[gtb], ((t / C::NGT) & 1) ^ 1);
    if (ROLE != 1 && first && !(SPCP_TC_DEBUG_BITS & 128)) mbar_wait(&bar->gv_empty[gvb], ((run >> 1) & 1) ^ 1);
    TC_TS(t, ROLE == 2 ? 28 : 3);
    tc_fence_after();
    const uint64_t dUn = dUn0 + uint64_t(ubuf * (C::U_BYTES >> 4));
    const uint64_t goff = uint64_t((C::GB == 1 ? 0 : b) * (C::G_BYTES >> 4));
    auto issue_gt = [&]() {
    const uint32_t gt = tm + C::T_GT + gtb * C::GTW;
    if (C::KC && ROLE != 2 && do_mma && !(SPCP_TC_DEBUG_BITS & 16)) {
      // stacked [gh; gl]^T U: 8 K-steps of 16 tile rows (A += 2048 B, B += 16 RB)
      mma_ss_batch<8, 128, C::RB>(gt, dGm + goff, dUn, ID_GT, 0u);
    } else if (ROLE != 2 && do_mma && !(SPCP_TC_DEBUG_BITS & 16)) {
      static_for<8>([&](auto I) {
        constexpr int ks = I;
        constexpr int uo = (ks * 16 * C::RB) >> 4, go = (2048 * ks) >> 4;
        constexpr int gl_o = go + (C::G_SPLIT >> 4);
        if constexpr (C::KC) {
          mma_ss_1<go, uo>(gt, dGm + goff, dUn, ID_GT, ks > 0);
        } else if constexpr (C::GCAT == 2) {
          // B = [uh | um]: two N-atoms of the U image (LBO = split stride)
          mma_ss_1<go, uo>(gt, dGm + goff, dUn, ID_GT, ks > 0);
          mma_ss_1<gl_o, uo>(gt, dGm + goff, dUn, ID_GT, 1);
        } else {
          mma_ss_1<go, uo>(gt, dGm + goff, dUn, ID_GT, ks > 0);
          mma_ss_1<go, uo + (C::U_SPLIT >> 4)>(gt, dGm + goff, dUn, ID_GT, 1);
          mma_ss_1<gl_o, uo>(gt, dGm + goff, dUn, ID_GT, 1);
        }
      });
    }
    if (ROLE != 2) tc_commit<C::KC>(&bar->gt_full[gtb]);
    if (C::KC && ROLE != 2) tc_commit<C::KC>(&bar->gs_empty[b]);  // G image: G^T U's operand only
    TC_TS(t, ROLE == 2 ? 29 : 25);
    };
    auto issue_gv = [&]() {
    const uint64_t dVn = dVn0 + uint64_t(st * (C::V_BYTES >> 4));
    const uint32_t gv = tm + C::T_GV + gvb * C::GVW;
    if (C::KC && ROLE != 1 && do_mma && !(SPCP_TC_DEBUG_BITS & 32)) {
      mma_gv_ts_batch<C::RB>(gv, tm + C::T_S + (t % C::NSB) * 64, dVn, ID_GV, first ? 0u : 1u);
    } else if (ROLE != 1 && do_mma && !(SPCP_TC_DEBUG_BITS & 32)) {
      static_for<4>([&](auto I) {
        constexpr int ks = I;
        constexpr int vo = (ks * 16 * C::RB) >> 4;
        constexpr int ao = (32 * ks) >> 4, alo = ao + (C::G_SPLIT >> 4);
        if constexpr (C::KC) {
          // A = G from TMEM (the tile's S columns: 32 per half, gh then gl)
          constexpr int ca = 32 * (ks >> 1) + 8 * (ks & 1);
          const uint32_t sa = tm + C::T_S + (t % C::NSB) * 64 + ca;
          mma_ts_1<vo>(gv, sa, dVn, ID_GV, !(first && ks == 0));
          mma_ts_1<vo>(gv, sa + 16, dVn, ID_GV, 1);
        } else if constexpr (C::GVC == 2) {
          // B = [vh | vm] (N-concatenated), A = gh then gl (K-step of 16 columns)
          mma_ss_1<ao, vo>(gv, dGk + goff, dVn, ID_GV, !(first && ks == 0));
          mma_ss_1<alo, vo>(gv, dGk + goff, dVn, ID_GV, 1);
        } else {
          mma_ss_1<ao, vo>(gv, dGk + goff, dVn, ID_GV, !(first && ks == 0));
          mma_ss_1<ao, vo + (C::V_SPLIT >> 4)>(gv, dGk + goff, dVn, ID_GV, 1);
          mma_ss_1<alo, vo>(gv, dGk + goff, dVn, ID_GV, 1);
        }
      });
    }
    if (!C::KC) mma_commit(&bar->gs_empty[b]);  // per tile parity (see the epilogue's wait)
    else if (ROLE != 1) tc_commit<C::KC>(&bar->s_empty[t % C::NSB]);  // S / G columns
    if (ROLE != 1) tc_commit<C::KC>(&bar->v_empty[st]);
    };
    // KC + SPCP_TC_GV_FIRST: G.V first (its completion frees the tile's S
    // columns for the residual of tile t + NSB), then G^T U (frees the G image)
    if constexpr (C::KC && SPCP_TC_GV_FIRST) {
      issue_gv();
      issue_gt();
    } else {
      issue_gt();
      issue_gv();
    }
    if (un.flags & TCU_LAST_OF_RUN) {
      if (ROLE != 1) tc_commit<C::KC>(&bar->gv_full[gvb]);
      if (ROLE != 2) tc_commit<C::KC>(&bar->u_empty[ubuf]);
    }
    TC_TS(t, ROLE == 2 ? 30 : 15);
  }
  // decoupled-timing mode: nobody else waited for the last reductions
  if ((SPCP_TC_DEBUG_BITS & 128) && T > 0) mbar_wait(&bar->gs_empty[(T - 1) & 1], ((T - 1) >> 1) & 1);
}

template <int KP16, bool MASK, int SEG = 0>
__global__ void __launch_bounds__(TcCfg<KP16, MASK, SEG>::NTHREADS, 1)
    tc_eval_kernel(const __grid_constant__ CUtensorMap xmap,
                   const __grid_constant__ CUtensorMap mmap, const TcParams p) {
  using C = TcCfg<KP16, MASK, SEG>;
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* sm = smem_dyn;
  if ((smem_u32(sm) & 1023u) != 0u) __trap();  // swizzled TMA/UMMA images need 1 KB alignment
  TcBarriers* bar = reinterpret_cast<TcBarriers*>(sm + C::OFF_BAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ub = p.cta_begin[blockIdx.x], ue = p.cta_begin[blockIdx.x + 1];
  const int T = ue - ub;
  const TcUnit* units = p.units + ub;
  const int run0 = T > 0 ? units[0].gv_slot : 0;  // CTA-local run index = gv_slot - run0
  pdl_wait();  // the operand images / scales of this evaluation are complete
  pdl_launch_next();  // the reduce kernel's CTAs queue for the SMs as they free up
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // the image pass (the only reader of the maxima) has completed: reset them
    // for the next evaluation's max pass instead of a separate memset
    TcScales* scw = const_cast<TcScales*>(p.scales);
    scw->max_bits[0] = 0ull;
    scw->max_bits[1] = 0ull;
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NST; ++i) {
      mbar_init(&bar->stage_full[i], 1);
      mbar_init(&bar->stage_empty[i], C::NEG);
    }
    for (int i = 0; i < C::NSV; ++i) {
      mbar_init(&bar->v_full[i], 1);
      mbar_init(&bar->v_empty[i], 2);  // residual + G.V issuers
    }
    for (int i = 0; i < C::NSB; ++i) {
      mbar_init(&bar->s_full[i], 1);
      mbar_init(&bar->s_empty[i], C::KC ? 1 : C::NEG);  // KC: G.V commit; else epilogue
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar->u_full[i], 1);
      mbar_init(&bar->u_empty[i], 2);  // residual + G^T U issuers
      mbar_init(&bar->g_full[i], C::NEG);
      mbar_init(&bar->gs_empty[i], (C::SPLIT_RED && !C::KC) ? 2 : 1);
      mbar_init(&bar->gv_full[i], 1);
      mbar_init(&bar->gv_empty[i], C::NEG);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bar->gt_full[i], 1);
      mbar_init(&bar->gt_empty[i], C::NEG);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&bar->tmem_base, C::TMEM_COLS);
  if (warp == 0 && lane == 0) {
    prefetch_tensormap(&xmap);
    if (MASK) prefetch_tensormap(&mmap);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // broadcast from lane 0: provably warp-uniform, so MMA operands stay in uniform registers
  const uint32_t tm = __shfl_sync(0xffffffffu, bar->tmem_base, 0);

  if (warp == 0) {
    // ======================= X / mask producer (TMA) ====================
    // X tiles are also prefetched into L2 PF tiles ahead of their shared-
    // memory load: the bytes in flight needed to cover HBM latency then live
    // in L2 rather than in the (small) stage ring
    constexpr int PF = SPCP_TC_XPF;
    UnitWindow uw(units, T), uwp(units, T);
    const uint64_t pol_x = policy_evict_first();
    for (int tp = 0; tp < PF; ++tp) {
      const TcUnit up = uwp.get(tp);
      if (lane == 0 && tp < T) {
        tma_prefetch_2d(&xmap, int(up.tc) * 64, int(up.sb) * 128);
        tma_prefetch_2d(&xmap, int(up.tc) * 64 + 32, int(up.sb) * 128);
      }
    }
    for (int t = 0; t < T; ++t) {
      const TcUnit un = uw.get(t);
      if (PF > 0) {
        const TcUnit up = uwp.get(t + PF);
        if (lane == 0 && t + PF < T) {
          tma_prefetch_2d(&xmap, int(up.tc) * 64, int(up.sb) * 128);
          tma_prefetch_2d(&xmap, int(up.tc) * 64 + 32, int(up.sb) * 128);
        }
      }
      if (lane == 0) {
        const int st = t % C::NST;
        mbar_wait(&bar->stage_empty[st], ((t / C::NST) & 1) ^ 1);
        TC_TS(t, 0);
#ifdef SPCP_TC_BISECT_NO_TMA
        mbar_arrive(&bar->stage_full[st]);
        if (st >= 0) goto x_done;
#endif
        mbar_arrive_expect_tx(&bar->stage_full[st], C::X_BYTES + C::M_BYTES);
        unsigned char* xs = sm + C::OFF_X + st * C::X_BYTES;
        tma_load_2d_hint(xs, &xmap, int(un.tc) * 64, int(un.sb) * 128, &bar->stage_full[st],
                         pol_x);
        tma_load_2d_hint(xs + 16384, &xmap, int(un.tc) * 64 + 32, int(un.sb) * 128,
                         &bar->stage_full[st], pol_x);
        if (MASK)
          tma_load_2d_hint(sm + C::OFF_M + st * 2048, &mmap, (int(un.tc) * 2) & ~3,
                           int(un.sb) * 128, &bar->stage_full[st], pol_x);
      }
#ifdef SPCP_TC_BISECT_NO_TMA
    x_done:
#endif
      __syncwarp();
    }
  } else if (warp == 2) {
    // ======================= U / V operand-image producer (bulk copies) ==
    // Asynchronous TMA bulk copies of the L2-resident images: several stay in
    // flight, so their latency is hidden by the V ring and the U buffers.
    if (lane == 0) {
      int prev_run = -1;
      TcUnit un_next = T > 0 ? units[0] : TcUnit{};
      for (int t = 0; t < T; ++t) {
        const TcUnit un = un_next;
        if (t + 1 < T) un_next = units[t + 1];
        const int run = un.gv_slot - run0;
        if (run != prev_run) {
          const int b = run % C::UB;
          mbar_wait(&bar->u_empty[b], ((run / C::UB) & 1) ^ 1);
          mbar_arrive_expect_tx(&bar->u_full[b], C::U_BYTES);
          bulk_load(sm + C::OFF_U + b * C::U_BYTES, p.u_img + size_t(un.sb) * C::U_BYTES,
                    C::U_BYTES, &bar->u_full[b]);
          prev_run = run;
        }
        const int sv = t % C::NSV;
        mbar_wait(&bar->v_empty[sv], ((t / C::NSV) & 1) ^ 1);
        TC_TS(t, 11);
        mbar_arrive_expect_tx(&bar->v_full[sv], C::V_BYTES);
        bulk_load(sm + C::OFF_V + sv * C::V_BYTES, p.v_img + size_t(un.tc) * C::V_BYTES,
                  C::V_BYTES, &bar->v_full[sv]);
      }
    }
  } else if (warp == 1 || warp == 3 || (C::SPLIT_RED && warp == 4)) {
    // ======================= MMA issuers ================================
    // Two warps issue into the one tensor pipe, each on a single lane (no
    // elect: ptxas keeps the descriptors on the uniform datapath, ~6
    // instructions per MMA): warp 1 the residual of every tile (runs ahead,
    // bounded only by the S / V / U buffers), warp 3 the reductions (G^T U,
    // then G.V) of each tile once its G is staged.  Base descriptors are built
    // once; every MMA adds a compile-time offset (descriptor address field =
    // byte address >> 4, no carry for shared memory).
    // (K-concatenated layout: the whole warp runs the issuer, one elect per batch)
    if (C::KC || lane == 0) {
      if (warp == 1)
        tc_residual_issuer<KP16, MASK, SEG>(sm, bar, units, T, run0, tm, p);
      else if (!C::SPLIT_RED)
        tc_reduction_issuer<KP16, MASK, SEG, 0>(sm, bar, units, T, run0, tm, p);
      else if (warp == 3)
        tc_reduction_issuer<KP16, MASK, SEG, 1>(sm, bar, units, T, run0, tm, p);
      else
        tc_reduction_issuer<KP16, MASK, SEG, 2>(sm, bar, units, T, run0, tm, p);
    }
  } else {
    // ======================= epilogue warps =============================
    const int q = warp & 3;               // TMEM lane quarter
    const int e = warp - C::FIRST_EPI;
    const int grp = (e >> 2) & 1;         // tile parity this warp serves
    const int h = e >> 3;                 // column half of the tile
    const int row = 32 * q + lane;
    const uint32_t lane_addr = uint32_t(32 * q) << 16;
    const TcScales sc = *p.scales;
    const float sigma = sc.sigma, tau_s = sc.tau_s, kappa = sc.kappa;
    const float2 sig2 = make_float2(sigma, sigma), kap2 = make_float2(kappa, kappa);
    const float2 nhalf2 = make_float2(-0.5f, -0.5f);
    double phi_acc = 0.0;
    constexpr int GTC = KP16 / 2;  // accumulator columns drained per warp (of KP16)
    const int kst = p.kstore;      // partial row stride: k rounded up to 4 (<= KP16)
    unsigned char* gimg = sm + C::OFF_G + (C::GB == 1 ? 0 : grp) * C::G_BYTES;

    // G^T U of tile t2 (this group's previous tile) -> CTA-private slot
    auto drain_gt = [&](int t2, const TcUnit& u2) {
      const int b = t2 % C::NGT;
      if (!(SPCP_TC_DEBUG_BITS & 128)) mbar_wait(&bar->gt_full[b], (t2 / C::NGT) & 1);
      tc_fence_after();
      if constexpr (C::KC) {
        if (!(SPCP_TC_DEBUG_BITS & 1)) {
          if constexpr (C::GT_FOLD) {
          // M = 128 stacked accumulator: lanes 0..63 hold the gh part of tile
          // columns 0..63, lanes 64..127 the gl part; output column c = D[c]
          // (um) + D[SEG + c] (uh).  Quarters 2, 3 park their gl part in the
          // group's G image (free: its last reader, this tile's G^T U, has
          // completed), quarters 0, 1 add it to the gh part (fixed order) and
          // write 64-row slots: half the slot bytes, half the L2 reductions
          // and half the reduce kernel's gather of a 128-row slot.
          // slot layout [kst / 4][64 rows][4]: a warp's float4 stores cover 512
          // contiguous bytes (coalesced)
          constexpr int NC = C::CW / 4;
          const bool hi_q = q >= 2;
          const int r64 = 32 * (q & 1) + lane;
          float* xb = reinterpret_cast<float*>(gimg);  // [SEG / 4][64 rows][4]
          float* dst = p.pright + size_t(u2.gt_slot) * 64 * kst + r64 * 4;
          const bool first = (u2.flags & TCU_FIRST_TOUCH) != 0;
          const uint32_t col = tm + lane_addr + C::T_GT + b * C::GTW;
          float4 o[NC];
          static_for<NC>([&](auto I) {
            constexpr int c = I * 4;
            const int cc = h * C::CW + c;
            if (cc < SEG) {  // warp-uniform
              uint32_t v[4], w[4];
              tmem_ld4(col + cc, v);
              tmem_ld4(col + SEG + cc, w);
              tmem_wait_ld();
              o[I] = make_float4(__uint_as_float(v[0]) + __uint_as_float(w[0]),
                                 __uint_as_float(v[1]) + __uint_as_float(w[1]),
                                 __uint_as_float(v[2]) + __uint_as_float(w[2]),
                                 __uint_as_float(v[3]) + __uint_as_float(w[3]));
              if (hi_q) *reinterpret_cast<float4*>(xb + (cc * 64 + r64 * 4)) = o[I];
            }
          });
          named_bar_sync(1 + grp, 32 * C::NEG);  // gl parts parked
          if (!hi_q) {
            static_for<NC>([&](auto I) {
              constexpr int c = I * 4;
              const int cc = h * C::CW + c;
              if (cc < SEG) {
                const float4 l4 = *reinterpret_cast<const float4*>(xb + (cc * 64 + r64 * 4));
                const float4 s4 = make_float4(o[I].x + l4.x, o[I].y + l4.y, o[I].z + l4.z,
                                              o[I].w + l4.w);
                float* d4 = dst + cc * 64;  // chunk cc / 4 of 64 rows x 4
                if (first)
                  *reinterpret_cast<float4*>(d4) = s4;
                else
                  red_add_v4(d4, __float_as_uint(s4.x), __float_as_uint(s4.y),
                             __float_as_uint(s4.z), __float_as_uint(s4.w));
              }
            });
          }
          named_bar_sync(1 + grp, 32 * C::NEG);  // read before G(t) reuses the image
} else {
          // M = 128 stacked accumulator: lane = slot row (0..63 gh part, 64..127 gl
          // part), kept as separate 128-row slots (summed by the reduce kernel);
          // output column c = D[c] (um) + D[SEG + c] (uh)
          float* dst = p.pright + size_t(u2.gt_slot) * 128 * kst + (32 * q + lane) * 4;
          const bool first = (u2.flags & TCU_FIRST_TOUCH) != 0;
          const uint32_t col = tm + lane_addr + C::T_GT + b * C::GTW;
          static_for<C::CW / 4>([&](auto I) {
            constexpr int c = I * 4;
            const int cc = h * C::CW + c;
            if (cc < SEG) {  // warp-uniform
              uint32_t v[4], w[4];
              tmem_ld4(col + cc, v);
              tmem_ld4(col + SEG + cc, w);
              tmem_wait_ld();
              const float4 o = make_float4(__uint_as_float(v[0]) + __uint_as_float(w[0]),
                                           __uint_as_float(v[1]) + __uint_as_float(w[1]),
                                           __uint_as_float(v[2]) + __uint_as_float(w[2]),
                                           __uint_as_float(v[3]) + __uint_as_float(w[3]));
              float* d4 = dst + cc * 128;  // chunk cc / 4 of 128 rows x 4
              if (first)
                *reinterpret_cast<float4*>(d4) = o;
              else
                red_add_v4(d4, __float_as_uint(o.x), __float_as_uint(o.y), __float_as_uint(o.z),
                           __float_as_uint(o.w));
            }
          });
}
        }
      } else if (!(SPCP_TC_DEBUG_BITS & 1)) {
        // chunked slot [kst / 4][64 rows][4] (coalesced float4 stores)
        float* dst = p.pright + size_t(u2.gt_slot) * 64 * kst + (16 * q + lane) * 4;
        const bool first = (u2.flags & TCU_FIRST_TOUCH) != 0;
        constexpr int CH = GTC < 16 ? GTC : 16;
#pragma unroll
        for (int c0 = 0; c0 < GTC; c0 += CH) {
          uint32_t v[CH], w[CH];
          const uint32_t col = tm + lane_addr + C::T_GT + b * C::GTW + h * GTC + c0;
          tmem_ldn<CH>(col, v);
          if constexpr (C::GCAT == 2) {
            tmem_ldn<CH>(col + KP16, w);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < CH; ++c)
              v[c] = __float_as_uint(__uint_as_float(v[c]) + __uint_as_float(w[c]));
          } else {
            tmem_wait_ld();
          }
          if (lane < 16) {  // M = 64 accumulator: row j = 16 q + lane in lanes 0..15
#pragma unroll
            for (int c = 0; c < CH; c += 4) {
              const int cc = h * GTC + c0 + c;
              if (cc >= kst) continue;  // padded rank columns are not stored
              if (first)
                *reinterpret_cast<uint4*>(dst + cc * 64) =
                    make_uint4(v[c], v[c + 1], v[c + 2], v[c + 3]);
              else
                red_add_v4(dst + cc * 64, v[c], v[c + 1], v[c + 2], v[c + 3]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar->gt_empty[b]);
    };

    // G.V of a finished run -> its slot (M = 128: row = TMEM lane)
    auto drain_gv = [&](const TcUnit& u2) {
      const int run = u2.gv_slot - run0;
      const int gvb = run & 1;
      if (!(SPCP_TC_DEBUG_BITS & 128)) mbar_wait(&bar->gv_full[gvb], (run >> 1) & 1);
      tc_fence_after();
      if constexpr (C::KC) {
        if (!(SPCP_TC_DEBUG_BITS & 2)) {
          // output column c = D[c] (vh) + D[SEG + c] (vm)
          float* dst = p.pleft + size_t(u2.gv_slot) * 128 * kst + row * 4;  // [kst/4][128][4]
          const uint32_t col = tm + lane_addr + C::T_GV + gvb * C::GVW;
          static_for<C::CW / 4>([&](auto I) {
            constexpr int c = I * 4;
            const int cc = h * C::CW + c;
            if (cc < SEG) {
              uint32_t v[4], w[4];
              tmem_ld4(col + cc, v);
              tmem_ld4(col + SEG + cc, w);
              tmem_wait_ld();
              *reinterpret_cast<float4*>(dst + cc * 128) =
                  make_float4(__uint_as_float(v[0]) + __uint_as_float(w[0]),
                              __uint_as_float(v[1]) + __uint_as_float(w[1]),
                              __uint_as_float(v[2]) + __uint_as_float(w[2]),
                              __uint_as_float(v[3]) + __uint_as_float(w[3]));
            }
          });
        }
      } else if (!(SPCP_TC_DEBUG_BITS & 2)) {
        float* dst = p.pleft + size_t(u2.gv_slot) * 128 * kst + row * 4;  // [kst/4][128][4]
        constexpr int CH = GTC < 16 ? GTC : 16;
#pragma unroll
        for (int c0 = 0; c0 < GTC; c0 += CH) {
          uint32_t v[CH], w[CH];
          const uint32_t col = tm + lane_addr + C::T_GV + gvb * C::GVW + h * GTC + c0;
          tmem_ldn<CH>(col, v);
          if constexpr (C::GVC == 2) {
            tmem_ldn<CH>(col + KP16, w);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < CH; ++c)
              v[c] = __float_as_uint(__uint_as_float(v[c]) + __uint_as_float(w[c]));
          } else {
            tmem_wait_ld();
          }
#pragma unroll
          for (int c = 0; c < CH; c += 4)
            if (h * GTC + c0 + c < kst)
              *reinterpret_cast<uint4*>(dst + (h * GTC + c0 + c) * 128) =
                  make_uint4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar->gv_empty[gvb]);
    };

    TcUnit prev{};
    TcUnit un_next = grp < T ? units[grp] : TcUnit{};
    for (int t = grp; t < T; t += 2) {
      const TcUnit un = un_next;
      if (t + 2 < T) un_next = units[t + 2];  // consumed next iteration: latency hidden
      const int st = t % C::NST, b = grp, sbuf = t % C::NSB;
      const bool ts_w = ((e == 0 || e == 4) && lane == 0);
      if (ts_w) TC_TS(t, 4);
      // ---- S tile and X tile (32 columns: two chunks of 16)
      mbar_wait(&bar->s_full[sbuf], (t / C::NSB) & 1);
      if (ts_w) TC_TS(t, 5);
      tc_fence_after();
      mbar_wait(&bar->stage_full[st], (t / C::NST) & 1);
      if (ts_w) TC_TS(t, 6);
      const unsigned char* xs = sm + C::OFF_X + st * C::X_BYTES + h * 16384;
      uint32_t mw = 0xffffffffu;
      if (MASK)
        mw = reinterpret_cast<const uint32_t*>(sm + C::OFF_M + st * 2048)[row * 4 +
                                                                        (un.tc & 1) * 2 + h];
      uint32_t hi[16], lo[16];
      float2 hs2 = make_float2(0.f, 0.f);
#ifdef SPCP_TC_EPI_PAD
      // sensitivity probe: extra FFMA2s per pair into hs2 with a runtime zero
      // (TcScales::pad0 = 0), no extra live registers, results unchanged
      const float2 pad2 = make_float2(sc.pad0, sc.pad0);
#endif
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t sv[16];
#if defined(SPCP_TC_BISECT_EPI_SKIP)
#pragma unroll
        for (int c = 0; c < 16; ++c) sv[c] = c;
#else
        tmem_ldn<16>(tm + lane_addr + C::T_S + sbuf * 64 + 32 * h + 16 * ch, sv);
#endif
        float xv[16];
#if defined(SPCP_TC_BISECT_EPI_SKIP) || defined(SPCP_TC_BISECT_NO_SMEM)
#pragma unroll
        for (int c = 0; c < 16; ++c) xv[c] = __uint_as_float(sv[c] ^ lane);
#else
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 f = lds128(xs + Swz<128>::offset(row, (4 * ch + c) * 16));
          xv[4 * c] = f.x;
          xv[4 * c + 1] = f.y;
          xv[4 * c + 2] = f.z;
          xv[4 * c + 3] = f.w;
        }
#endif
        tmem_wait_ld();
        if (ch == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (!C::KC) mbar_arrive(&bar->s_empty[sbuf]);
            mbar_arrive(&bar->stage_empty[st]);
          }
        }
        // The MMA produced S'' = -sigma L (U image negated), so r'' = sigma r =
        // fma(x, sigma, S'').  cs = clamp(r'', +-tau''), huber'' = cs (r'' - cs/2)
        // (quadratic on ties, as the reference), gp = kappa cs = -G'' (|gp| <
        // 2^14), split in floating point: hi = fp16(gp), lo = fp16(gp - hi), so
        // gp = hi + lo to 2^-22 of |gp| for every entry (a fixed-quantum split
        // was exact only relative to tau: residuals far below tau, the noise at
        // a good iterate, lost ~1e-5 of their value).
#pragma unroll
        for (int e2 = 0; e2 < 16; e2 += 2) {
          float2 r2 = ffma2(make_float2(xv[e2], xv[e2 + 1]), sig2,
                            make_float2(__uint_as_float(sv[e2]), __uint_as_float(sv[e2 + 1])));
          if (MASK) {
            r2.x = ((mw >> (16 * ch + e2)) & 1u) ? r2.x : 0.f;
            r2.y = ((mw >> (16 * ch + e2 + 1)) & 1u) ? r2.y : 0.f;
          }
          const float2 cs2 = make_float2(fminf(fmaxf(r2.x, -tau_s), tau_s),
                                         fminf(fmaxf(r2.y, -tau_s), tau_s));
          hs2 = ffma2(cs2, ffma2(nhalf2, cs2, r2), hs2);
#ifdef SPCP_TC_EPI_PAD
#pragma unroll
          for (int pp = 0; pp < SPCP_TC_EPI_PAD; ++pp) hs2 = ffma2(r2, pad2, hs2);
#endif
          const float2 gp2 = fmul2(cs2, kap2);
          const __half2 hh2 = __float22half2_rn(gp2);
#if SPCP_TC_FHFMA
          const float2 lo2 = sub_half2_from(gp2, *reinterpret_cast<const uint32_t*>(&hh2));
#else
          const float2 lo2 = fsub2(gp2, __half22float2(hh2));
#endif
          hi[8 * ch + (e2 >> 1)] = *reinterpret_cast<const uint32_t*>(&hh2);
          lo[8 * ch + (e2 >> 1)] = pack_half2(lo2.x, lo2.y);
        }
      }
      phi_acc += double(hs2.x) + double(hs2.y);
      if constexpr (C::KC) {
        // G over this warp's own S columns: the A operand of the TS G.V MMA
        const uint32_t gcol = tm + lane_addr + C::T_S + sbuf * 64 + 32 * h;
        tmem_st16(gcol, hi);
        tmem_st16(gcol + 16, lo);
      }
      if (ts_w) TC_TS(t, 7);
      if (ts_w) TC_TS(t, 8);
      // ---- G to smem: A of both G^T.U (MN-major view) and G.V (K-major view)
      if (C::GB == 1) {
        // one image shared by both groups: wait for tile t-1's reductions
        // (the other parity's barrier, phase (t-1)/2; in-order MMA completion
        // covers tile t-2).  Per-parity barriers never lag two phases behind.
        if (t >= 1) mbar_wait(&bar->gs_empty[(t - 1) & 1], ((t - 1) >> 1) & 1);
      } else if (!(SPCP_TC_DEBUG_BITS & 128)) {
        mbar_wait(&bar->gs_empty[b], ((t >> 1) & 1) ^ 1);
      }
      if (ts_w) TC_TS(t, 9);
      // KC: drain G^T U of this group's previous tile BEFORE handing over G(t).
      // Its completion is the event just waited for (gs_empty is committed right
      // after G^T U), so this adds no wait; in exchange the accumulator is free
      // before the reduction issuer can reach tile t (two G^T U buffers suffice,
      // and the issuer never waits on gt_empty).
      if constexpr (C::KC) {
        if (t >= 2) drain_gt(t - 2, prev);
      }
#if defined(SPCP_TC_BISECT_EPI_SKIP)
      if (hi[0] == 0x12345 && lo[3] == 0x777) phi_acc += 1.0;  // keep the math alive
#endif
#if !defined(SPCP_TC_BISECT_EPI_SKIP) && !defined(SPCP_TC_BISECT_NO_SMEM)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t o = Swz<128>::offset(row, 64 * h + 16 * c);
        *reinterpret_cast<uint4*>(gimg + o) =
            make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
        *reinterpret_cast<uint4*>(gimg + C::G_SPLIT + o) =
            make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
      }
#endif
      fence_proxy_async_smem();
      if constexpr (C::KC) {
        tmem_wait_st();
        tc_fence_before();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar->g_full[b]);
      if (ts_w) TC_TS(t, 10);
      if (lane == 0) TC_TS(t, 16 + (e & 3) + 4 * h);  // per-warp arrival: quarter + 4 * half
      // ---- deferred drains of this group's previous tile (off the G hand-off
      // path: G^T U accumulators are double-buffered per group)
      if (t >= 2) {
        if constexpr (!C::KC) drain_gt(t - 2, prev);
        if (prev.flags & TCU_LAST_OF_RUN) drain_gv(prev);
      }
      prev = un;
    }
    // flush: this group's last tile
    const int tl = ((T - 1 - grp) >= 0) ? (T - 1 - ((T - 1 - grp) & 1)) : -1;
    if (tl >= 0) {
      drain_gt(tl, prev);
      if (prev.flags & TCU_LAST_OF_RUN) drain_gv(prev);
    }
    // phi: per-thread fp64, fold over the epilogue warps in a fixed order
    double w = warp_sum(phi_acc);
    if (lane == 0) bar->phi[e] = w;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < C::NEPI; ++i) s += bar->phi[i];
    p.pphi[blockIdx.x] = s * p.scales->phi_unscale;
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tm, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ prep
// pass 1: max |w| over the U and V parts of the trial point (bit patterns of
// non-negative doubles order like unsigned integers).
// Per-block maxima go to bmax[2 b], bmax[2 b + 1] (plain stores: hundreds of
// blocks hitting two addresses with atomicMax serialised in L2 and cost more
// than the loads); the image pass folds them.
constexpr int kTcMaxBlocks = 296;
__global__ void __launch_bounds__(256) tc_max_kernel(const double* __restrict__ z,
                                                     const double* __restrict__ dz, double alpha,
                                                     int64_t nu, int64_t nv,
                                                     unsigned long long* bmax) {
  tc::pdl_wait();
  tc::pdl_launch_next();
  unsigned long long mu = 0, mv = 0;
  const int64_t tot = nu + nv, stride = int64_t(gridDim.x) * blockDim.x;
  // four elements per thread per sweep, all loads in flight before the maxima
  for (int64_t q0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q0 < tot;
       q0 += 4 * stride) {
    double zv[4], dv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t q = q0 + u * stride;
      zv[u] = q < tot ? __ldg(z + q) : 0.0;
      dv[u] = (dz && q < tot) ? __ldg(dz + q) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t q = q0 + u * stride;
      double w = zv[u];
      if (dz) w += alpha * dv[u];
      const unsigned long long bits = q < tot ? __double_as_longlong(fabs(w)) : 0ull;
      if (q < nu)
        mu = bits > mu ? bits : mu;
      else
        mv = bits > mv ? bits : mv;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mu, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, mv, o);
    mu = a > mu ? a : mu;
    mv = b > mv ? b : mv;
  }
  __shared__ unsigned long long wm[2][8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    wm[0][w] = mu;
    wm[1][w] = mv;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    unsigned long long m = 0ull;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) m = wm[threadIdx.x][i] > m ? wm[threadIdx.x][i] : m;
    bmax[2 * blockIdx.x + threadIdx.x] = m;
  }
}

// fold of tc_max_kernel's per-block maxima, done by every block of the image
// pass (2 x nblk loads, L2-resident); result in all threads
__device__ __forceinline__ void tc_fold_max(const unsigned long long* __restrict__ bmax, int nblk,
                                            double& mu, double& mv) {
  __shared__ unsigned long long red[2][8];
  unsigned long long a = 0ull, b = 0ull;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    const unsigned long long x = __ldcg(bmax + 2 * i), y = __ldcg(bmax + 2 * i + 1);
    a = x > a ? x : a;
    b = y > b ? y : b;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, a, o);
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, b, o);
    a = x > a ? x : a;
    b = y > b ? y : b;
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a;
    red[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  a = b = 0ull;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) {
    a = red[0][i] > a ? red[0][i] : a;
    b = red[1][i] > b ? red[1][i] : b;
  }
  mu = __longlong_as_double(a);
  mv = __longlong_as_double(b);
}

// pass 2 (folded into the image pass): power-of-two scales from the maxima
__device__ __forceinline__ TcScales tc_compute_scales(double mu, double mv, double tau) {
  auto pow2_for = [](double mx) {  // largest 2^e with mx * 2^e <= 2^14
    if (!(mx > 0.0)) return 1.0;
    int e;
    frexp(mx, &e);  // mx = f * 2^e, f in [0.5, 1)
    return ldexp(1.0, 14 - e);
  };
  TcScales r{};
  const double su = pow2_for(mu), sv = pow2_for(mv);
  const double sigma = su * sv;
  const double taus = sigma * tau;
  int e;
  frexp(taus, &e);
  const double kappa = ldexp(1.0, 14 - e);
  r.su = su;
  r.sv = sv;
  r.sigma = float(sigma);
  r.tau_s = float(taus);
  r.kappa = float(kappa);
  r.gv_unscale = float(-1.0 / (kappa * sigma * sv));  // G.V partials carry gp = -G''
  r.gt_unscale = float(1.0 / (kappa * sigma * su));
  r.phi_unscale = 1.0 / (sigma * sigma);
  return r;
}

template <int RB>
__device__ __forceinline__ void split2_store(unsigned char* base, int split_bytes, int row, int c,
                                             double x) {
  const __half h = __double2half(x);
  const __half m = __double2half(x - double(__half2float(h)));
  const uint32_t o = tc::Swz<RB>::offset(row, c * 2);
  *reinterpret_cast<__half*>(base + o) = h;
  *reinterpret_cast<__half*>(base + split_bytes + o) = m;
}

// pass 3: fp16 two-way split images of U (per 128-row sub-band) and V (per 64-row tile)
template <int KP16>
__global__ void tc_images_kernel(const double* __restrict__ z, const double* __restrict__ dz,
                                 double alpha, int64_t m, int64_t n, int64_t k, int64_t m_pad,
                                 int64_t n_pad, TcScales* sc, double tau, unsigned char* u_img,
                                 unsigned char* v_img, const unsigned long long* bmax, int nbmax) {
  constexpr int RB = KP16 * 2;
  double mu, mv;
  tc_fold_max(bmax, nbmax, mu, mv);
  const TcScales scl = tc_compute_scales(mu, mv, tau);  // every block: same maxima, same scales
  const double su = scl.su, sv = scl.sv;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // publish for the fused kernel and the reduce
    sc->su = scl.su;
    sc->sv = scl.sv;
    sc->sigma = scl.sigma;
    sc->tau_s = scl.tau_s;
    sc->kappa = scl.kappa;
    sc->gv_unscale = scl.gv_unscale;
    sc->gt_unscale = scl.gt_unscale;
    sc->phi_unscale = scl.phi_unscale;
  }
  const int64_t total = (m_pad + n_pad) * KP16;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = q / KP16;
    const int c = int(q % KP16);
    if (row < m_pad) {
      double w = 0.0;
      if (row < m && c < k) {
        const int64_t o = row * k + c;
        w = z[o] + (dz ? alpha * dz[o] : 0.0);
      }
      const int64_t sb = row >> 7;
      // U is stored negated: the residual MMA then yields -sigma L directly
      split2_store<RB>(u_img + sb * (2 * 128 * RB), 128 * RB, int(row & 127), c, -w * su);
    } else {
      const int64_t j = row - m_pad;
      double w = 0.0;
      if (j < n && c < k) {
        const int64_t o = m * k + j * k + c;
        w = z[o] + (dz ? alpha * dz[o] : 0.0);
      }
      const int64_t tcol = j >> 6;
      split2_store<RB>(v_img + tcol * (2 * 64 * RB), 64 * RB, int(j & 63), c, w * sv);
    }
  }
}

// pass 3 (K-concatenated layout, TcCfg<.., SEG>::KC): one fp16 image per 128-row
// sub-band of U, rows [um | uh | uh | 0] (U negated, as above), and per 64-row
// tile of V, rows [vh | vm | vh | 0]; entry e of a row lives in K-atom
// e / (RB / 2) (atoms of all rows stored one after another)
template <int SEG>
__device__ __forceinline__ void tc_images_kc_body(const double* __restrict__ z,
                                                  const double* __restrict__ dz, double alpha,
                                                  int64_t m, int64_t n, int64_t k, int64_t m_pad,
                                                  int64_t n_pad, TcScales* sc, double tau,
                                                  unsigned char* u_img, unsigned char* v_img,
                                                  double mu, double mv) {
  using C = TcCfg<16, false, SEG>;
  constexpr int RB = C::RB, EPA = RB / 2, NE = C::NA * EPA;  // entries per atom / per row
  const TcScales scl = tc_compute_scales(mu, mv, tau);
  const double su = scl.su, sv = scl.sv;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->su = scl.su;
    sc->sv = scl.sv;
    sc->sigma = scl.sigma;
    sc->tau_s = scl.tau_s;
    sc->kappa = scl.kappa;
    sc->gv_unscale = scl.gv_unscale;
    sc->gt_unscale = scl.gt_unscale;
    sc->phi_unscale = scl.phi_unscale;
  }
  // one thread per (row, rank index c < SEG): the split is computed once and
  // written to its three segments; the threads also clear the padding entries
  const int64_t total = (m_pad + n_pad) * SEG;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = q / SEG;
    const int c = int(q % SEG);
    const bool is_u = row < m_pad;
    const int64_t r = is_u ? row : row - m_pad;
    double w = 0.0;
    if (c < k && r < (is_u ? m : n)) {
      const int64_t o = (is_u ? 0 : m * k) + r * k + c;
      w = z[o] + (dz ? alpha * dz[o] : 0.0);
      w = is_u ? -w * su : w * sv;
    }
    const __half hh = __double2half(w);
    const __half lo = __double2half(w - double(__half2float(hh)));
    unsigned char* base = is_u ? u_img + (r >> 7) * C::U_BYTES : v_img + (r >> 6) * C::V_BYTES;
    const int atom = is_u ? C::U_ATOM : C::V_ATOM;
    const int rr = int(is_u ? (r & 127) : (r & 63));
    auto put = [&](int e, __half val) {
      *reinterpret_cast<__half*>(base + (e / EPA) * atom +
                                 tc::Swz<RB>::offset(rr, (e % EPA) * 2)) = val;
    };
    // U: segments (m, h, h); V: (h, m, h) (REUSE: the first two only)
    put(c, is_u ? lo : hh);
    put(SEG + c, is_u ? hh : lo);
    if constexpr (!C::REUSE) put(2 * SEG + c, hh);
    for (int e = 3 * SEG + c; e < NE; e += SEG) put(e, __half(0.f));
  }
}

template <int SEG>
__global__ void tc_images_kc_kernel(const double* __restrict__ z, const double* __restrict__ dz,
                                    double alpha, int64_t m, int64_t n, int64_t k, int64_t m_pad,
                                    int64_t n_pad, TcScales* sc, double tau, unsigned char* u_img,
                                    unsigned char* v_img, const unsigned long long* bmax,
                                    int nbmax) {
  tc::pdl_wait();
  tc::pdl_launch_next();
  double mu, mv;
  tc_fold_max(bmax, nbmax, mu, mv);
  tc_images_kc_body<SEG>(z, dz, alpha, m, n, k, m_pad, n_pad, sc, tau, u_img, v_img, mu, mv);
}

// Grid-wide barrier for a kernel whose blocks are all resident (grid sized
// from the occupancy): arrival counter + generation word, both in the
// problem's counter buffer (zeroed at creation, the counter re-armed here).
__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen,
                                             unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1u) {
      *count = 0u;
      __threadfence();
      atomicAdd(const_cast<unsigned*>(gen), 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// passes 1-3 in ONE launch (K-concatenated layout): max |U|, |V| of the trial
// point, a grid barrier, then scales and images.  The dependent fused pass is
// released (PDL) only after the barrier, when every block of this grid is
// resident, so it cannot take the SMs the remaining blocks need.
template <int SEG>
__global__ void __launch_bounds__(256) tc_prep_kc_kernel(
    const double* __restrict__ z, const double* __restrict__ dz, double alpha, int64_t m,
    int64_t n, int64_t k, int64_t m_pad, int64_t n_pad, TcScales* sc, double tau,
    unsigned char* u_img, unsigned char* v_img, unsigned* bar_count, unsigned* bar_gen) {
  tc::pdl_wait();
  {  // pass 1 (tc_max_kernel's loop)
    unsigned long long mu = 0, mv = 0;
    const int64_t nu = m * k, tot = (m + n) * k, stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t q0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q0 < tot;
         q0 += 4 * stride) {
      double zv[4], dv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = q0 + u * stride;
        zv[u] = q < tot ? __ldg(z + q) : 0.0;
        dv[u] = (dz && q < tot) ? __ldg(dz + q) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = q0 + u * stride;
        double w = zv[u];
        if (dz) w += alpha * dv[u];
        const unsigned long long bits = q < tot ? __double_as_longlong(fabs(w)) : 0ull;
        if (q < nu)
          mu = bits > mu ? bits : mu;
        else
          mv = bits > mv ? bits : mv;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, mu, o);
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, mv, o);
      mu = x > mu ? x : mu;
      mv = y > mv ? y : mv;
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&sc->max_bits[0], mu);
      atomicMax(&sc->max_bits[1], mv);
    }
  }
  grid_barrier(bar_count, bar_gen, gridDim.x);
  tc::pdl_launch_next();
  // L2 reads (the maxima were just produced by atomics of other blocks)
  const double mu = __longlong_as_double(__ldcg(&sc->max_bits[0]));
  const double mv = __longlong_as_double(__ldcg(&sc->max_bits[1]));
  tc_images_kc_body<SEG>(z, dz, alpha, m, n, k, m_pad, n_pad, sc, tau, u_img, v_img, mu, mv);
}

}  // namespace spcp
