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
// fp16 pieces computed in fp64 on the device: U'' = uh + um + ul, V'' = vh +
// vm + vl, so the residual uses the 6 products of total order <= 2 (relative
// error ~2^-33 before fp32 accumulation); G'' = gh + gl and the reductions
// use gh.vh + gh.vm + gl.vh (~2^-22).  Each product is exact in the fp32
// accumulator; scales are exact powers of two and are undone at the drain.
//
// Roles: warp 0 = X/mask TMA producer, warp 1 = MMA issuer (+TMEM owner),
// warp 2 = U/V operand-image bulk producer,
// warps 2..9 = epilogue (warp w owns TMEM lane quarter w % 4 and column half
// (w - 2) / 4 of each tile).  Work: a static, exactly balanced range of tiles
// per CTA (one CTA per SM) in 2-D super-block order; GV accumulates in TMEM
// over a run of tiles with the same sub-band and is drained once per run,
// GT is drained per tile and summed into a CTA-private slot per column tile
// (read-modify-write in L2).  Partials are reduced in a fixed order later:
// deterministic, no float atomics.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"

#ifndef SPCP_TC_NRES
#define SPCP_TC_NRES 6
#endif

namespace spcp {

struct TcUnit {
  uint16_t sb, tc;
  int32_t gt_slot;
  int32_t gv_slot;
  uint32_t flags;
};
enum : uint32_t { TCU_FIRST_OF_RUN = 1u, TCU_LAST_OF_RUN = 2u, TCU_FIRST_TOUCH = 4u };

struct TcScales {
  float sigma;       // s_u * s_v: S'' = sigma * L
  float tau_s;       // sigma * tau
  float kappa;       // G'' = kappa * (sigma g)
  float gv_unscale;  // 1 / (kappa sigma s_v)
  float gt_unscale;  // 1 / (kappa sigma s_u)
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
  int kstore;
  int debug;  // bisection switches (SPCP_TC_DEBUG): 1 skip GT stores, 2 skip GV stores,
              // 4 record per-tile timestamps of CTA 0 into dbg_ts
  long long* dbg_ts;  // [64][16]
};

template <int KP16, bool MASK>
struct TcCfg {
  static constexpr int RB = KP16 * 2;           // operand image row bytes (32/64/128)
  static constexpr uint32_t SWK = RB == 128 ? tc::SW_128 : (RB == 64 ? tc::SW_64 : tc::SW_32);
  // X ring (released by the epilogue as soon as it has read the tile) and a
  // separate V-image ring (released when the tile's G.V MMA has finished)
  static constexpr int NST = KP16 == 16 ? 4 : ((KP16 == 64 && MASK) ? 2 : 3);
  static constexpr int NSV = KP16 == 64 ? 2 : 3;
  static constexpr int UB = KP16 == 64 ? 1 : 2;  // U image buffers
  static constexpr int X_BYTES = 128 * 64 * 4;
  static constexpr int V_SPLIT = 64 * RB;
  static constexpr int V_BYTES = 3 * V_SPLIT;
  static constexpr int U_SPLIT = 128 * RB;
  static constexpr int U_BYTES = 3 * U_SPLIT;
  static constexpr int M_BYTES = MASK ? 128 * 4 * 4 : 0;  // box {4 words, 128 rows}
  static constexpr int G_BYTES = 128 * 64 * 2;  // one fp16 G image (MN-major SW128)
  // smem carve (all offsets multiples of 1 KB)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_V = OFF_X + NST * X_BYTES;
  static constexpr int OFF_U = OFF_V + NSV * V_BYTES;
  static constexpr int OFF_GH = OFF_U + UB * U_BYTES;
  static constexpr int OFF_GL = OFF_GH + G_BYTES;
  static constexpr int OFF_M = OFF_GL + G_BYTES;
  static constexpr int OFF_BAR = OFF_M + (MASK ? NST * 2048 : 0);
  static constexpr int SMEM = OFF_BAR + 512;  // dynamic smem base is 1 KB aligned
  // TMEM columns
  // GT holds [G^T uh | G^T um] (N = GCAT * KP16, halves summed at the drain)
  // when TMEM allows; KP16 = 64 keeps the three-product form
  static constexpr int GCAT = KP16 <= 32 ? 2 : 1;
  static constexpr int NRES = SPCP_TC_NRES;  // residual split products (6: order <= 2, 3: order <= 1)
  static constexpr uint32_t T_S = 0, T_GA = 128, T_GV = 256, T_GT = 256 + 2 * KP16;
  static_assert(T_GT + 2 * GCAT * KP16 <= 512, "TMEM budget");
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr int NEPI = 16;  // epilogue warps (4 per SM sub-partition)
  static constexpr int NTHREADS = 32 * (3 + NEPI);  // X producer, MMA, U/V producer, epilogue
};

struct TcBarriers {
  uint64_t stage_full[4], stage_empty[4];
  uint64_t v_full[3], v_empty[3];
  uint64_t u_full[2], u_empty[2];
  uint64_t s_full[2], s_empty[2];
  uint64_t ga_full[2], ga_empty[2];
  uint64_t gs_empty;
  uint64_t gt_full[2], gt_empty[2];
  uint64_t gv_full[2], gv_empty[2];
  uint32_t tmem_base;
  double phi[16];
};

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

#define TC_TS(t, slot)                                                              \
  do {                                                                             \
    if ((p.debug & 4) && blockIdx.x == 0 && (t) < 64) p.dbg_ts[(t) * 16 + (slot)] = clock64(); \
  } while (0)

template <int KP16, bool MASK>
__global__ void __launch_bounds__(TcCfg<KP16, MASK>::NTHREADS, 1)
    tc_eval_kernel(const __grid_constant__ CUtensorMap xmap,
                   const __grid_constant__ CUtensorMap mmap, const TcParams p) {
  using C = TcCfg<KP16, MASK>;
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* sm = smem_dyn;
  if ((smem_u32(sm) & 1023u) != 0u) __trap();  // swizzled TMA/UMMA images need 1 KB alignment
  TcBarriers* bar = reinterpret_cast<TcBarriers*>(sm + C::OFF_BAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ub = p.cta_begin[blockIdx.x], ue = p.cta_begin[blockIdx.x + 1];
  const int T = ue - ub;
  const TcUnit* units = p.units + ub;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NST; ++i) {
      mbar_init(&bar->stage_full[i], 1);
      mbar_init(&bar->stage_empty[i], C::NEPI);
    }
    for (int i = 0; i < C::NSV; ++i) {
      mbar_init(&bar->v_full[i], 1);
      mbar_init(&bar->v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar->u_full[i], 1);
      mbar_init(&bar->u_empty[i], 1);
      mbar_init(&bar->s_full[i], 1);
      mbar_init(&bar->s_empty[i], C::NEPI);
      mbar_init(&bar->ga_full[i], C::NEPI);
      mbar_init(&bar->ga_empty[i], 1);
      mbar_init(&bar->gt_full[i], 1);
      mbar_init(&bar->gt_empty[i], C::NEPI);
      mbar_init(&bar->gv_full[i], 1);
      mbar_init(&bar->gv_empty[i], C::NEPI);
    }
    mbar_init(&bar->gs_empty, 1);
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
  const uint32_t tm = bar->tmem_base;

  if (warp == 0) {
    // ======================= X / mask producer (TMA) ====================
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_first();
      for (int t = 0; t < T; ++t) {
        const TcUnit un = units[t];
        const int st = t % C::NST;
        mbar_wait(&bar->stage_empty[st], ((t / C::NST) & 1) ^ 1);
        TC_TS(t, 0);
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
    }
  } else if (warp == 2) {
    // ======================= U / V operand-image producer (bulk) ========
    if (lane == 0) {
      int prev_sb = -1, fills = 0;
      for (int t = 0; t < T; ++t) {
        const TcUnit un = units[t];
        if ((un.flags & TCU_FIRST_OF_RUN) || un.sb != prev_sb) {
          const int b = fills % C::UB;
          mbar_wait(&bar->u_empty[b], ((fills / C::UB) & 1) ^ 1);
          mbar_arrive_expect_tx(&bar->u_full[b], C::U_BYTES);
          bulk_load(sm + C::OFF_U + b * C::U_BYTES, p.u_img + size_t(un.sb) * C::U_BYTES,
                    C::U_BYTES, &bar->u_full[b]);
          ++fills;
          prev_sb = un.sb;
        }
        const int sv = t % C::NSV;
        mbar_wait(&bar->v_empty[sv], ((t / C::NSV) & 1) ^ 1);
        mbar_arrive_expect_tx(&bar->v_full[sv], C::V_BYTES);
        bulk_load(sm + C::OFF_V + sv * C::V_BYTES, p.v_img + size_t(un.tc) * C::V_BYTES,
                  C::V_BYTES, &bar->v_full[sv]);
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =================================
    constexpr uint32_t ID_RES = idesc_f16(128, 64, false, false);
    constexpr uint32_t ID_GV = idesc_f16(128, KP16, false, true);
    constexpr uint32_t ID_GT = idesc_f16(64, C::GCAT * KP16, true, true);
    constexpr int KS = KP16 / 16;
    const uint32_t u0 = smem_u32(sm + C::OFF_U), v0 = smem_u32(sm + C::OFF_V);
    const uint32_t gh0 = smem_u32(sm + C::OFF_GH), gl0 = smem_u32(sm + C::OFF_GL);
    int run = -1;       // run index of the tile being issued (residual)
    int prev_sb = -1;

    auto residual = [&](int t, int ubuf) {
      const int st = t % C::NSV, b = t & 1;
      mbar_wait(&bar->v_full[st], (t / C::NSV) & 1);
      if (lane == 0) TC_TS(t, 1);
      mbar_wait(&bar->s_empty[b], ((t >> 1) & 1) ^ 1);
      if (lane == 0) TC_TS(t, 2);
      tc_fence_after();
      {
        const uint32_t ua = u0 + ubuf * C::U_BYTES;
        const uint32_t vb = v0 + st * C::V_BYTES;
        // products of total split order <= 2: (h,h) (h,m) (m,h) (h,l) (m,m) (l,h)
        const int pa[6] = {0, 0, 1, 0, 1, 2};
        const int pb[6] = {0, 1, 0, 2, 1, 0};
#pragma unroll
        for (int q = 0; q < C::NRES; ++q)
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
            mma_ss_w(tm + C::T_S + b * 64,
                   umma_desc(ua + pa[q] * C::U_SPLIT + ks * 32, 16, 8 * C::RB, C::SWK),
                   umma_desc(vb + pb[q] * C::V_SPLIT + ks * 32, 16, 8 * C::RB, C::SWK), ID_RES,
                   (q | ks) != 0);
        mma_commit_w(&bar->s_full[b]);
      }
    };

    auto reductions = [&](int t, int ubuf, int rrun, uint32_t flags) {
      const int st = t % C::NSV, b = t & 1, gvb = rrun & 1;
      mbar_wait(&bar->ga_full[b], (t >> 1) & 1);
      if (lane == 0) TC_TS(t, 3);
      mbar_wait(&bar->gt_empty[b], ((t >> 1) & 1) ^ 1);
      if (flags & TCU_FIRST_OF_RUN) mbar_wait(&bar->gv_empty[gvb], ((rrun >> 1) & 1) ^ 1);
      tc_fence_after();
      {
        // G^T U first: it releases the single G staging image the epilogue
        // needs for the next tile
        const uint32_t ua = u0 + ubuf * C::U_BYTES;
        const uint32_t gt = tm + C::T_GT + b * C::GCAT * KP16;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t uo = ks * 16 * C::RB;
          if constexpr (C::GCAT == 2) {
            // B = [uh | um]: two N-atoms of the U image (LBO = split stride);
            // every G byte is read once
            mma_ss_w(gt, umma_desc(gh0 + 2048 * ks, 16384, 1024, SW_128),
                     umma_desc(ua + uo, C::U_SPLIT, 8 * C::RB, C::SWK), ID_GT, ks > 0);
            mma_ss_w(gt, umma_desc(gl0 + 2048 * ks, 16384, 1024, SW_128),
                     umma_desc(ua + uo, C::U_SPLIT, 8 * C::RB, C::SWK), ID_GT, 1);
          } else {
            mma_ss_w(gt, umma_desc(gh0 + 2048 * ks, 16384, 1024, SW_128),
                     umma_desc(ua + uo, 8192, 8 * C::RB, C::SWK), ID_GT, ks > 0);
            mma_ss_w(gt, umma_desc(gh0 + 2048 * ks, 16384, 1024, SW_128),
                     umma_desc(ua + C::U_SPLIT + uo, 8192, 8 * C::RB, C::SWK), ID_GT, 1);
            mma_ss_w(gt, umma_desc(gl0 + 2048 * ks, 16384, 1024, SW_128),
                     umma_desc(ua + uo, 8192, 8 * C::RB, C::SWK), ID_GT, 1);
          }
        }
        mma_commit_w(&bar->gt_full[b]);
        mma_commit_w(&bar->gs_empty);
        const uint32_t vb = v0 + st * C::V_BYTES;
        const uint32_t gv = tm + C::T_GV + gvb * KP16;
        const uint32_t ga = tm + C::T_GA + b * 64;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t vo = ks * 16 * C::RB;
          mma_ts_w(gv, ga + 8 * ks, umma_desc(vb + vo, 8192, 8 * C::RB, C::SWK), ID_GV,
                 !((flags & TCU_FIRST_OF_RUN) && ks == 0));
          mma_ts_w(gv, ga + 8 * ks, umma_desc(vb + C::V_SPLIT + vo, 8192, 8 * C::RB, C::SWK),
                 ID_GV, 1);
          mma_ts_w(gv, ga + 32 + 8 * ks, umma_desc(vb + vo, 8192, 8 * C::RB, C::SWK), ID_GV, 1);
        }
        mma_commit_w(&bar->ga_empty[b]);
        mma_commit_w(&bar->v_empty[st]);
        if (flags & TCU_LAST_OF_RUN) {
          mma_commit_w(&bar->gv_full[gvb]);
          mma_commit_w(&bar->u_empty[ubuf]);
        }
      }
    };

    // bookkeeping of the previous tile (its reductions trail its residual)
    int p_ubuf = 0, p_run = 0;
    uint32_t p_flags = 0;
    for (int t = 0; t < T; ++t) {
      const TcUnit un = units[t];
      const bool new_run = (un.flags & TCU_FIRST_OF_RUN) || un.sb != prev_sb;
      if (new_run) {
        ++run;
        prev_sb = un.sb;
      }
      const int ubuf = run % C::UB;
      const bool reduce_first = new_run && C::UB == 1 && t >= 1;
      if (reduce_first) reductions(t - 1, p_ubuf, p_run, p_flags);
      if (new_run) mbar_wait(&bar->u_full[ubuf], (run / C::UB) & 1);
      residual(t, ubuf);
      if (!reduce_first && t >= 1) reductions(t - 1, p_ubuf, p_run, p_flags);
      p_ubuf = ubuf;
      p_run = run;
      p_flags = un.flags;
    }
    if (T >= 1) reductions(T - 1, p_ubuf, p_run, p_flags);
  } else {
    // ======================= epilogue warps =============================
    // warp e = warp - 3 owns TMEM lane quarter q = warp % 4 (rows 32q..32q+31)
    // and columns [part * CPW, part * CPW + CPW) of every 64-column tile.
    constexpr int CPW = 256 / C::NEPI;      // columns per epilogue warp (16 or 32)
    constexpr int NPAIR = CPW / 2;          // packed half2 registers per split
    const int q = warp & 3;
    const int part = (warp - 3) >> 2;
    const int row = 32 * q + lane;
    const uint32_t lane_addr = uint32_t(32 * q) << 16;
    const TcScales sc = *p.scales;
    const float sigma = sc.sigma, tau_s = sc.tau_s, kappa = sc.kappa;
    double phi_acc = 0.0;
    int run = -1, prev_sb = -1;
    int prev_gv_slot = -1;
    constexpr int GTC = KP16 / 2;  // accumulator columns drained per draining warp
    const bool drainer = part < 2;  // two warps per lane quarter drain G.V / G^T.U
    const int dpart = part & 1;
    // swizzled byte offsets of this thread's X row chunks (box = 32 columns)
    const int xbox = (part * CPW) >> 5;
    const int xc0 = ((part * CPW) & 31) >> 2;  // first 16 B chunk within the box row

    // G^T U of tile t2 -> this CTA's private slot for the column tile: plain
    // stores on first touch, then fp32x4 reductions in L2.  Each (row, col)
    // of a slot is owned by one thread, whose same-address operations apply
    // in program order: deterministic without staging or fences.
    auto drain_gt = [&](int t2, const TcUnit& u2) {
      const int b = t2 & 1;
      mbar_wait(&bar->gt_full[b], (t2 >> 1) & 1);
      tc_fence_after();
      if (drainer && !(p.debug & 1)) {
        float* dst =
            p.pright + (size_t(u2.gt_slot) * 64 + 16 * q + lane) * KP16 + dpart * GTC;
        const bool first = (u2.flags & TCU_FIRST_TOUCH) != 0;
        constexpr int CH = GTC < 16 ? GTC : 16;
#pragma unroll
        for (int c0 = 0; c0 < GTC; c0 += CH) {
          uint32_t v[CH], w[CH];
          const uint32_t col =
              tm + lane_addr + C::T_GT + b * C::GCAT * KP16 + dpart * GTC + c0;
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
              if (first)
                *reinterpret_cast<uint4*>(dst + c0 + c) =
                    make_uint4(v[c], v[c + 1], v[c + 2], v[c + 3]);
              else
                red_add_v4(dst + c0 + c, v[c], v[c + 1], v[c + 2], v[c + 3]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar->gt_empty[b]);
    };

    auto drain_gv = [&](int rrun, int slot) {
      const int gvb = rrun & 1;
      mbar_wait(&bar->gv_full[gvb], (rrun >> 1) & 1);
      tc_fence_after();
      if (drainer && !(p.debug & 2)) {
        float* dst = p.pleft + (size_t(slot) * 128 + row) * KP16 + dpart * GTC;
        constexpr int CH = GTC < 16 ? GTC : 16;
#pragma unroll
        for (int c0 = 0; c0 < GTC; c0 += CH) {
          uint32_t v[CH];
          tmem_ldn<CH>(tm + lane_addr + C::T_GV + gvb * KP16 + dpart * GTC + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < CH; c += 4)
            *reinterpret_cast<uint4*>(dst + c0 + c) = make_uint4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar->gv_empty[gvb]);
    };

    TcUnit prev_unit{};
    TcUnit un_next = T > 0 ? units[0] : TcUnit{};
    for (int t = 0; t < T; ++t) {
      const TcUnit un = un_next;
      if (t + 1 < T) un_next = units[t + 1];  // consumed next iteration: latency hidden
      const bool new_run = (un.flags & TCU_FIRST_OF_RUN) || un.sb != prev_sb;
      if (new_run) {
        ++run;
        prev_sb = un.sb;
      }
      const int st = t % C::NST, b = t & 1;
      // ---- S tile and X tile
      const bool ts_w = (warp == 3 && lane == 0);
      if (ts_w) TC_TS(t, 4);
      mbar_wait(&bar->s_full[b], (t >> 1) & 1);
      if (ts_w) TC_TS(t, 5);
      tc_fence_after();
      uint32_t sv[CPW];
      tmem_ldn<CPW>(tm + lane_addr + C::T_S + b * 64 + part * CPW, sv);
      mbar_wait(&bar->stage_full[st], (t / C::NST) & 1);
      if (ts_w) TC_TS(t, 6);
      const unsigned char* xs = sm + C::OFF_X + st * C::X_BYTES + xbox * 16384;
      float xv[CPW];
#pragma unroll
      for (int c = 0; c < CPW / 4; ++c) {
        const float4 f =
            *reinterpret_cast<const float4*>(xs + Swz<128>::offset(row, (xc0 + c) * 16));
        xv[4 * c] = f.x;
        xv[4 * c + 1] = f.y;
        xv[4 * c + 2] = f.z;
        xv[4 * c + 3] = f.w;
      }
      uint32_t mw = 0xffffffffu;
      if (MASK) {
        mw = reinterpret_cast<const uint32_t*>(sm + C::OFF_M + st * 2048)[row * 4 +
                                                                          (un.tc & 1) * 2 +
                                                                          ((part * CPW) >> 5)];
        mw >>= (part * CPW) & 31;
      }
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bar->s_empty[b]);
        mbar_arrive(&bar->stage_empty[st]);
      }
      // ---- epilogue math: r = x - L (scaled), clip, huber, split
      uint32_t hi[NPAIR], lo[NPAIR];
      float hs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < CPW; e += 2) {
        float g2[2];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const int c = e + f;
          float r = fmaf(xv[c], sigma, -__uint_as_float(sv[c]));
          if (MASK) r = ((mw >> c) & 1u) ? r : 0.f;
          const float a = fabsf(r);
          const float cl = fminf(a, tau_s);
          hs[c & 3] = fmaf(cl, fmaf(-0.5f, cl, a), hs[c & 3]);
          g2[f] = -copysignf(cl, r) * kappa;
        }
        const __half2 hh = __floats2half2_rn(g2[0], g2[1]);
        const float2 hf = __half22float2(hh);
        hi[e >> 1] = *reinterpret_cast<const uint32_t*>(&hh);
        lo[e >> 1] = pack_half2(g2[0] - hf.x, g2[1] - hf.y);
      }
      phi_acc += double((hs[0] + hs[1]) + (hs[2] + hs[3]));
      // ---- G to TMEM (A of G.V) and to smem (A of G^T.U)
      mbar_wait(&bar->ga_empty[b], ((t >> 1) & 1) ^ 1);
      if constexpr (NPAIR == 16) {
        tmem_st16(tm + lane_addr + C::T_GA + b * 64 + part * NPAIR, hi);
        tmem_st16(tm + lane_addr + C::T_GA + b * 64 + 32 + part * NPAIR, lo);
      } else {
        tmem_st8(tm + lane_addr + C::T_GA + b * 64 + part * NPAIR, hi);
        tmem_st8(tm + lane_addr + C::T_GA + b * 64 + 32 + part * NPAIR, lo);
      }
      if (ts_w) TC_TS(t, 7);
      mbar_wait(&bar->gs_empty, (t & 1) ^ 1);
      if (ts_w) TC_TS(t, 8);
      unsigned char* gh = sm + C::OFF_GH;
      unsigned char* gl = sm + C::OFF_GL;
#pragma unroll
      for (int c = 0; c < NPAIR / 4; ++c) {
        const uint32_t o = Swz<128>::offset(row, part * CPW * 2 + 16 * c);
        *reinterpret_cast<uint4*>(gh + o) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2],
                                                       hi[4 * c + 3]);
        *reinterpret_cast<uint4*>(gl + o) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2],
                                                       lo[4 * c + 3]);
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar->ga_full[b]);
      if (ts_w) TC_TS(t, 9);
      // ---- deferred drains
      if (t >= 1) drain_gt(t - 1, prev_unit);
      if (new_run && t >= 1) drain_gv(run - 1, prev_gv_slot);
      if (ts_w) TC_TS(t, 10);
      prev_unit = un;
      prev_gv_slot = un.gv_slot;
    }
    if (T >= 1) {
      drain_gt(T - 1, prev_unit);
      drain_gv(run, prev_gv_slot);
    }
    // phi: per-thread fp64, fold over the epilogue warps in a fixed order
    double w = warp_sum(phi_acc);
    if (lane == 0) bar->phi[warp - 3] = w;
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
__global__ void tc_max_kernel(const double* __restrict__ z, const double* __restrict__ dz,
                              double alpha, int64_t nu, int64_t nv, TcScales* sc) {
  unsigned long long mu = 0, mv = 0;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < nu + nv;
       q += int64_t(gridDim.x) * blockDim.x) {
    double w = z[q];
    if (dz) w += alpha * dz[q];
    const unsigned long long bits = __double_as_longlong(fabs(w));
    if (q < nu)
      mu = bits > mu ? bits : mu;
    else
      mv = bits > mv ? bits : mv;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mu, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, mv, o);
    mu = a > mu ? a : mu;
    mv = b > mv ? b : mv;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&sc->max_bits[0], mu);
    atomicMax(&sc->max_bits[1], mv);
  }
}

// pass 2: power-of-two scales (one thread)
__global__ void tc_scales_kernel(TcScales* sc, double tau) {
  const double mu = __longlong_as_double(sc->max_bits[0]);
  const double mv = __longlong_as_double(sc->max_bits[1]);
  auto pow2_for = [](double mx) {  // largest 2^e with mx * 2^e <= 2^14
    if (!(mx > 0.0)) return 1.0;
    int e;
    frexp(mx, &e);  // mx = f * 2^e, f in [0.5, 1)
    return ldexp(1.0, 14 - e);
  };
  const double su = pow2_for(mu), sv = pow2_for(mv);
  const double sigma = su * sv;
  const double taus = sigma * tau;
  int e;
  frexp(taus, &e);
  const double kappa = ldexp(1.0, 14 - e);
  sc->su = su;
  sc->sv = sv;
  sc->sigma = float(sigma);
  sc->tau_s = float(taus);
  sc->kappa = float(kappa);
  sc->gv_unscale = float(1.0 / (kappa * sigma * sv));
  sc->gt_unscale = float(1.0 / (kappa * sigma * su));
  sc->phi_unscale = 1.0 / (sigma * sigma);
}

template <int RB>
__device__ __forceinline__ void split3_store(unsigned char* base, int split_bytes, int row, int c,
                                             double x) {
  const __half h = __double2half(x);
  const double r1 = x - double(__half2float(h));
  const __half m = __double2half(r1);
  const double r2 = r1 - double(__half2float(m));
  const __half l = __double2half(r2);
  const uint32_t o = tc::Swz<RB>::offset(row, c * 2);
  *reinterpret_cast<__half*>(base + o) = h;
  *reinterpret_cast<__half*>(base + split_bytes + o) = m;
  *reinterpret_cast<__half*>(base + 2 * split_bytes + o) = l;
}

// pass 3: fp16 split images of U (per 128-row sub-band) and V (per 64-row tile)
template <int KP16>
__global__ void tc_images_kernel(const double* __restrict__ z, const double* __restrict__ dz,
                                 double alpha, int64_t m, int64_t n, int64_t k, int64_t m_pad,
                                 int64_t n_pad, const TcScales* sc, unsigned char* u_img,
                                 unsigned char* v_img) {
  constexpr int RB = KP16 * 2;
  const double su = sc->su, sv = sc->sv;
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
      split3_store<RB>(u_img + sb * (3 * 128 * RB), 128 * RB, int(row & 127), c, w * su);
    } else {
      const int64_t j = row - m_pad;
      double w = 0.0;
      if (j < n && c < k) {
        const int64_t o = m * k + j * k + c;
        w = z[o] + (dz ? alpha * dz[o] : 0.0);
      }
      const int64_t tcol = j >> 6;
      split3_store<RB>(v_img + tcol * (3 * 64 * RB), 64 * RB, int(j & 63), c, w * sv);
    }
  }
}

}  // namespace spcp
