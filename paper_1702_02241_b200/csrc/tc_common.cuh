// tc_common.cuh — sm_100a primitives for the tensor-core streaming kernel:
// mbarriers, TMA / bulk copies, TMEM allocation and access, tcgen05.mma with
// UMMA shared-memory descriptors.  Inline PTX only (no CUTLASS dependency).
//
// Layout conventions used by this repo (all verified by tools/tc_probe.cu):
//  * UMMA smem operands are "canonical" images: 8-row groups of R-byte rows,
//    R in {32, 64, 128} with the matching hardware swizzle
//    (byte bits [4, 4+B) ^= bits [7, 7+B), B = log2(R/16)), groups SBO bytes
//    apart.  The same image is a K-major operand (rows = M/N, row = K) and an
//    MN-major operand (rows = K, row = M/N) — the residual's B (V, K = rank)
//    and the G.V product's B (V, K = columns) share one copy.
//  * TMEM addresses: bits [31:16] lane, [15:0] column.  An M = 128 fp32
//    accumulator puts row i in lane i, column j in column base + j.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace spcp {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef SPCP_MBAR_SPIN
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep in HW until the phase flips
      : "memory");
}

// non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.b32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// 16-byte shared load pinned to one LDS.128 (the compiler otherwise splits some
// of the swizzled X reads into LDS.64 pairs, which double their wavefronts)
__device__ __forceinline__ float4 lds128(const void* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// Programmatic dependent launch: wait for the preceding grid (a no-op unless
// this kernel was launched with programmatic stream serialization) / let the
// next one start launching its CTAs.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_next() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------------ packed fp32 pairs
// Blackwell FFMA2 / FADD2 / FMUL2 on float2 (one instruction per pair)
__device__ __forceinline__ uint64_t f2_bits(float2 v) {
  return (uint64_t(__float_as_uint(v.y)) << 32) | __float_as_uint(v.x);
}
__device__ __forceinline__ float2 f2_from(uint64_t b) {
  return make_float2(__uint_as_float(uint32_t(b)), __uint_as_float(uint32_t(b >> 32)));
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return f2_from(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(d);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(d);
}

// ------------------------------------------------------------------ async copies
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 2-D TMA tile load into shared memory, completion counted on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// L2-only prefetch of a 2-D tensor tile (no shared memory, no completion)
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
// Same with an L2 cache policy (createpolicy) — X is streamed once: evict first.
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// fire-and-forget fp32x4 reduction in L2; same-thread same-address operations
// are applied in program order, so a slot owned by one thread stays deterministic
__device__ __forceinline__ void red_add_v4(float* p, uint32_t a, uint32_t b, uint32_t c,
                                           uint32_t d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
// 1-D bulk copy global -> shared (16 B aligned, size multiple of 16).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global bulk store / fp32 reduce-add (async, bulk_group completion)
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_reduce_add_f32(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::
                   "l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// lo = g - float(h) for the two fp16 halves of h2, one mixed-precision FMA
// each (FHFMA: h * -1 + g, a single rounding of an exact difference, so
// bitwise the same as converting h back to fp32 and subtracting)
__device__ __forceinline__ float2 sub_half2_from(float2 g, uint32_t h2) {
  float2 r;
  asm("{\n.reg .b16 l, h, m;\nmov.b32 {l, h}, %2;\nmov.b16 m, 0xBC00;\n"
      "fma.rn.f32.f16 %0, l, m, %3;\nfma.rn.f32.f16 %1, h, m, %4;\n}\n"
      : "=f"(r.x), "=f"(r.y)
      : "r"(h2), "f"(g.x), "f"(g.y));
  return r;
}

// named barrier over `count` threads (id 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ------------------------------------------------------------------ TMEM
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 32 lanes x 16 columns of 32-bit: thread t gets lane (base lane + t),
// r[i] = column (base col + i).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
// N consecutive 32-bit columns (N in {4, 8, 16, 32}) into r[0..N)
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t* r) {
  if constexpr (N == 4) {
    uint32_t t[4];
    tmem_ld4(taddr, t);
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = t[i];
  } else if constexpr (N == 8) {
    uint32_t t[8];
    tmem_ld8(taddr, t);
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = t[i];
  } else {
#pragma unroll
    for (int c = 0; c < N; c += 16) {
      uint32_t t[16];
      tmem_ld16(taddr + c, t);
#pragma unroll
      for (int i = 0; i < 16; ++i) r[c + i] = t[i];
    }
  }
}

// ------------------------------------------------------------------ UMMA
enum SwizzleKind : uint32_t { SW_NONE = 0, SW_128 = 2, SW_64 = 4, SW_32 = 6 };

template <int ROW_BYTES>
struct Swz {
  static constexpr uint32_t kind = ROW_BYTES == 128 ? SW_128 : (ROW_BYTES == 64 ? SW_64 : SW_32);
  static constexpr int bits = ROW_BYTES == 128 ? 3 : (ROW_BYTES == 64 ? 2 : 1);
  // physical byte offset of logical (row, byte) in a canonical image whose
  // 8-row groups are contiguous (SBO = 8 * ROW_BYTES)
  __host__ __device__ static constexpr uint32_t offset(uint32_t row, uint32_t byte) {
    const uint32_t o = row * ROW_BYTES + byte;
    return o ^ (((o >> 7) & ((1u << bits) - 1u)) << 4);
  }
};

// Shared-memory matrix descriptor (sm_100 "version 1").
__device__ __forceinline__ uint64_t umma_desc(uint32_t smem_addr, uint32_t lbo_bytes,
                                              uint32_t sbo_bytes, uint32_t swizzle_kind) {
  uint64_t d = 0;
  d |= uint64_t((smem_addr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // version
  d |= uint64_t(swizzle_kind & 7u) << 61;
  return d;
}

// Instruction descriptor for kind::f16 with fp16 A/B and fp32 accumulate.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, bool a_mn_major,
                                                  bool b_mn_major) {
  return (1u << 4)                                   // D format F32
         | (0u << 7) | (0u << 10)                    // A, B = F16
         | (uint32_t(a_mn_major) << 15) | (uint32_t(b_mn_major) << 16) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// D[tmem] (+)= A[smem desc] * B[smem desc]
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-uniform variants: the whole (converged) warp executes the asm with
// uniform operands and elect.sync picks the one lane that issues.  Keeping the
// call site non-divergent lets descriptors live in uniform registers (no
// per-instruction R2UR / ELECT waterfall loop around each UTCHMMA).
__device__ __forceinline__ void mma_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 r;\nsetp.ne.b32 p, %4, 0;\n"
      "elect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 r;\nsetp.ne.b32 p, %4, 0;\n"
      "elect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Same, with compile-time descriptor offsets (descriptor units = bytes >> 4)
// added inside the asm: the base descriptors stay the only per-tile values,
// so consecutive MMAs of a batch share their conversion to uniform registers.
template <int OA, int OB>
__device__ __forceinline__ void mma_ss_o(uint32_t d_tmem, uint64_t a_base, uint64_t b_base,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 r;\n.reg .b64 ad, bd;\nsetp.ne.b32 p, %4, 0;\n"
      "add.s64 ad, %1, %5;\nadd.s64 bd, %2, %6;\n"
      "elect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_base), "l"(b_base), "r"(idesc), "r"(accumulate), "n"(OA), "n"(OB)
      : "memory");
}
template <int OB>
__device__ __forceinline__ void mma_ts_o(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_base,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 r;\n.reg .b64 bd;\nsetp.ne.b32 p, %4, 0;\n"
      "add.s64 bd, %2, %5;\n"
      "elect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], bd, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_base), "r"(idesc), "r"(accumulate), "n"(OB)
      : "memory");
}
// Single-thread variants (the issuing loop runs on one lane): no elect, and
// ptxas keeps base descriptors + immediate offsets on the uniform datapath.
template <int OA, int OB>
__device__ __forceinline__ void mma_ss_1(uint32_t d_tmem, uint64_t a_base, uint64_t b_base,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b64 ad, bd;\nsetp.ne.b32 p, %4, 0;\n"
      "add.s64 ad, %1, %5;\nadd.s64 bd, %2, %6;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_base), "l"(b_base), "r"(idesc), "r"(accumulate), "n"(OA), "n"(OB)
      : "memory");
}
template <int OB>
__device__ __forceinline__ void mma_ts_1(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_base,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b64 bd;\nsetp.ne.b32 p, %4, 0;\n"
      "add.s64 bd, %2, %5;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], bd, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_base), "r"(idesc), "r"(accumulate), "n"(OB)
      : "memory");
}

// ---- whole MMA batches in one asm block: one elect.sync per batch, the
// descriptors stepped by immediate strides inside the block.

// Residual: NQ products x KS K-steps into one accumulator.  Product q reads
// A split qa(q) and B split qb(q) (the residual uses (0,0) (0,1) (1,0)).
// A-split stride SA, B-split stride SB, K-step stride KSTEP (descriptor units).
#define SPCP_MMA_SS(ACC) "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, " ACC ";\n"
template <int KS, int SA, int SB, int KSTEP>
__device__ __forceinline__ void mma_residual_batch(uint32_t d, uint64_t a0, uint64_t b0,
                                                   uint32_t idesc) {
  static_assert(KS == 1 || KS == 2 || KS == 4, "KS");
  if constexpr (KS == 1) {
    asm volatile(
        "{\n.reg .pred e, pf, pt;\n.reg .b32 r;\n.reg .b64 a, b;\n"
        "setp.ne.b32 pf, 0, 0;\nsetp.eq.b32 pt, 0, 0;\nelect.sync r|e, 0xffffffff;\n"
        "mov.b64 a, %1;\nmov.b64 b, %2;\n" SPCP_MMA_SS("pf")
        "add.s64 b, %2, %5;\n" SPCP_MMA_SS("pt")
        "add.s64 a, %1, %4;\nmov.b64 b, %2;\n" SPCP_MMA_SS("pt") "}\n"
        ::"r"(d), "l"(a0), "l"(b0), "r"(idesc), "n"(SA), "n"(SB) : "memory");
  } else if constexpr (KS == 2) {
    asm volatile(
        "{\n.reg .pred e, pf, pt;\n.reg .b32 r;\n.reg .b64 a, b, a1, b1;\n"
        "setp.ne.b32 pf, 0, 0;\nsetp.eq.b32 pt, 0, 0;\nelect.sync r|e, 0xffffffff;\n"
        "mov.b64 a, %1;\nmov.b64 b, %2;\n" SPCP_MMA_SS("pf")
        "add.s64 a, %1, %6;\nadd.s64 b, %2, %6;\n" SPCP_MMA_SS("pt")
        "mov.b64 a, %1;\nadd.s64 b, %2, %5;\n" SPCP_MMA_SS("pt")
        "add.s64 a, %1, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        "add.s64 a, %1, %4;\nmov.b64 b, %2;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, %2, %6;\n" SPCP_MMA_SS("pt") "}\n"
        ::"r"(d), "l"(a0), "l"(b0), "r"(idesc), "n"(SA), "n"(SB), "n"(KSTEP) : "memory");
  } else {
    asm volatile(
        "{\n.reg .pred e, pf, pt;\n.reg .b32 r;\n.reg .b64 a, b;\n"
        "setp.ne.b32 pf, 0, 0;\nsetp.eq.b32 pt, 0, 0;\nelect.sync r|e, 0xffffffff;\n"
        // (0,0)
        "mov.b64 a, %1;\nmov.b64 b, %2;\n" SPCP_MMA_SS("pf")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        // (0,1)
        "mov.b64 a, %1;\nadd.s64 b, %2, %5;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        // (1,0)
        "add.s64 a, %1, %4;\nmov.b64 b, %2;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt")
        "add.s64 a, a, %6;\nadd.s64 b, b, %6;\n" SPCP_MMA_SS("pt") "}\n"
        ::"r"(d), "l"(a0), "l"(b0), "r"(idesc), "n"(SA), "n"(SB), "n"(KSTEP) : "memory");
  }
}

// G^T U with B = [uh|um] N-concatenated: 8 K-steps x {gh, gl}.
// A stride per K-step SAK, gl offset SGL, B stride per K-step SBK.
#define SPCP_GT2 SPCP_MMA_SS("pt") "add.s64 a, a, %5;\n" SPCP_MMA_SS("pt") \
  "sub.s64 a, a, %5;\nadd.s64 a, a, %4;\nadd.s64 b, b, %6;\n"
template <int SAK, int SGL, int SBK>
__device__ __forceinline__ void mma_gtu_batch2(uint32_t d, uint64_t a0, uint64_t b0,
                                               uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred e, pf, pt;\n.reg .b32 r;\n.reg .b64 a, b;\n"
      "setp.ne.b32 pf, 0, 0;\nsetp.eq.b32 pt, 0, 0;\nelect.sync r|e, 0xffffffff;\n"
      "mov.b64 a, %1;\nmov.b64 b, %2;\n"
      SPCP_MMA_SS("pf") "add.s64 a, a, %5;\n" SPCP_MMA_SS("pt")
      "sub.s64 a, a, %5;\nadd.s64 a, a, %4;\nadd.s64 b, b, %6;\n"
      SPCP_GT2 SPCP_GT2 SPCP_GT2 SPCP_GT2 SPCP_GT2 SPCP_GT2 SPCP_GT2 "}\n"
      ::"r"(d), "l"(a0), "l"(b0), "r"(idesc), "n"(SAK), "n"(SGL), "n"(SBK) : "memory");
}

// G.V with A = G from TMEM (hi at +0, lo at +32 columns), B = [vh|vm]:
// 4 K-steps x {gh, gl}; the first MMA accumulates unless `first`.
#define SPCP_MMA_TS(ACC) "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, " ACC ";\n"
#define SPCP_GV2 "add.s32 ta, ta, 8;\n" SPCP_MMA_TS("pt") "add.s32 ta, ta, 32;\n" SPCP_MMA_TS("pt") \
  "sub.s32 ta, ta, 32;\n"
template <int SBK>
__device__ __forceinline__ void mma_gv_batch2(uint32_t d, uint32_t a_tmem, uint64_t b0,
                                              uint32_t idesc, uint32_t acc_first) {
  asm volatile(
      "{\n.reg .pred e, pa, pt;\n.reg .b32 r, ta;\n.reg .b64 b;\n"
      "setp.ne.b32 pa, %4, 0;\nsetp.eq.b32 pt, 0, 0;\nelect.sync r|e, 0xffffffff;\n"
      "mov.b32 ta, %1;\nmov.b64 b, %2;\n"
      SPCP_MMA_TS("pa") "add.s32 ta, ta, 32;\n" SPCP_MMA_TS("pt") "sub.s32 ta, ta, 32;\n"
      "add.s64 b, b, %5;\n" SPCP_GV2
      "add.s64 b, b, %5;\n" SPCP_GV2
      "add.s64 b, b, %5;\n" SPCP_GV2 "}\n"
      ::"r"(d), "r"(a_tmem), "l"(b0), "r"(idesc), "r"(acc_first), "n"(SBK) : "memory");
}

// ---- warp-wide batches for the K-concatenated kernel: the whole (converged)
// warp executes ONE asm block, one elect.sync, N MMAs with the descriptors
// stepped by immediates (no per-MMA waterfall loop around a single lane).
#define SPCP_SSB(ACC) "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, " ACC ";\n"
#define SPCP_SSB_STEP "add.s64 a, a, %5;\nadd.s64 b, b, %6;\n"
template <int N, int SA, int SB>
__device__ __forceinline__ void mma_ss_batch(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc,
                                             uint32_t acc0) {
  static_assert(N >= 1 && N <= 8, "batch size");
#define SPCP_SSB_HEAD                                                                       \
  "{\n.reg .pred e, p0, pt;\n.reg .b32 r;\n.reg .b64 a, b;\n"                               \
  "setp.ne.b32 p0, %4, 0;\nsetp.eq.b32 pt, 0, 0;\nelect.sync r|e, 0xffffffff;\n"            \
  "mov.b64 a, %1;\nmov.b64 b, %2;\n" SPCP_SSB("p0")
#define SPCP_SSB_ARGS \
  ::"r"(d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "n"(SA), "n"(SB) : "memory"
  if constexpr (N == 1) {
    asm volatile(SPCP_SSB_HEAD "}\n" SPCP_SSB_ARGS);
  } else if constexpr (N == 2) {
    asm volatile(SPCP_SSB_HEAD SPCP_SSB_STEP SPCP_SSB("pt") "}\n" SPCP_SSB_ARGS);
  } else if constexpr (N == 3) {
    asm volatile(SPCP_SSB_HEAD SPCP_SSB_STEP SPCP_SSB("pt") SPCP_SSB_STEP SPCP_SSB("pt") "}\n"
                 SPCP_SSB_ARGS);
  } else if constexpr (N == 4) {
    asm volatile(SPCP_SSB_HEAD SPCP_SSB_STEP SPCP_SSB("pt") SPCP_SSB_STEP SPCP_SSB("pt")
                     SPCP_SSB_STEP SPCP_SSB("pt") "}\n" SPCP_SSB_ARGS);
  } else {
    static_assert(N == 8, "batch size 1-4 or 8");
    asm volatile(SPCP_SSB_HEAD SPCP_SSB_STEP SPCP_SSB("pt") SPCP_SSB_STEP SPCP_SSB("pt")
                     SPCP_SSB_STEP SPCP_SSB("pt") SPCP_SSB_STEP SPCP_SSB("pt") SPCP_SSB_STEP
                         SPCP_SSB("pt") SPCP_SSB_STEP SPCP_SSB("pt") SPCP_SSB_STEP SPCP_SSB("pt")
                             "}\n" SPCP_SSB_ARGS);
  }
#undef SPCP_SSB_HEAD
#undef SPCP_SSB_ARGS
}

// G.V with A = G from TMEM over the tile's S columns (per 32-column half: gh at
// +0, gl at +16; K-step ks covers columns 32 (ks / 2) + 8 (ks % 2)), B = V
// image stepped by SB per K-step: 4 K-steps x {gh, gl} = 8 TS MMAs.
#define SPCP_TSB(ACC) "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], b, %3, " ACC ";\n"
template <int SB>
__device__ __forceinline__ void mma_gv_ts_batch(uint32_t d, uint32_t s_tmem, uint64_t b0,
                                                uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n.reg .pred e, p0, pt;\n.reg .b32 r, t;\n.reg .b64 b;\n"
      "setp.ne.b32 p0, %4, 0;\nsetp.eq.b32 pt, 0, 0;\nelect.sync r|e, 0xffffffff;\n"
      "mov.b64 b, %2;\n"
      "add.s32 t, %1, 0;\n" SPCP_TSB("p0") "add.s32 t, %1, 16;\n" SPCP_TSB("pt")
      "add.s64 b, b, %5;\n"
      "add.s32 t, %1, 8;\n" SPCP_TSB("pt") "add.s32 t, %1, 24;\n" SPCP_TSB("pt")
      "add.s64 b, b, %5;\n"
      "add.s32 t, %1, 32;\n" SPCP_TSB("pt") "add.s32 t, %1, 48;\n" SPCP_TSB("pt")
      "add.s64 b, b, %5;\n"
      "add.s32 t, %1, 40;\n" SPCP_TSB("pt") "add.s32 t, %1, 56;\n" SPCP_TSB("pt") "}\n"
      ::"r"(d), "r"(s_tmem), "l"(b0), "r"(idesc), "r"(acc0), "n"(SB) : "memory");
}
#undef SPCP_TSB

// smem -> TMEM copy of one 128-row x 32-byte K-step of a K-major operand image
// (lane i <- row i, 8 columns of fp16 pairs: the A-from-TMEM layout; verified
// against tcgen05.st by tools/tc_probe.cu P7).  Warp-wide, one elected issuer.
__device__ __forceinline__ void tmem_cp_128x256b_w(uint32_t taddr, uint64_t desc) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n}\n" ::"r"(taddr),
      "l"(desc)
      : "memory");
}

// N TS MMAs (A from TMEM, stepped by 8 columns = one fp16 K-step of 16; B
// descriptor stepped by SB units), warp-wide with one elect.
#define SPCP_TSN(ACC) "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], b, %3, " ACC ";\n"
#define SPCP_TSN_STEP "add.s32 t, t, 8;\nadd.s64 b, b, %5;\n"
template <int N, int SB>
__device__ __forceinline__ void mma_ts_batch(uint32_t d, uint32_t a_tmem, uint64_t b0,
                                             uint32_t idesc, uint32_t acc0) {
  static_assert(N >= 1 && N <= 4, "batch size");
#define SPCP_TSN_HEAD                                                                   \
  "{\n.reg .pred e, p0, pt;\n.reg .b32 r, t;\n.reg .b64 b;\n"                           \
  "setp.ne.b32 p0, %4, 0;\nsetp.eq.b32 pt, 0, 0;\nelect.sync r|e, 0xffffffff;\n"        \
  "mov.b32 t, %1;\nmov.b64 b, %2;\n" SPCP_TSN("p0")
#define SPCP_TSN_ARGS ::"r"(d), "r"(a_tmem), "l"(b0), "r"(idesc), "r"(acc0), "n"(SB) : "memory"
  if constexpr (N == 1) {
    asm volatile(SPCP_TSN_HEAD "}\n" SPCP_TSN_ARGS);
  } else if constexpr (N == 2) {
    asm volatile(SPCP_TSN_HEAD SPCP_TSN_STEP SPCP_TSN("pt") "}\n" SPCP_TSN_ARGS);
  } else if constexpr (N == 3) {
    asm volatile(SPCP_TSN_HEAD SPCP_TSN_STEP SPCP_TSN("pt") SPCP_TSN_STEP SPCP_TSN("pt") "}\n"
                 SPCP_TSN_ARGS);
  } else {
    asm volatile(SPCP_TSN_HEAD SPCP_TSN_STEP SPCP_TSN("pt") SPCP_TSN_STEP SPCP_TSN("pt")
                     SPCP_TSN_STEP SPCP_TSN("pt") "}\n" SPCP_TSN_ARGS);
  }
#undef SPCP_TSN_HEAD
#undef SPCP_TSN_ARGS
}
#undef SPCP_TSN
#undef SPCP_TSN_STEP

__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, %1;\nselp.b32 %0, 1, 0, px;\n}\n"
      : "=r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}

}  // namespace tc
}  // namespace spcp
