// sddmm.cuh — sparse-observation evaluation.
//
// When few entries are observed (objective.py:108-110 zeroes the rest), the
// dense pass streams and multiplies mostly dead entries.  This path stores
// only the observed entries, twice:
//   CSR (row_ptr, col, x) for the row pass:    r_ij = x_ij - u_i . v_j,
//        g_ij = -clip(r_ij, +-tau), phi += huber(r_ij), (G V)_i = sum_j g_ij v_j
//   CSC (col_ptr, row, x) for the column pass: (G^T U)_j = sum_i g_ij u_i
//        (the residual is recomputed: no g buffer, one read of each copy)
// Both passes put one warp on a row (column): sub-groups of lanes walk its
// nonzeros, each lane holding a 16-byte slice of the rank dimension, u_i
// (v_j) in registers, the other factor's row gathered from L2 with coalesced
// 16-byte loads (U, V are small), the rank-k accumulators in registers folded
// by fixed butterflies — the summation order depends only on the sparsity
// pattern, so results are bitwise reproducible.  Outputs use the one-chunk / one-band partial layout
// of the streaming kernels (pleft[m_pad][KP], pright[n_pad][KP]), folded by
// reduce_kernel<T> with the objective partials per block.
//
// Work per observed entry: 4 k FMA + 2 gathers of k values (L2); bytes per
// observed entry from HBM: 2 x (4 B index + 4 B value) (fp32 mode).
#pragma once

#include "common.cuh"

namespace spcp {

// ---- construction (problem creation; from the bit-packed mask and the
// device copy of X)

// nonzeros per row: popcount of the row's mask words
__global__ void sddmm_row_count_kernel(const uint32_t* __restrict__ mbits, int64_t ldm,
                                       int64_t m, int64_t words, int64_t* cnt) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < m; i += nw) {
    int64_t c = 0;
    for (int64_t w = lane; w < words; w += 32) c += __popc(mbits[i * ldm + w]);
    c = warp_sum(c);
    if (lane == 0) cnt[i] = c;
  }
}

// nonzeros per column: a warp takes 32 consecutive columns (one mask word) and
// walks the rows
__global__ void sddmm_col_count_kernel(const uint32_t* __restrict__ mbits, int64_t ldm,
                                       int64_t m, int64_t n, int64_t* cnt) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int64_t words = (n + 31) / 32;
  for (int64_t w = warp; w < words; w += nw) {
    int64_t c = 0;
    for (int64_t i = 0; i < m; ++i) c += (mbits[i * ldm + w] >> lane) & 1u;
    const int64_t j = w * 32 + lane;
    if (j < n) cnt[j] = c;
  }
}

// exclusive scan of counts -> pointers (one block; setup only)
__global__ void sddmm_scan_kernel(const int64_t* __restrict__ cnt, int64_t len, int64_t* ptr) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x, nt = blockDim.x;
  const int64_t per = (len + nt - 1) / nt;
  const int64_t b = t * per, e = b + per < len ? b + per : len;
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += cnt[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < nt; ++i) {
      const int64_t v = part[i];
      part[i] = acc;
      acc += v;
    }
    ptr[len] = acc;
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int64_t i = b; i < e; ++i) {
    ptr[i] = acc;
    acc += cnt[i];
  }
}

// CSR fill: warp per row, 32 mask words per round, ballot-free prefix of popcounts
template <typename TX>
__global__ void sddmm_csr_fill_kernel(const uint32_t* __restrict__ mbits, int64_t ldm,
                                      int64_t m, int64_t n, const TX* __restrict__ x,
                                      int64_t ldx, const int64_t* __restrict__ ptr, int32_t* col,
                                      TX* val) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int64_t words = (n + 31) / 32;
  for (int64_t i = warp; i < m; i += nw) {
    int64_t base = ptr[i];
    for (int64_t w0 = 0; w0 < words; w0 += 32) {
      const int64_t w = w0 + lane;
      uint32_t bits = w < words ? mbits[i * ldm + w] : 0u;
      const int c = __popc(bits);
      int pre = c;  // inclusive warp scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += y;
      }
      int64_t pos = base + pre - c;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        const int64_t j = w * 32 + b;
        col[pos] = int32_t(j);
        val[pos] = x[i * ldx + j];
        ++pos;
      }
      base += __shfl_sync(0xffffffffu, pre, 31);
    }
  }
}

// CSC fill: warp per mask word (32 columns), rows in order
template <typename TX>
__global__ void sddmm_csc_fill_kernel(const uint32_t* __restrict__ mbits, int64_t ldm,
                                      int64_t m, int64_t n, const TX* __restrict__ x,
                                      int64_t ldx, const int64_t* __restrict__ ptr, int32_t* row,
                                      TX* val) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int64_t words = (n + 31) / 32;
  for (int64_t w = warp; w < words; w += nw) {
    const int64_t j = w * 32 + lane;
    int64_t pos = j < n ? ptr[j] : 0;
    for (int64_t i = 0; i < m; ++i) {
      if (j < n && ((mbits[i * ldm + w] >> lane) & 1u)) {
        row[pos] = int32_t(i);
        val[pos] = x[i * ldx + j];
        ++pos;
      }
    }
  }
}

// ---- evaluation

struct SddmmParams {
  const int64_t* ptr;   // [rows + 1] (CSR: m, CSC: n)
  const int32_t* idx;   // column (CSR) / row (CSC) of each nonzero
  const void* val;      // TX values
  const void* own;      // T[rows][KP]: the factor of the walked dimension (U for CSR)
  const void* other;    // T[..][KP]: the gathered factor (V for CSR)
  void* out;            // T[rows][KP]: (G V) rows (CSR) / (G^T U) rows (CSC)
  double* pphi;         // [grid] objective partials (CSR pass) or nullptr
  double tau;
  int64_t rows;
};

// One warp per row (CSR) or column (CSC).  The warp splits into NPW
// sub-groups of G lanes; a sub-group takes one nonzero at a time and its lanes
// hold VEC consecutive rank columns each (G * VEC >= KP): the gathered row of
// the other factor is one coalesced 16-byte load per lane, the dot product is
// reduced over the sub-group by xor shuffles, and each lane accumulates g times
// its columns.  At the end of the row the NPW sub-group accumulators are folded
// by a fixed xor butterfly.  The walked factor's row stays in registers.
template <typename T, typename TX, int KP>
__global__ void __launch_bounds__(256) sddmm_pass_kernel(const SddmmParams p) {
  constexpr int VEC = 16 / int(sizeof(T));
  constexpr int G0 = (KP + VEC - 1) / VEC;
  constexpr int G = G0 <= 1 ? 1 : G0 <= 2 ? 2 : G0 <= 4 ? 4 : G0 <= 8 ? 8 : G0 <= 16 ? 16 : 32;
  constexpr int NPW = 32 / G;  // nonzeros per warp step
  static_assert(G * VEC >= KP, "lane columns cover the rank");
  using VT = VecT<T, VEC>;
  __shared__ double red[8];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cg = lane % G, sg = lane / G;  // column group, sub-group
  const int c0 = cg * VEC;
  const bool live_c = c0 < KP;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const T* __restrict__ own = reinterpret_cast<const T*>(p.own);
  const T* __restrict__ oth = reinterpret_cast<const T*>(p.other);
  const TX* __restrict__ val = reinterpret_cast<const TX*>(p.val);
  T* out = reinterpret_cast<T*>(p.out);
  const T tau = T(p.tau);
  double phi = 0.0;
  for (int64_t i = warp; i < p.rows; i += nw) {
    VT u{};
    if (live_c) u = *reinterpret_cast<const VT*>(own + i * KP + c0);
    T acc[VEC];
#pragma unroll
    for (int c = 0; c < VEC; ++c) acc[c] = T(0);
    T hs = T(0);
    const int64_t eb = p.ptr[i], e1 = p.ptr[i + 1];
    for (int64_t e0 = eb; e0 < e1; e0 += 32) {  // warp-uniform trip count
      // 32 nonzeros per round: indices and values in one coalesced load
      // (lane l holds nonzero e0 + l), then every sub-group's gathers of the
      // round are issued before any is used (memory-level parallelism)
      constexpr int NS = 32 / NPW;  // steps per round
      const int64_t el = e0 + lane;
      const int32_t jl = el < e1 ? p.idx[el] : -1;
      const T xl = el < e1 ? T(val[el]) : T(0);
      VT v[NS];
#pragma unroll
      for (int st = 0; st < NS; ++st) {
        const int j = __shfl_sync(0xffffffffu, jl, st * NPW + sg);
        VT t{};
        if (j >= 0 && live_c) t = *reinterpret_cast<const VT*>(oth + int64_t(j) * KP + c0);
        v[st] = t;
      }
#pragma unroll
      for (int st = 0; st < NS; ++st) {
        const int src = st * NPW + sg;
        const int j = __shfl_sync(0xffffffffu, jl, src);
        const T x = __shfl_sync(0xffffffffu, xl, src);
        T d = T(0);
#pragma unroll
        for (int c = 0; c < VEC; ++c) d = fma(u.v[c], v[st].v[c], d);
#pragma unroll
        for (int o = 1; o < G; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        T g = T(0);
        if (j >= 0) {
          T h = T(0);
          g = huber_clip<T>(x - d, tau, h);
          if (cg == 0) hs += h;
        }
#pragma unroll
        for (int c = 0; c < VEC; ++c) acc[c] = fma(g, v[st].v[c], acc[c]);
      }
    }
    phi += double(hs);
    // fold the NPW sub-groups (lanes with the same column group), fixed order
#pragma unroll
    for (int c = 0; c < VEC; ++c) {
      T a = acc[c];
#pragma unroll
      for (int o = G; o < 32; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      acc[c] = a;
    }
    if (sg == 0 && live_c) {
      VT o;
#pragma unroll
      for (int c = 0; c < VEC; ++c) o.v[c] = acc[c];
      *reinterpret_cast<VT*>(out + i * KP + c0) = o;
    }
  }
  if (p.pphi) {
    phi = warp_sum(phi);
    if (lane == 0) red[wib] = phi;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s2 = 0.0;
      for (int w = 0; w < (blockDim.x >> 5); ++w) s2 += red[w];
      p.pphi[blockIdx.x] = s2;
    }
  }
}

}  // namespace spcp
