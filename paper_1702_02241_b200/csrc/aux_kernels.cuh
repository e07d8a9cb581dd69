// aux_kernels.cuh — the small kernels around the streaming pass: operand prep,
// fixed-order partial reductions, upload/convert, dense materialisation and
// the L-BFGS / factor-space vector algebra.  None of these touch X more than
// once per call except the dense (materialising) kernels used for final L/S
// and for rank bounds beyond the fused kernel's register budget.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"

namespace spcp {

// ------------------------------------------------------------------ upload
// Convert rows [row0, row0+rows) of a dense source (ld = lds, dtype S) into the
// padded device X copies and accumulate 0.5*sum_{Omega} x^2 / count per block.
template <typename S>
__global__ void convert_x_kernel(const S* __restrict__ src, int64_t lds, int64_t rows,
                                 int64_t n, int64_t row0, float* x32, double* x64,
                                 int64_t ldx, const uint8_t* __restrict__ mask_rows,
                                 double* part_sq, double* part_cnt) {
  __shared__ double scratch[32];
  double sq = 0.0, cnt = 0.0;
  const int64_t total = rows * n;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / n, j = q % n;
    const double v = double(src[i * lds + j]);
    const int64_t o = (row0 + i) * ldx + j;
    if (x32) x32[o] = float(v);
    if (x64) x64[o] = v;
    const bool obs = mask_rows == nullptr || mask_rows[i * n + j] != 0;
    if (obs) {
      sq += v * v;
      cnt += 1.0;
    }
  }
  const double a = block_sum(sq, scratch);
  const double b = block_sum(cnt, scratch);
  if (threadIdx.x == 0) {
    part_sq[blockIdx.x] += 0.5 * a;
    part_cnt[blockIdx.x] += b;
  }
}

// bit-pack rows of a bool mask: word w of row i holds columns 32w..32w+31
__global__ void pack_mask_kernel(const uint8_t* __restrict__ mask_rows, int64_t rows,
                                 int64_t n, int64_t row0, uint32_t* mbits, int64_t ldm) {
  const int64_t words = (n + 31) / 32;
  const int64_t total = rows * words;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / words, w = q % words;
    uint32_t bits = 0u;
    for (int b = 0; b < 32; ++b) {
      const int64_t j = w * 32 + b;
      if (j < n && mask_rows[i * n + j] != 0) bits |= (1u << b);
    }
    mbits[(row0 + i) * ldm + w] = bits;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ a, int n, double* out) {
  __shared__ double scratch[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += a[i];
  // fixed order: strided per-thread sums then a fixed tree
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) *out = s;
}

// ------------------------------------------------------------------ prep
// Trial point w = z + alpha*dz (float64) -> padded compute-dtype operands.
// rows of U: [0, m), of V: [0, n); columns [0, k) of KP; pads are zero.
template <typename T>
__global__ void prep_operands_kernel(const double* __restrict__ z, const double* __restrict__ dz,
                                     double alpha, int64_t m, int64_t n, int64_t k,
                                     int64_t m_pad, int64_t n_pad, int kp, T* uc, T* vc) {
  const int64_t total = (m_pad + n_pad) * kp;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = q / kp;
    const int c = int(q % kp);
    double w = 0.0;
    if (row < m_pad) {
      if (row < m && c < k) {
        const int64_t o = row * k + c;
        w = z[o];
        if (dz) w += alpha * dz[o];
      }
      uc[q] = T(w);
    } else {
      const int64_t j = row - m_pad;
      if (j < n && c < k) {
        const int64_t o = m * k + j * k + c;
        w = z[o];
        if (dz) w += alpha * dz[o];
      }
      vc[j * kp + c] = T(w);
    }
  }
}

// Same, for a product operand given directly as a float64 (rows x b) matrix.
template <typename T>
__global__ void pad_operand_kernel(const double* __restrict__ w, int64_t rows, int64_t b,
                                   int64_t rows_pad, int bp, T* out) {
  const int64_t total = rows_pad * bp;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / bp;
    const int c = int(q % bp);
    out[q] = (r < rows && c < b) ? T(w[r * b + c]) : T(0);
  }
}

// Columns [c0, c0 + bw) of a row-major float64 (rows x ld) matrix into a
// zero-padded (rows_pad x pw) operand of type T (the apply passes' W / Y).
template <typename T>
__global__ void stage_cols_kernel(const double* __restrict__ w, int64_t ld, int64_t c0, int64_t bw,
                                  int64_t rows, int64_t rows_pad, int pw, T* out) {
  const int64_t total = rows_pad * pw;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / pw;
    const int c = int(q % pw);
    out[q] = (r < rows && c < bw) ? T(w[r * ld + c0 + c]) : T(0);
  }
}

// ------------------------------------------------------------------ reduce
enum UMode { U_SKIP = 0, U_FULL = 1, U_PARTIAL = 2, U_FROM_SUM = 3 };

struct ReduceParams {
  int64_t m, n, k, m_pad, n_pad;
  int kp;
  const double* z;
  const double* dz;
  double alpha, lambda_l;
  const void* pleft;   // T[nchunks][m_pad][kp]
  int nchunks;
  const void* pright;  // T[nrb][n_pad][kp]
  int nrb;
  const void* gu_sum;  // T[m][k] (U_FROM_SUM)
  void* gu_part;       // T[m][k] (U_PARTIAL)
  double* g_out;       // flat [U | V]
  int u_mode, v_mode;  // v_mode: 1 = full V gradient, 0 = skip
  double* blk;         // [gridDim][6]: gU2, gUdU, regU, gV2, gVdV, regV
  unsigned* counter;   // last-block detector
  const double* pphi;
  int nphi;
  const double* scal_sum;  // U_FROM_SUM: [phi, regV, gVdV, gV2] summed over ranks
  double* scal_out;        // U_PARTIAL: shard scalars out
  double* out;             // [8] totals (U_FULL / U_FROM_SUM)
  // tensor-core partial layout (csr_u_off != nullptr): pleft[slot][128][kst],
  // pright[slot][gt_rows][kst], sources per 128-row sub-band / 64-column tile
  const int32_t* csr_u_off;
  const int32_t* csr_u_idx;
  const int32_t* csr_v_off;
  const int32_t* csr_v_idx;
  int kst;                  // partial row stride (the kernel's padded rank)
  int gt_rows;              // G^T.U slot rows: 64, or 128 = [gh part; gl part] (summed here)
  int chunked;              // slots laid out [kst / 4][rows][4] (K-concatenated kernel)
  const float* tc_unscale;  // [0]: G.V partials, [1]: G^T.U partials
};

// Block partials of the six vector sums -> the last block folds them (and the
// phi partials) in a fixed order into the scalar outputs.
// `scratch` holds 6 * 32 doubles.  The six block sums share one barrier; each
// follows block_sum's tree (warp butterfly, then warp 0 over the warp sums).
__device__ __forceinline__ void reduce_tail(const ReduceParams& p, const double (&s)[6],
                                            double* scratch, bool& am_last) {
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      const double v = warp_sum(s[r]);
      if (lane == 0) scratch[r * 32 + w] = v;
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double v = warp_sum(lane < nw ? scratch[r * 32 + lane] : 0.0);
        if (lane == 0) p.blk[blockIdx.x * 6 + r] = v;
      }
    }
  }
  // last block folds the block partials in a fixed order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned done = atomicAdd(p.counter, 1u);
    am_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double tot[6];
  for (int r = 0; r < 6; ++r) {
    double v = 0.0;
    for (int b = threadIdx.x; b < int(gridDim.x); b += blockDim.x) v += p.blk[b * 6 + r];
    tot[r] = block_sum(v, scratch);
  }
  double phi = 0.0;
  {
    double v = 0.0;
    for (int b = threadIdx.x; b < p.nphi; b += blockDim.x) v += p.pphi ? p.pphi[b] : 0.0;
    phi = block_sum(v, scratch);
  }
  if (threadIdx.x == 0) {
    const double half_l = 0.5 * p.lambda_l;
    if (p.u_mode == U_PARTIAL) {
      p.scal_out[0] = phi;
      p.scal_out[1] = half_l * tot[5];
      p.scal_out[2] = tot[4];
      p.scal_out[3] = tot[3];
    } else if (p.u_mode == U_FROM_SUM) {
      const double regU = half_l * tot[2];
      p.out[0] = p.scal_sum[0] + regU + p.scal_sum[1];
      p.out[1] = p.scal_sum[0];
      p.out[2] = regU + p.scal_sum[1];
      p.out[3] = tot[1] + p.scal_sum[2];
      p.out[4] = tot[0] + p.scal_sum[3];
      p.out[5] = tot[0];
      p.out[6] = tot[1];
      p.out[7] = 0.0;
    } else {
      const double reg = half_l * (tot[2] + tot[5]);
      p.out[0] = phi + reg;
      p.out[1] = phi;
      p.out[2] = reg;
      p.out[3] = tot[1] + tot[4];
      p.out[4] = tot[0] + tot[3];
      p.out[5] = tot[0];
      p.out[6] = tot[1];
      p.out[7] = 0.0;
    }
    *p.counter = 0u;  // re-arm for the next launch
  }
}

template <typename T>
__global__ void __launch_bounds__(256) reduce_kernel(const ReduceParams p) {
  __shared__ double scratch[6 * 32];
  __shared__ bool am_last;
  const int64_t nu = p.m * p.k, nv = p.n * p.k;
  double s[6] = {0, 0, 0, 0, 0, 0};
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p.u_mode != U_SKIP) {
    const T* pl = reinterpret_cast<const T*>(p.pleft);
    for (int64_t q = t0; q < nu; q += stride) {
      const int64_t i = q / p.k, c = q % p.k;
      double acc;
      if (p.u_mode == U_FROM_SUM) {
        acc = double(reinterpret_cast<const T*>(p.gu_sum)[q]);
      } else {
        acc = 0.0;
        if (p.csr_u_off) {
          const int sb = int(i >> 7);
          const float* plf = reinterpret_cast<const float*>(p.pleft);
          for (int e = p.csr_u_off[sb]; e < p.csr_u_off[sb + 1]; ++e)
            acc += double(plf[(int64_t(p.csr_u_idx[e]) * 128 + (i & 127)) * p.kst + c]);
          acc *= double(p.tc_unscale[0]);
        } else {
          for (int ch = 0; ch < p.nchunks; ++ch)
            acc += double(pl[(int64_t(ch) * p.m_pad + i) * p.kp + c]);
        }
      }
      if (p.u_mode == U_PARTIAL) {
        reinterpret_cast<T*>(p.gu_part)[q] = T(acc);
        continue;
      }
      double w = p.z[q];
      const double d = p.dz ? p.dz[q] : 0.0;
      w += p.alpha * d;
      const double g = acc + p.lambda_l * w;
      p.g_out[q] = g;
      s[0] += g * g;
      s[1] += g * d;
      s[2] += w * w;
    }
  }
  if (p.v_mode) {
    const T* pr = reinterpret_cast<const T*>(p.pright);
    for (int64_t q = t0; q < nv; q += stride) {
      const int64_t j = q / p.k, c = q % p.k;
      double acc = 0.0;
      if (p.csr_v_off) {
        const int tcol = int(j >> 6);
        const float* prf = reinterpret_cast<const float*>(p.pright);
        for (int e = p.csr_v_off[tcol]; e < p.csr_v_off[tcol + 1]; ++e) {
          const float* sl = prf + int64_t(p.csr_v_idx[e]) * p.gt_rows * p.kst;
          acc += double(sl[(j & 63) * p.kst + c]);
          if (p.gt_rows == 128) acc += double(sl[(64 + (j & 63)) * p.kst + c]);
        }
        acc *= double(p.tc_unscale[1]);
      } else {
        for (int b = 0; b < p.nrb; ++b) acc += double(pr[(int64_t(b) * p.n_pad + j) * p.kp + c]);
      }
      const int64_t o = nu + q;
      double w = p.z[o];
      const double d = p.dz ? p.dz[o] : 0.0;
      w += p.alpha * d;
      const double g = acc + p.lambda_l * w;
      p.g_out[o] = g;
      s[3] += g * g;
      s[4] += g * d;
      s[5] += w * w;
    }
  }
  reduce_tail(p, s, scratch, am_last);
}

// Tensor-core partial layout (CSR slots, TcParams): one thread per (row, 4
// columns); the slot sources of a sub-band / column tile are read as float4
// and summed in fp64 in the CSR's fixed order (deterministic).  U side:
// U_FULL or U_PARTIAL; V side always.
// Balanced source counts (square-ish super-blocks, e.g. C2): one item space over
// both sides, LPI lanes per item.
template <int LPI>
__global__ void __launch_bounds__(256) tc_reduce_lpi_kernel(const ReduceParams p) {
  tc::pdl_wait();  // the fused pass's partial slots are complete
  tc::pdl_launch_next();
  // LPI lanes per output item (row r, 4 columns): lane j sums the CSR sources
  // e = j, j + LPI, ... of the item (all its loads in flight at once), then the
  // LPI partial sums are combined in a fixed butterfly order.
  __shared__ double scratch[6 * 32];
  __shared__ bool am_last;
  const int c4n = p.kst >> 2;
  const int64_t nu4 = p.m * c4n, nv4 = p.n * c4n;
  double s[6] = {0, 0, 0, 0, 0, 0};
  constexpr int IPW = 32 / LPI;  // items per warp
  const int j = threadIdx.x & (LPI - 1);
  const int64_t stride = (int64_t(gridDim.x) * blockDim.x) / LPI;  // items per sweep
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const float* plf = reinterpret_cast<const float*>(p.pleft);
  const float* prf = reinterpret_cast<const float*>(p.pright);
  const float gvs = p.tc_unscale[0], gts = p.tc_unscale[1];
  const int64_t n_items = nu4 + nv4;
  // warp-uniform trip count: a warp's IPW items start at (gtid >> 5) * IPW
  for (int64_t w0 = (gtid >> 5) * IPW; w0 < n_items; w0 += stride) {
    const int64_t q0 = w0 + ((threadIdx.x & 31) / LPI);
    const bool live = q0 < n_items;  // dead lanes still join the shuffles
    const int64_t q = live ? q0 : w0;  // dead lanes shadow lane 0's item
    const bool is_u = q < nu4;
    const int64_t qq = is_u ? q : q - nu4;
    // chunked slots: consecutive items take consecutive rows of one 4-column
    // chunk (contiguous float4 reads); row-major slots: consecutive chunks of a row
    const int64_t rows = is_u ? p.m : p.n;
    // 32-bit index split (items < 2^31: the TC path caps m, n at 65535 tiles):
    // a 64-bit div/mod pair per item was a large share of the instructions
    const uint32_t q32 = uint32_t(qq), d32 = p.chunked ? uint32_t(rows) : uint32_t(c4n);
    const uint32_t quo = q32 / d32, rem = q32 - quo * d32;
    const int64_t r = p.chunked ? rem : quo;
    const int c0 = int(p.chunked ? quo : rem) * 4;
    // warp-uniform source list (every item of the warp in one sub-band / one
    // column tile, <= 32 sources): one coalesced load of the CSR indices, then
    // shuffles, so each batch is a single dependent memory round trip
    const int tile = is_u ? int(r >> 7) : int(r >> 6);
    const int* coff = is_u ? p.csr_u_off : p.csr_v_off;
    const int e0 = coff[tile], e1 = coff[tile + 1];
    const int key = is_u ? tile : -1 - tile;
    const bool uni = __all_sync(0xffffffffu, key == __shfl_sync(0xffffffffu, key, 0)) &&
                     e1 - e0 <= 32;
    int lidx = -1;
    if (uni) {
      const int lane = threadIdx.x & 31;
      lidx = lane < e1 - e0 ? __ldg((is_u ? p.csr_u_idx : p.csr_v_idx) + e0 + lane) : -1;
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (is_u) {
      const float* base = p.chunked ? plf + (int64_t(c0 >> 2) * 128 + (r & 127)) * 4
                                    : plf + (r & 127) * p.kst + c0;
      const int64_t sst = int64_t(128) * p.kst;
      // batches of 8 sources per lane: the 8 index loads, then the 8 data
      // loads are all in flight before the (in-order) adds.  Uniform warps run
      // the same trip count on every lane (shuffles need all 32 lanes).
      const int ebeg = uni ? e0 : e0 + j;
      for (int eb = ebeg; eb < e1; eb += 8 * LPI) {
        int idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
        {
          // source e (absolute CSR position) of this lane's batch slot
          const int e = eb + (uni ? j : 0) + LPI * u;
          const int sh = uni ? __shfl_sync(0xffffffffu, lidx, (e - e0) & 31) : -1;
          idx[u] = e < e1 ? (uni ? sh : __ldg(p.csr_u_idx + e)) : -1;
        }
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = idx[u] >= 0 ? *reinterpret_cast<const float4*>(base + idx[u] * sst)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a0 += v[u].x; a1 += v[u].y; a2 += v[u].z; a3 += v[u].w;
        }
      }
    } else {
      const float* base = p.chunked ? prf + (int64_t(c0 >> 2) * p.gt_rows + (r & 63)) * 4
                                    : prf + (r & 63) * p.kst + c0;
      const int64_t sst = int64_t(p.gt_rows) * p.kst;
      const int64_t hoff = p.chunked ? int64_t(64) * 4 : int64_t(64) * p.kst;
      const bool two = p.gt_rows == 128;
      const int ebeg = uni ? e0 : e0 + j;
      for (int eb = ebeg; eb < e1; eb += 4 * LPI) {
        int idx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
        {
          // source e (absolute CSR position) of this lane's batch slot
          const int e = eb + (uni ? j : 0) + LPI * u;
          const int sh = uni ? __shfl_sync(0xffffffffu, lidx, (e - e0) & 31) : -1;
          idx[u] = e < e1 ? (uni ? sh : __ldg(p.csr_v_idx + e)) : -1;
        }
        float4 v[4], w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float* b0 = base + (idx[u] >= 0 ? idx[u] : 0) * sst;
          v[u] = idx[u] >= 0 ? *reinterpret_cast<const float4*>(b0) : make_float4(0.f, 0.f, 0.f, 0.f);
          w[u] = (idx[u] >= 0 && two) ? *reinterpret_cast<const float4*>(b0 + hoff)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a0 += v[u].x; a1 += v[u].y; a2 += v[u].z; a3 += v[u].w;
          a0 += w[u].x; a1 += w[u].y; a2 += w[u].z; a3 += w[u].w;
        }
      }
    }
    // fixed-order combine of the LPI lanes
#pragma unroll
    for (int o = 1; o < LPI; o <<= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      a3 += __shfl_xor_sync(0xffffffffu, a3, o);
    }
    if (!live || j != 0) continue;
    const double sc = is_u ? gvs : gts;
    const double acc[4] = {a0 * sc, a1 * sc, a2 * sc, a3 * sc};
    const int64_t obase = (is_u ? 0 : p.m * p.k) + r * p.k;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int c = c0 + jj;
      if (c >= p.k) break;
      const int64_t o = obase + c;
      if (is_u && p.u_mode == U_PARTIAL) {
        reinterpret_cast<float*>(p.gu_part)[r * p.k + c] = float(acc[jj]);
        continue;
      }
      double w = p.z[o];
      const double d = p.dz ? p.dz[o] : 0.0;
      w += p.alpha * d;
      const double g = acc[jj] + p.lambda_l * w;
      p.g_out[o] = g;
      const int sidx = is_u ? 0 : 3;
      s[sidx] += g * g;
      s[sidx + 1] += g * d;
      s[sidx + 2] += w * w;
    }
  }
  reduce_tail(p, s, scratch, am_last);
}

// One side of the tensor-core partial fold: `lp` lanes per output item (row r,
// 4 columns); lane j sums the item's CSR sources e = j, j + lp, ... in batches
// of 4 (all loads in flight), then the lp partial sums are combined by a fixed
// butterfly.  lp is chosen per side from its source count (tall-skinny shapes
// have many G^T U sources per column tile and few G.V sources per sub-band).
__device__ __forceinline__ void tc_reduce_side(const ReduceParams& p, bool is_u, int lp,
                                               double (&s)[6]) {
  const int c4n = p.kst >> 2;
  const int64_t rows = is_u ? p.m : p.n;
  const int64_t n_items = rows * c4n;
  const int ipw = 32 / lp;  // items per warp
  const int j = threadIdx.x & (lp - 1);
  const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t stride = (int64_t(gridDim.x) * blockDim.x >> 5) * ipw;  // items per sweep
  const float* part = reinterpret_cast<const float*>(is_u ? p.pleft : p.pright);
  const int* off = is_u ? p.csr_u_off : p.csr_v_off;
  const int* idxs = is_u ? p.csr_u_idx : p.csr_v_idx;
  const int slot_rows = is_u ? 128 : p.gt_rows;
  const int tile_rows = is_u ? 128 : 64;
  const int tile_shift = is_u ? 7 : 6;
  const bool two = !is_u && p.gt_rows == 128;  // gh part + gl part rows
  const int64_t sst = int64_t(slot_rows) * p.kst;
  const int64_t hoff = p.chunked ? int64_t(64) * 4 : int64_t(64) * p.kst;
  const double sc = double(p.tc_unscale[is_u ? 0 : 1]);
  for (int64_t w0 = (gtid >> 5) * ipw; w0 < n_items; w0 += stride) {
    const int64_t q0 = w0 + ((threadIdx.x & 31) / lp);
    const bool live = q0 < n_items;  // dead lanes still join the shuffles
    const int64_t qq = live ? q0 : 0;
    // chunked slots: consecutive items take consecutive rows of one chunk
    // 32-bit index split (items < 2^31: the TC path caps m, n at 65535 tiles):
    // a 64-bit div/mod pair per item was a large share of the instructions
    const uint32_t q32 = uint32_t(qq), d32 = p.chunked ? uint32_t(rows) : uint32_t(c4n);
    const uint32_t quo = q32 / d32, rem = q32 - quo * d32;
    const int64_t r = p.chunked ? rem : quo;
    const int c0 = int(p.chunked ? quo : rem) * 4;
    const int tile = int(r >> tile_shift);
    const int e0 = off[tile], e1 = off[tile + 1];
    const int64_t rr = r & (tile_rows - 1);
    const float* base = p.chunked ? part + (int64_t(c0 >> 2) * slot_rows + rr) * 4
                                  : part + rr * p.kst + c0;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int eb = e0 + j; eb < e1; eb += 4 * lp) {
      int id[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) id[u] = (eb + lp * u < e1) ? __ldg(idxs + eb + lp * u) : -1;
      float4 v[4], w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float* b0 = base + (id[u] >= 0 ? id[u] : 0) * sst;
        v[u] = id[u] >= 0 ? *reinterpret_cast<const float4*>(b0) : make_float4(0.f, 0.f, 0.f, 0.f);
        w[u] = (id[u] >= 0 && two) ? *reinterpret_cast<const float4*>(b0 + hoff)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 += v[u].x; a1 += v[u].y; a2 += v[u].z; a3 += v[u].w;
        a0 += w[u].x; a1 += w[u].y; a2 += w[u].z; a3 += w[u].w;
      }
    }
    for (int o = 1; o < lp; o <<= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      a3 += __shfl_xor_sync(0xffffffffu, a3, o);
    }
    if (!live || j != 0) continue;
    const double acc[4] = {a0 * sc, a1 * sc, a2 * sc, a3 * sc};
    const int64_t obase = (is_u ? 0 : p.m * p.k) + r * p.k;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int c = c0 + jj;
      if (c >= p.k) break;
      const int64_t o = obase + c;
      if (is_u && p.u_mode == U_PARTIAL) {
        reinterpret_cast<float*>(p.gu_part)[r * p.k + c] = float(acc[jj]);
        continue;
      }
      double wv = p.z[o];
      const double d = p.dz ? p.dz[o] : 0.0;
      wv += p.alpha * d;
      const double g = acc[jj] + p.lambda_l * wv;
      p.g_out[o] = g;
      const int sidx = is_u ? 0 : 3;
      s[sidx] += g * g;
      s[sidx + 1] += g * d;
      s[sidx + 2] += wv * wv;
    }
  }
}

__global__ void __launch_bounds__(256, 4) tc_reduce_kernel(const ReduceParams p, int lp_u, int lp_v) {
  tc::pdl_wait();  // the fused pass's partial slots are complete
  tc::pdl_launch_next();
  __shared__ double scratch[6 * 32];
  __shared__ bool am_last;
  double s[6] = {0, 0, 0, 0, 0, 0};
  tc_reduce_side(p, true, lp_u, s);
  tc_reduce_side(p, false, lp_v, s);
  reduce_tail(p, s, scratch, am_last);
}

// Fold of the tensor-core partial slots, one block per output segment: a
// 128-row sub-band of grad_U or a 64-row column tile of grad_V.  The
// segment's CSR source list sits in shared memory; one thread per (row, 4
// columns) item sums its sources in CSR order in fp64, batches of 8 loads in
// flight (consecutive threads take consecutive rows of a chunk: coalesced).
// Every item has one fixed summation order: bitwise reproducible.
constexpr int kFoldMaxSrc = 64;
__global__ void __launch_bounds__(256, 4) tc_fold_kernel(const ReduceParams p, int nsb) {
  tc::pdl_wait();  // the fused pass's partial slots are complete
  tc::pdl_launch_next();
  __shared__ double scratch[6 * 32];
  __shared__ bool am_last;
  __shared__ int64_t src[2 * kFoldMaxSrc];  // element offsets of the segment's slots
  double s[6] = {0, 0, 0, 0, 0, 0};
  const int seg = blockIdx.x;
  const bool is_u = seg < nsb;
  const int tile = is_u ? seg : seg - nsb;
  const int* off = is_u ? p.csr_u_off : p.csr_v_off;
  const int* idxs = is_u ? p.csr_u_idx : p.csr_v_idx;
  const int e0 = off[tile], ne = off[tile + 1] - e0;
  const int slot_rows = is_u ? 128 : p.gt_rows;
  const bool two = !is_u && p.gt_rows == 128;  // gh part + gl part rows: two sources
  const int64_t sst = int64_t(slot_rows) * p.kst;
  const int nsrc = two ? 2 * ne : ne;
  for (int i = threadIdx.x; i < nsrc; i += blockDim.x)
    src[i] = two ? int64_t(idxs[e0 + (i >> 1)]) * sst + (i & 1) * 64 * 4
                 : int64_t(idxs[e0 + i]) * sst;
  __syncthreads();
  const int tile_rows = is_u ? 128 : 64;
  const int64_t rows_total = is_u ? p.m : p.n;
  const int64_t r_base = int64_t(tile) * tile_rows;
  const int c4n = p.kst >> 2;
  const float* part = reinterpret_cast<const float*>(is_u ? p.pleft : p.pright);
  const double sc = double(p.tc_unscale[is_u ? 0 : 1]);
  for (int it = threadIdx.x; it < tile_rows * c4n; it += blockDim.x) {
    const int chunk = it / tile_rows, rr = it - chunk * tile_rows;
    const int64_t r = r_base + rr;
    if (r >= rows_total) continue;
    const float* base = part + (int64_t(chunk) * slot_rows + rr) * 4;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int eb = 0; eb < nsrc; eb += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = eb + u < nsrc ? *reinterpret_cast<const float4*>(base + src[eb + u])
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0 += v[u].x; a1 += v[u].y; a2 += v[u].z; a3 += v[u].w;
      }
    }
    const double acc[4] = {a0 * sc, a1 * sc, a2 * sc, a3 * sc};
    const int c0 = chunk * 4;
    const int64_t obase = (is_u ? 0 : p.m * p.k) + r * p.k;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int c = c0 + jj;
      if (c >= p.k) break;
      const int64_t o = obase + c;
      if (is_u && p.u_mode == U_PARTIAL) {
        reinterpret_cast<float*>(p.gu_part)[r * p.k + c] = float(acc[jj]);
        continue;
      }
      double wv = p.z[o];
      const double d = p.dz ? p.dz[o] : 0.0;
      wv += p.alpha * d;
      const double g = acc[jj] + p.lambda_l * wv;
      p.g_out[o] = g;
      const int sidx = is_u ? 0 : 3;
      s[sidx] += g * g;
      s[sidx + 1] += g * d;
      s[sidx + 2] += wv * wv;
    }
  }
  reduce_tail(p, s, scratch, am_last);
}

// Reduce apply() partials to float64 outputs (rows x b, b <= bp).
template <typename T>
__global__ void reduce_apply_kernel(const T* __restrict__ part, int nparts, int64_t rows,
                                    int64_t rows_pad, int bp, int64_t b, double* out) {
  const int64_t total = rows * b;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / b, c = q % b;
    double acc = 0.0;
    for (int s = 0; s < nparts; ++s) acc += double(part[(int64_t(s) * rows_pad + r) * bp + c]);
    out[q] = acc;
  }
}

// ------------------------------------------------------------------ dense
// L tile = U V^T for a 64x64 tile from the float64 iterate z (any k), then
//   MODE 0: write L (ld = ldo) and S* = shrink(X - L) on Omega
//   MODE 1: write G = -clip(X - L) on Omega (float64, ld = ldo) + phi partials
//   (TO: the element type of l_out in MODE 1 — float for the certificate's
//   stored fp32 G)
template <typename TX, int MODE, typename TO = double>
__global__ void __launch_bounds__(256) dense_kernel(
    const double* __restrict__ z, int64_t m, int64_t n, int64_t k, const TX* __restrict__ x,
    int64_t ldx, const uint32_t* __restrict__ mbits, int64_t ldm, double tau, int64_t row0,
    int64_t rows, TO* l_out, double* s_out, int64_t ldo, double* pphi) {
  constexpr int TB = 64, KC = 16;
  __shared__ double ut[KC][TB + 1];
  __shared__ double vt[KC][TB + 1];
  __shared__ double scratch[32];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t i0 = row0 + int64_t(blockIdx.y) * TB;
  const int64_t j0 = int64_t(blockIdx.x) * TB;
  const double* U = z;
  const double* V = z + m * k;
  double acc[4][4] = {};
  for (int64_t kc = 0; kc < k; kc += KC) {
    for (int q = threadIdx.x; q < KC * TB; q += 256) {
      const int r = q / KC, c = q % KC;
      const int64_t gi = i0 + r, gj = j0 + r, gk = kc + c;
      ut[c][r] = (gi < row0 + rows && gi < m && gk < k) ? U[gi * k + gk] : 0.0;
      vt[c][r] = (gj < n && gk < k) ? V[gj * k + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      double a[4], b[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = ut[c][ty * 4 + e];
        b[e] = vt[c][tx * 4 + e];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int f = 0; f < 4; ++f) acc[e][f] = fma(a[e], b[f], acc[e][f]);
    }
    __syncthreads();
  }
  double h = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t gi = i0 + ty * 4 + e;
    if (gi >= row0 + rows || gi >= m) continue;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int64_t gj = j0 + tx * 4 + f;
      if (gj >= n) continue;
      const double l = acc[e][f];
      const bool obs = mbits == nullptr || ((mbits[gi * ldm + (gj >> 5)] >> (gj & 31)) & 1u);
      double r = obs ? double(x[gi * ldx + gj]) - l : 0.0;
      const int64_t o = (gi - row0) * ldo + gj;
      if constexpr (MODE == 0) {
        if (l_out) l_out[o] = l;
        if (s_out) {
          const double a = r < 0 ? -r : r;
          const double mag = a - tau > 0.0 ? a - tau : 0.0;
          s_out[o] = r > 0 ? mag : (r < 0 ? -mag : 0.0);
        }
      } else {
        l_out[o] = TO(huber_clip<double>(r, tau, h));
      }
    }
  }
  if (MODE == 1) {
    const double t = block_sum(h, scratch);
    if (threadIdx.x == 0) pphi[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = t;
  }
}

// phi_value_grad on a dense float64 L (objective.py:90-117)
template <typename TX>
__global__ void phi_dense_kernel(const double* __restrict__ l, int64_t m, int64_t n,
                                 const TX* __restrict__ x, int64_t ldx,
                                 const uint32_t* __restrict__ mbits, int64_t ldm, double tau,
                                 double* grad, double* s_out, double* part) {
  __shared__ double scratch[32];
  double h = 0.0;
  const int64_t total = m * n;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / n, j = q % n;
    const bool obs = mbits == nullptr || ((mbits[i * ldm + (j >> 5)] >> (j & 31)) & 1u);
    const double r = obs ? double(x[i * ldx + j]) - l[q] : 0.0;
    const double g = huber_clip<double>(r, tau, h);
    if (grad) grad[q] = g;
    if (s_out) {
      const double a = r < 0 ? -r : r;
      const double mag = a - tau > 0.0 ? a - tau : 0.0;
      s_out[q] = r > 0 ? mag : (r < 0 ? -mag : 0.0);
    }
  }
  const double t = block_sum(h, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// ------------------------------------------------------------------ vectors
constexpr int kMaxVec = 40;
struct VecPtrs {
  const double* a[kMaxVec];
  const double* b[kMaxVec];
  double coef[kMaxVec];
};

// grid (nblk, count): partial dots; then fold_kernel sums per pair in order.
__global__ void multidot_kernel(VecPtrs vp, int64_t len, double* part, int nblk) {
  __shared__ double scratch[32];
  const int pair = blockIdx.y;
  const double* a = vp.a[pair];
  const double* b = vp.b[pair];
  double s = 0.0;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < len;
       q += int64_t(nblk) * blockDim.x)
    s += a[q] * b[q];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) part[pair * nblk + blockIdx.x] = s;
}

__global__ void fold_kernel(const double* __restrict__ part, int nblk, double* out) {
  __shared__ double scratch[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) s += part[blockIdx.x * nblk + i];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// all dots <a_i, b_j> in one pass: grid-stride over the vectors, NB columns
// kept in registers, fixed-order block partials [blk][NA_MAX][NB].
constexpr int kGramNA = 24;
struct GramPtrs {
  const double* a[kGramNA];
  const double* b[4];
};
// a-vectors in groups of kGramGA over blockIdx.y: every accumulator index is a
// compile-time constant, so acc[][] lives in registers (indexing it with the
// runtime count put the whole array in local memory: a local read-modify-write
// per FMA); each group re-reads the NB b-vectors
constexpr int kGramGA = 8;
template <int NB>
__global__ void __launch_bounds__(256) vec_gram_kernel(GramPtrs gp, int na, int64_t len,
                                                       double* part) {
  __shared__ double scratch[32];
  const int i0 = int(blockIdx.y) * kGramGA;
  const int nga = na - i0 < kGramGA ? na - i0 : kGramGA;  // block-uniform
  double acc[kGramGA][NB];
#pragma unroll
  for (int i = 0; i < kGramGA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j] = 0.0;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < len;
       q += int64_t(gridDim.x) * blockDim.x) {
    double bv[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) bv[j] = gp.b[j][q];
#pragma unroll
    for (int i = 0; i < kGramGA; ++i) {
      if (i < nga) {
        const double av = gp.a[i0 + i][q];
#pragma unroll
        for (int j = 0; j < NB; ++j) acc[i][j] = fma(av, bv[j], acc[i][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kGramGA; ++i)
    if (i < nga) {
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const double s = block_sum(acc[i][j], scratch);
        if (threadIdx.x == 0) part[(int64_t(blockIdx.x) * kGramNA + i0 + i) * NB + j] = s;
      }
    }
}

__global__ void vec_gram_fold_kernel(const double* __restrict__ part, int nblk, int na, int nb,
                                     double* out) {
  __shared__ double scratch[32];
  for (int e = 0; e < na * nb; ++e) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += part[int64_t(b) * kGramNA * nb + e];
    s = block_sum(s, scratch);
    if (threadIdx.x == 0) out[e] = s;
  }
}

__global__ void lincomb_kernel(VecPtrs vp, int count, int64_t len, double* out) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < len;
       q += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < count; ++i) s += vp.coef[i] * vp.a[i][q];
    out[q] = s;
  }
}

// gram partials: block (rb, pb, qb) accumulates a 32x32 block of A^T B over a
// row range; grid.x = row blocks.
__global__ void __launch_bounds__(256) gram_kernel(const double* __restrict__ a, int64_t pa,
                                                   const double* __restrict__ b, int64_t qb,
                                                   int64_t rows, int64_t rows_per_blk,
                                                   double* part) {
  __shared__ double as[32][33];
  __shared__ double bs[32][33];
  const int64_t p0 = int64_t(blockIdx.y) * 32, q0 = int64_t(blockIdx.z) * 32;
  const int64_t rbeg = int64_t(blockIdx.x) * rows_per_blk;
  int64_t rend = rbeg + rows_per_blk;
  if (rend > rows) rend = rows;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // ty: 0..7
  double acc[4] = {0, 0, 0, 0};
  for (int64_t r = rbeg; r < rend; r += 32) {
    for (int q = threadIdx.x; q < 32 * 32; q += 256) {
      const int rr = q / 32, cc = q % 32;
      const int64_t gr = r + rr;
      as[rr][cc] = (gr < rend && p0 + cc < pa) ? a[gr * pa + p0 + cc] : 0.0;
      bs[rr][cc] = (gr < rend && q0 + cc < qb) ? b[gr * qb + q0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const double bv = bs[rr][tx];
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] = fma(as[rr][ty * 4 + e], bv, acc[e]);
    }
    __syncthreads();
  }
  // part layout: [row block][pa][qb]
  for (int e = 0; e < 4; ++e) {
    const int64_t pi = p0 + ty * 4 + e, qj = q0 + tx;
    if (pi < pa && qj < qb) part[(int64_t(blockIdx.x) * pa + pi) * qb + qj] = acc[e];
  }
}

__global__ void gram_fold_kernel(const double* __restrict__ part, int nblk, int64_t pq,
                                 double* out) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < pq;
       q += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[int64_t(b) * pq + q];
    out[q] = s;
  }
}

__global__ void matmul_small_kernel(const double* __restrict__ a, int64_t rows, int64_t pa,
                                    const double* __restrict__ mm, int64_t qb, double* c) {
  const int64_t total = rows * qb;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / qb, j = q % qb;
    double s = 0.0;
    for (int64_t l = 0; l < pa; ++l) s = fma(a[r * pa + l], mm[l * qb + j], s);
    c[q] = s;
  }
}

}  // namespace spcp
