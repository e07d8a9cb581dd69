// spcp_api.cu — C ABI (include/spcp_b200.h) over the sm_100a kernels.
//
// Owns the device copy of the problem (ProblemSpec, objective.py:20-59): X in
// a padded row-major layout (rows to 128, columns to 64, zero pads so padded
// entries contribute r = 0), the bit-packed observation mask and the
// workspaces of the fused streaming pass.  Every call is stream-ordered on the
// problem's stream; results that the reference returns as Python floats come
// back through a pinned host buffer after one stream synchronisation.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "aux_kernels.cuh"
#include "common.cuh"
#include "line.cuh"
#include "sddmm.cuh"
#include "stream_f64mma.cuh"
#include "stream_f64.cuh"
#include "stream_simt.cuh"
#include "stream_tc.cuh"

namespace spcp {

// Launch with programmatic stream serialization (PDL): the kernel may start
// launching while its predecessor drains; it calls griddepcontrol.wait before
// touching the predecessor's results.  SPCP_PDL=0 turns it off.
// Environment switches are read once per process (thread-safe static
// initialisation), never per launch.
static std::string env_str(const char* name) {
  const char* e = getenv(name);
  return e ? std::string(e) : std::string();
}
static bool pdl_enabled() {
  static const bool on = env_str("SPCP_PDL") != "0";
  return on;
}

// Per-device caches of one-time launch setup (kernel attributes, occupancy):
// cudaFuncSetAttribute applies to the current device only, so a process that
// drives several GPUs must set it once per device.  Zero = not yet set.
constexpr int kMaxDevices = 64;
using DevFlags = std::atomic<int>[kMaxDevices];
static int dev_slot(int device) { return device >= 0 && device < kMaxDevices ? device : 0; }
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}


static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
bool debug_sync() {
  static const bool v = env_str("SPCP_DEBUG_SYNC") == "1";
  return v;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  return SPCP_ERR_CUDA;
}

// ------------------------------------------------------------------ buffers
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t want) {
    if (want <= bytes) return SPCP_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(workspace)");
    bytes = want;
    return SPCP_OK;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(ptr);
  }
};

}  // namespace spcp

struct spcp_problem {
  int device = 0;
  int64_t m = 0, n = 0, n_total = 0, col0 = 0;
  int64_t m_pad = 0, n_pad = 0, ldx = 0, ldm = 0;
  bool masked = false;
  double lambda_l = 1.0, lambda_s = 1.0;
  cudaStream_t stream = nullptr;
  double f_zero = 0.0, n_obs = 0.0;
  unsigned stored = 0;
  spcp::DevBuf x32, x64, mbits;
  // workspaces
  spcp::DevBuf uc, vc, wr, wl, pleft, pright, pphi, blk, out_dev, counter, scratch, scal,
      gu_tmp, vec_part, small;
  double* host_out = nullptr;  // pinned [64]
  // profiling
  bool prof = false;
  // ring of (start, end) event pairs around the fused kernel: stream-ordered
  // evaluations keep recording; pairs are folded when the ring is full and on read
  static constexpr int kEvRing = 64;
  cudaEvent_t ev0[kEvRing] = {}, ev1[kEvRing] = {};
  int ev_head = 0, ev_count = 0;
  double prof_ms = 0.0;
  int64_t prof_count = 0;
  int64_t launches = 0;
  // tensor-core streaming path (fp32, k <= 64)
  bool tc_ready = false;
  int tc_grid = 0, tc_runs = 0, tc_slots = 0;
  int64_t tc_nsb = 0, tc_ntc = 0;
  CUtensorMap tc_xmap, tc_mmap;
  spcp::DevBuf tc_units, tc_begin, tc_csr, tc_uimg, tc_vimg, tc_scales, tc_bmax;
  int64_t tc_csr_u_off = 0, tc_csr_u_idx = 0, tc_csr_v_off = 0, tc_csr_v_idx = 0;
  int64_t tc_max_u_src = 0, tc_max_v_src = 0;  // largest CSR source lists (reduce sizing)
  int tc_nbmax = 0;                             // blocks of the last tc_max launch
  // sparse-observation path (sddmm.cuh): observed entries in CSR and CSC
  bool sddmm = false, sddmm32 = false;  // built; used by fp32 evaluations too
  int64_t nnz = 0;
  spcp::DevBuf csr_ptr, csr_idx, csr_v32, csr_v64, csc_ptr, csc_idx, csc_v32, csc_v64;
  // one large workspace shared by the stored ray (line.cuh: R0, D1, D2) and the
  // stored gradient (spcp_grad_store); kept between uses (cudaMalloc / cudaFree
  // of tens of GB measured 25-500 ms each), freed by spcp_workspace_trim or
  // spcp_problem_destroy
  spcp::DevBuf big, line_part;
  bool line_ready = false;
  // stored G of one iterate (spcp_grad_store): the certificate's products
  int gstore_type = -1;
  double line_zz = 0.0, line_zd = 0.0, line_dd = 0.0;
};

namespace spcp {

// ------------------------------------------------------------------ dispatch
template <typename T>
struct DT;
template <>
struct DT<float> {
  static constexpr int id = SPCP_F32;
};
template <>
struct DT<double> {
  static constexpr int id = SPCP_F64;
};

struct LaunchShape {
  int nphi = 0;  // > 0: number of objective partials (overrides the layout's count)
  int nchunks = 1, nrb = 1;
  int64_t chunk_cols = 0;
  int tc = 0;  // partials in the tensor-core (CSR slot) layout
  int kst = 0;
  int gt_rows = 64;
  int chunked = 0;
};

static int prof_fold(spcp_problem* p, int n);
static int prof_begin(spcp_problem* p) {
  if (p->ev_count == spcp_problem::kEvRing && prof_fold(p, 1)) return SPCP_ERR_CUDA;
  SPCP_CUDA(cudaEventRecord(p->ev0[p->ev_head], p->stream));
  return SPCP_OK;
}
static int prof_end(spcp_problem* p) {
  SPCP_CUDA(cudaEventRecord(p->ev1[p->ev_head], p->stream));
  p->ev_head = (p->ev_head + 1) % spcp_problem::kEvRing;
  p->ev_count++;
  return SPCP_OK;
}

// Column chunks per row band for the (band x chunk) grids of the streaming
// kernels: the smallest count whose last wave is nearly full (waste < 5% of
// the resident slots) with at least `min_waves` waves and >= 2 tiles per
// chunk.  (C2 in fp64: 157 bands; 2 chunks gave 2.12 waves of one-CTA-per-SM
// blocks, a third wave 12% full.)
static int64_t pick_chunks(int64_t nrb, int64_t ntiles, int per_sm, int min_waves) {
  const int64_t slots = int64_t(kSMs) * std::max(per_sm, 1);
  const int64_t cap = std::max<int64_t>(1, ntiles / 2);
  int64_t best = std::min<int64_t>(cap, std::max<int64_t>(1, ceil_div(slots * min_waves, nrb)));
  double best_waste = 1e9;
  for (int64_t nch = best; nch <= std::min<int64_t>(cap, best + 64); ++nch) {
    const int64_t per = ceil_div(ntiles, nch);
    const int64_t real = ceil_div(ntiles, per);  // chunks actually launched
    const int64_t u = real * nrb;
    const double waste = double(ceil_div(u, slots) * slots) / double(u) - 1.0;
    if (waste < best_waste - 1e-12) {
      best_waste = waste;
      best = nch;
    }
    if (waste < 0.05) break;
  }
  return best;
}

template <typename T, typename TX, int KR, int PW, int MODE, bool MASK>
static int launch_stream(spcp_problem* p, StreamParams sp, LaunchShape& shape, bool prof) {
  using G = StreamGeom<T>;
  auto kern = stream_kernel<T, TX, KR, PW, MODE, MASK>;
  constexpr size_t smem = stream_smem_bytes<T, TX, KR, PW, MODE, MASK>();
  static DevFlags occ_dev = {};  // per instantiation and device
  int occ = occ_dev[dev_slot(p->device)].load(std::memory_order_relaxed);
  if (occ == 0) {
    SPCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int o = 0;
    SPCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, G::NT, smem));
    occ = std::max(o, 1);
    occ_dev[dev_slot(p->device)].store(occ, std::memory_order_relaxed);
  }
  const int64_t nrb = p->m_pad / G::BM;
  const int64_t ntiles = p->n_pad / G::BN;
  int64_t nch = pick_chunks(nrb, ntiles, occ, 4);
  const int64_t tiles_per = ceil_div(ntiles, nch);
  nch = ceil_div(ntiles, tiles_per);
  sp.chunk_cols = tiles_per * G::BN;
  sp.nchunks = int(nch);
  shape.nchunks = int(nch);
  shape.nrb = int(nrb);
  shape.chunk_cols = sp.chunk_cols;
  // partial buffers
  int rc;
  if ((rc = p->pleft.ensure(size_t(nch) * p->m_pad * PW * sizeof(T)))) return rc;
  if ((rc = p->pright.ensure(size_t(nrb) * p->n_pad * PW * sizeof(T)))) return rc;
  if ((rc = p->pphi.ensure(size_t(nrb * nch) * sizeof(double)))) return rc;
  sp.pleft = p->pleft.ptr;
  sp.pright = p->pright.ptr;
  sp.pphi = p->pphi.as<double>();
  dim3 grid{unsigned(nch), unsigned(nrb), 1u};
  if (prof && prof_begin(p)) return SPCP_ERR_CUDA;
  kern<<<grid, G::NT, smem, p->stream>>>(sp);
  SPCP_CHECK_LAUNCH("stream_kernel");
  if (prof && prof_end(p)) return SPCP_ERR_CUDA;
  p->launches++;
  return SPCP_OK;
}

// fp64 register-blocked streaming pass (stream_f64.cuh)
template <int KP, int PW, int MODE, bool MASK, typename TX>
static int launch_f64(spcp_problem* p, StreamParams sp, LaunchShape& shape) {
  using G = F64Geom<KP, PW, MODE, TX>;
  auto kern = f64_stream_kernel<KP, PW, MODE, MASK, TX>;
  constexpr size_t smem = G::SMEM;
  static DevFlags occ_dev = {};
  int occ = occ_dev[dev_slot(p->device)].load(std::memory_order_relaxed);
  if (occ == 0) {
    SPCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int o = 0;
    SPCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, G::NT, smem));
    occ = std::max(o, 1);
    occ_dev[dev_slot(p->device)].store(occ, std::memory_order_relaxed);
  }
  const int64_t nrb = p->m_pad / G::BM;
  const int64_t ntiles = p->n_pad / G::BN;
  int64_t nch = pick_chunks(nrb, ntiles, occ, 2);
  const int64_t tiles_per = ceil_div(ntiles, nch);
  nch = ceil_div(ntiles, tiles_per);
  sp.chunk_cols = tiles_per * G::BN;
  sp.nchunks = int(nch);
  shape.nchunks = int(nch);
  shape.nrb = int(nrb);
  shape.chunk_cols = sp.chunk_cols;
  int rc;
  if ((rc = p->pleft.ensure(size_t(nch) * p->m_pad * PW * sizeof(double)))) return rc;
  if ((rc = p->pright.ensure(size_t(nrb) * p->n_pad * PW * sizeof(double)))) return rc;
  if ((rc = p->pphi.ensure(size_t(nrb * nch) * sizeof(double)))) return rc;
  sp.pleft = p->pleft.ptr;
  sp.pright = p->pright.ptr;
  sp.pphi = p->pphi.as<double>();
  dim3 grid{unsigned(nch), unsigned(nrb), 1u};
  if (p->prof && prof_begin(p)) return SPCP_ERR_CUDA;
  kern<<<grid, G::NT, smem, p->stream>>>(sp);
  SPCP_CHECK_LAUNCH("f64_stream_kernel");
  if (p->prof && prof_end(p)) return SPCP_ERR_CUDA;
  p->launches++;
  return SPCP_OK;
}

// fp64 evaluation on the FP64 tensor cores (stream_f64mma.cuh; fp32-exact X)
#ifndef SPCP_F64_MMA
#define SPCP_F64_MMA 1
#endif
template <int KP, bool MASK, bool RAW0 = false, int GOUT = 0>
static int launch_f64mma(spcp_problem* p, StreamParams sp, LaunchShape& shape) {
  using G = MmaGeom<KP>;
  auto kern = f64_mma_kernel<KP, MASK, RAW0, GOUT>;
  constexpr size_t smem = G::SMEM;
  static DevFlags attr = {};
  if (!attr[dev_slot(p->device)].load(std::memory_order_relaxed)) {
    SPCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr[dev_slot(p->device)].store(1, std::memory_order_relaxed);
  }
  const int64_t nrb = p->m_pad / G::BM;
  const int64_t ntiles = p->n_pad / G::BN;
  int64_t nch = pick_chunks(nrb, ntiles, 1, 2);
  const int64_t tiles_per = ceil_div(ntiles, nch);
  nch = ceil_div(ntiles, tiles_per);
  sp.chunk_cols = tiles_per * G::BN;
  sp.nchunks = int(nch);
  shape.nchunks = int(nch);
  shape.nrb = int(nrb);
  shape.chunk_cols = sp.chunk_cols;
  int rc;
  if ((rc = p->pphi.ensure(size_t(nrb * nch) * sizeof(double)))) return rc;
  sp.pphi = p->pphi.as<double>();
  if constexpr (GOUT == 0) {
    if ((rc = p->pleft.ensure(size_t(nch) * p->m_pad * KP * sizeof(double)))) return rc;
    if ((rc = p->pright.ensure(size_t(nrb) * p->n_pad * KP * sizeof(double)))) return rc;
    sp.pleft = p->pleft.ptr;
    sp.pright = p->pright.ptr;
  }  // GOUT: sp.pleft is the caller's G destination
  dim3 grid{unsigned(nch), unsigned(nrb), 1u};
  if (p->prof && prof_begin(p)) return SPCP_ERR_CUDA;
  kern<<<grid, G::NT, smem, p->stream>>>(sp);
  SPCP_CHECK_LAUNCH("f64_mma_kernel");
  if (p->prof && prof_end(p)) return SPCP_ERR_CUDA;
  p->launches++;
  return SPCP_OK;
}

// fused EVAL kernel widths
#define SPCP_EVAL_F32_LIST(X) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32) X(40) X(48) X(56) X(64)
// fp64: the per-row SIMT stream_kernel up to k = 32 (measured faster there:
// 4.15 vs 5.7 ms at C2), the register-blocked f64_stream_kernel above
#define SPCP_EVAL_F64_LIST(X) X(8) X(16) X(24) X(32)
#define SPCP_EVAL_F64W_LIST(X) X(40) X(48) X(56) X(64)

static int eval_kp(int dtype, int64_t k) {
  if (dtype == SPCP_F32) {
    static const int l[] = {4, 8, 12, 16, 20, 24, 28, 32, 40, 48, 56, 64};
    for (int v : l)
      if (k <= v) return v;
  } else if (k <= 64) {
    return int(round_up(k, 8));  // fp64: f64_mma_kernel / stream_kernel / f64_stream_kernel
  }
  return 0;  // beyond the fused kernels: dense fallback
}

template <typename T, typename TX, bool MASK>
static int dispatch_eval(spcp_problem* p, int kp, StreamParams sp, LaunchShape& sh) {
  bool prof = p->prof;
  (void)prof;
  if constexpr (sizeof(T) == 4) {
#define SPCP_CASE(K) \
  case K:            \
    return launch_stream<T, TX, K, K, MODE_EVAL, MASK>(p, sp, sh, prof);
    switch (kp) { SPCP_EVAL_F32_LIST(SPCP_CASE) }
#undef SPCP_CASE
  } else {
    if constexpr (std::is_same<TX, float>::value) {
      if (SPCP_F64_MMA) {  // fp32-exact X: the FP64 tensor-core pass
#define SPCP_CASE(K) \
  case K:            \
    return launch_f64mma<K, MASK>(p, sp, sh);
        switch (kp) { SPCP_CASE(8) SPCP_CASE(16) SPCP_CASE(24) SPCP_CASE(32) SPCP_CASE(40)
                      SPCP_CASE(48) SPCP_CASE(56) SPCP_CASE(64) }
#undef SPCP_CASE
      }
    }
#define SPCP_CASE(K) \
  case K:            \
    return launch_stream<T, TX, K, K, MODE_EVAL, MASK>(p, sp, sh, prof);
    switch (kp) { SPCP_EVAL_F64_LIST(SPCP_CASE) }
#undef SPCP_CASE
#define SPCP_CASE(K) \
  case K:            \
    return launch_f64<K, K, MODE_EVAL, MASK, TX>(p, sp, sh);
    switch (kp) { SPCP_EVAL_F64W_LIST(SPCP_CASE) }
#undef SPCP_CASE
  }
  return fail(SPCP_ERR_UNSUPPORTED, "no fused kernel for this rank bound");
}

// APPLY / RAW widths: fp32 SIMT stream_kernel (k <= 32), fp64 f64_stream_kernel (k <= 64)
static int apply_kr(int64_t k) {
  if (k == 0) return 0;
  if (k <= 32) return int(round_up(k, 8));
  return -1;
}
// fp32 products (the certificate's subspace iteration): k <= 64
static int apply_kr32(int64_t k) {
  if (k <= 32) return apply_kr(k);
  if (k <= 64) return int(round_up(k, 16));
  return -1;
}
static int apply_kr64(int64_t k) {
  if (k <= 32) return apply_kr(k);
  if (k <= 64) return int(round_up(k, 16));
  return -1;
}

// rank widths {8, 16, 24, 32} x product widths {8, 16, 32} for the SIMT
// stream_kernel (the certificate's subspace blocks are 16 wide, C2's k = 20
// pads to 24: each padding step is a third of the kernel's FMAs)
#define SPCP_AP_LIST(AP)                                                                 \
  AP(0, 8) AP(0, 16) AP(0, 32) AP(8, 8) AP(8, 16) AP(8, 32) AP(16, 8) AP(16, 16) AP(16, 32) \
      AP(24, 8) AP(24, 16) AP(24, 32) AP(32, 8) AP(32, 16) AP(32, 32)
template <typename T, typename TX, bool MASK>
static int dispatch_apply(spcp_problem* p, int kr, int pw, StreamParams sp, LaunchShape& sh) {
#define SPCP_AP(KR, PW)                                                            \
  if (kr == KR && pw == PW)                                                      \
    return KR == 0 ? launch_stream<T, TX, 0, PW, MODE_RAW, MASK>(p, sp, sh, false) \
                   : launch_stream<T, TX, KR, PW, MODE_APPLY, MASK>(p, sp, sh, false);
  SPCP_AP_LIST(SPCP_AP)
  if constexpr (sizeof(T) == 4) {  // wide ranks for the fp32 certificate products
    SPCP_AP(48, 8)
    SPCP_AP(48, 16)
    SPCP_AP(48, 32)
    SPCP_AP(64, 8)
    SPCP_AP(64, 16)
    SPCP_AP(64, 32)
  }
#undef SPCP_AP
  if constexpr (sizeof(T) == 8) {
#define SPCP_AP(KR, PW)            \
  if (kr == KR && pw == PW)      \
    return launch_f64<KR, PW, MODE_APPLY, MASK, TX>(p, sp, sh);
    SPCP_AP(48, 8)
    SPCP_AP(48, 32)
    SPCP_AP(64, 8)
    SPCP_AP(64, 32)
#undef SPCP_AP
  }
  return fail(SPCP_ERR_UNSUPPORTED, "no apply kernel for this width");
}

static inline int grid_for(int64_t total, int threads = 256, int64_t cap = 148 * 16) {
  int64_t g = ceil_div(std::max<int64_t>(total, 1), threads);
  return int(std::min<int64_t>(g, cap));
}

static int ensure_common(spcp_problem* p) {
  int rc;
  if ((rc = p->out_dev.ensure(256 * sizeof(double)))) return rc;
  if ((rc = p->counter.ensure(64))) return rc;
  if (!p->host_out) {
    SPCP_CUDA(cudaMallocHost(&p->host_out, 256 * sizeof(double)));
    SPCP_CUDA(cudaMemsetAsync(p->counter.ptr, 0, 64, p->stream));
  }
  return SPCP_OK;
}

// fold the oldest `n` recorded pairs (waits for them)
static int prof_fold(spcp_problem* p, int n) {
  for (int i = 0; i < n && p->ev_count > 0; ++i) {
    const int slot = (p->ev_head - p->ev_count + spcp_problem::kEvRing) % spcp_problem::kEvRing;
    float ms = 0.f;
    SPCP_CUDA(cudaEventSynchronize(p->ev1[slot]));
    SPCP_CUDA(cudaEventElapsedTime(&ms, p->ev0[slot], p->ev1[slot]));
    p->prof_ms += ms;
    p->prof_count++;
    p->ev_count--;
  }
  return SPCP_OK;
}
static int prof_collect(spcp_problem* p) { return prof_fold(p, p->ev_count); }

static int check_k(spcp_problem* p, int64_t k) {
  if (k < 1 || k > std::min(p->m, p->n_total))
    return fail(SPCP_ERR_DIMENSION, "rank bound k=" + std::to_string(k) + " out of range [1, " +
                                        std::to_string(std::min(p->m, p->n_total)) + "]");
  return SPCP_OK;
}

// Run prep + fused kernel; fills the partial buffers. kp == 0: dense fallback
// (G materialised in float64, then RAW products), used for large rank bounds.
static int run_stream_eval(spcp_problem* p, int64_t k, int dtype, const double* z,
                           const double* dz, double alpha, int& kp_used, LaunchShape& sh,
                           int& part_dtype);

template <typename T>
static int prep(spcp_problem* p, int64_t k, int kp, const double* z, const double* dz,
                double alpha) {
  int rc;
  if ((rc = p->uc.ensure(size_t(p->m_pad) * kp * sizeof(T)))) return rc;
  if ((rc = p->vc.ensure(size_t(p->n_pad) * kp * sizeof(T)))) return rc;
  const int64_t total = (p->m_pad + p->n_pad) * kp;
  prep_operands_kernel<T><<<grid_for(total), 256, 0, p->stream>>>(
      z, dz, alpha, p->m, p->n, k, p->m_pad, p->n_pad, kp, p->uc.as<T>(), p->vc.as<T>());
  SPCP_CHECK_LAUNCH("prep_operands");
  p->launches++;
  return SPCP_OK;
}

static StreamParams base_params(spcp_problem* p, bool want_f64) {
  StreamParams sp{};
  sp.m_pad = p->m_pad;
  sp.n_pad = p->n_pad;
  sp.ldx = p->ldx;
  sp.x = want_f64 && p->x64.ptr ? p->x64.ptr : p->x32.ptr;
  sp.mbits = p->masked ? p->mbits.as<uint32_t>() : nullptr;
  sp.ldm = p->ldm;
  sp.tau = p->lambda_s;
  sp.do_left = 1;
  sp.do_right = 1;
  return sp;
}

static int dense_fallback_eval(spcp_problem* p, int64_t k, const double* z, const double* dz,
                               double alpha, LaunchShape& sh);

// ======================================================== tensor-core path
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool tc_env_enabled() {
  static const bool on = env_str("SPCP_FP32_KERNEL") != "simt";
  return on;
}

// Static schedule: tiles (sb, tc) in 2-D super-block order, exactly balanced
// contiguous ranges per CTA, run/slot bookkeeping and the CSR source lists
// the reduce kernel folds in a fixed order.
static int tc_build(spcp_problem* p) {
  if (p->tc_ready) return SPCP_OK;
  static const EncodeTiledFn enc = []() -> EncodeTiledFn {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<EncodeTiledFn>(fn);
  }();
  if (!enc) return fail(SPCP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  {
    cuuint64_t dims[2] = {cuuint64_t(p->ldx), cuuint64_t(p->m_pad)};
    cuuint64_t strides[1] = {cuuint64_t(p->ldx) * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t es[2] = {1, 1};
    // SPCP_X_L2PROMO = none | 64 | 128 | 256 (default): L2 promotion of the X stream
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    static const std::string promo_env = env_str("SPCP_X_L2PROMO");
    if (!promo_env.empty()) {
      const std::string& v = promo_env;
      promo = v == "none" ? CU_TENSOR_MAP_L2_PROMOTION_NONE
              : v == "64" ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : v == "128" ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                           : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    CUresult r = enc(&p->tc_xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p->x32.ptr, dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SPCP_ERR_CUDA, "tensor map (X) encode failed");
  }
  if (p->masked) {
    cuuint64_t dims[2] = {cuuint64_t(p->ldm), cuuint64_t(p->m_pad)};
    cuuint64_t strides[1] = {cuuint64_t(p->ldm) * 4};
    cuuint32_t box[2] = {4, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&p->tc_mmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, p->mbits.ptr, dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SPCP_ERR_CUDA, "tensor map (mask) encode failed");
  } else {
    p->tc_mmap = p->tc_xmap;  // unused
  }
  const int64_t nsb = p->m_pad / 128, ntc = p->n_pad / 64;
  if (nsb > 65535 || ntc > 65535) return fail(SPCP_ERR_UNSUPPORTED, "matrix too large for TC tiles");
  const int64_t U = nsb * ntc;
  const int G = int(std::min<int64_t>(kSMs, U));
  const double per = double(U) / G;
  int side = std::max(1, int(std::lround(std::sqrt(per))));
  const int sbr = int(std::min<int64_t>(side, nsb));
  // an even super-block width keeps every column tile on one tile parity (one
  // epilogue group) within a CTA, so G^T U slots need no per-parity split
  int64_t sbc0 = std::max<int64_t>(2, std::lround(per / sbr));
  sbc0 += sbc0 & 1;
  const int sbc = int(std::min<int64_t>(sbc0, ntc));
  std::vector<TcUnit> units;
  units.reserve(U);
  for (int64_t r0 = 0; r0 < nsb; r0 += sbr)
    for (int64_t c0 = 0; c0 < ntc; c0 += sbc)
      for (int64_t sb = r0; sb < std::min<int64_t>(r0 + sbr, nsb); ++sb)
        for (int64_t tc = c0; tc < std::min<int64_t>(c0 + sbc, ntc); ++tc) {
          TcUnit u{};
          u.sb = uint16_t(sb);
          u.tc = uint16_t(tc);
          units.push_back(u);
        }
  std::vector<int32_t> begin(G + 1);
  for (int c = 0; c <= G; ++c) begin[c] = int32_t((int64_t(c) * U) / G);
  int runs = 0, slots = 0;
  std::vector<std::vector<int32_t>> u_src(nsb), v_src(ntc);
  for (int c = 0; c < G; ++c) {
    // G^T U slot per (column tile, tile parity): the two epilogue groups take
    // alternate tiles, so every slot is written by one thread per address
    // (program order => deterministic store-then-reduce)
    std::map<int, int> slot_of;  // 2 * tc (+ parity if the tile parity varies) -> slot
    std::map<int, int> par_of;   // tc -> parity mask seen in this CTA
    for (int i = begin[c]; i < begin[c + 1]; ++i)
      par_of[units[i].tc] |= 1 << ((i - begin[c]) & 1);
    for (int i = begin[c]; i < begin[c + 1]; ++i) {
      TcUnit& u = units[i];
      const bool first = (i == begin[c]) || units[i - 1].sb != u.sb;
      const bool last = (i + 1 == begin[c + 1]) || units[i + 1].sb != u.sb;
      if (first) {
        u_src[u.sb].push_back(runs);
        ++runs;
      }
      u.gv_slot = runs - 1;
      u.flags = (first ? TCU_FIRST_OF_RUN : 0u) | (last ? TCU_LAST_OF_RUN : 0u);
      const int key = 2 * int(u.tc) + (par_of[u.tc] == 3 ? ((i - begin[c]) & 1) : 0);
      auto it = slot_of.find(key);
      if (it == slot_of.end()) {
        slot_of[key] = slots;
        v_src[u.tc].push_back(slots);
        u.gt_slot = slots++;
        u.flags |= TCU_FIRST_TOUCH;
      } else {
        u.gt_slot = it->second;
      }
    }
  }
  p->tc_max_u_src = 0;
  p->tc_max_v_src = 0;
  for (auto& v : u_src) p->tc_max_u_src = std::max<int64_t>(p->tc_max_u_src, int64_t(v.size()));
  for (auto& v : v_src) p->tc_max_v_src = std::max<int64_t>(p->tc_max_v_src, int64_t(v.size()));
  std::vector<int32_t> csr;
  p->tc_csr_u_off = 0;
  csr.push_back(0);
  for (int64_t s = 0; s < nsb; ++s) csr.push_back(csr.back() + int32_t(u_src[s].size()));
  p->tc_csr_u_idx = int64_t(csr.size());
  for (auto& v : u_src) csr.insert(csr.end(), v.begin(), v.end());
  p->tc_csr_v_off = int64_t(csr.size());
  csr.push_back(0);
  for (int64_t t = 0; t < ntc; ++t)
    csr.push_back(csr[p->tc_csr_v_off + t] + int32_t(v_src[t].size()));
  p->tc_csr_v_idx = int64_t(csr.size());
  for (auto& v : v_src) csr.insert(csr.end(), v.begin(), v.end());
  int rc;
  if ((rc = p->tc_units.ensure(units.size() * sizeof(TcUnit)))) return rc;
  if ((rc = p->tc_begin.ensure(begin.size() * sizeof(int32_t)))) return rc;
  if ((rc = p->tc_csr.ensure(csr.size() * sizeof(int32_t)))) return rc;
  if ((rc = p->tc_scales.ensure(sizeof(TcScales)))) return rc;
  SPCP_CUDA(cudaMemset(p->tc_scales.ptr, 0, sizeof(TcScales)));
  if ((rc = p->tc_bmax.ensure(2 * kTcMaxBlocks * sizeof(unsigned long long)))) return rc;
  SPCP_CUDA(cudaMemcpy(p->tc_units.ptr, units.data(), units.size() * sizeof(TcUnit),
                       cudaMemcpyHostToDevice));
  SPCP_CUDA(cudaMemcpy(p->tc_begin.ptr, begin.data(), begin.size() * sizeof(int32_t),
                       cudaMemcpyHostToDevice));
  SPCP_CUDA(cudaMemcpy(p->tc_csr.ptr, csr.data(), csr.size() * sizeof(int32_t),
                       cudaMemcpyHostToDevice));
  p->tc_grid = G;
  p->tc_runs = runs;
  p->tc_slots = slots;
  p->tc_nsb = nsb;
  p->tc_ntc = ntc;
  p->tc_ready = true;
  return SPCP_OK;
}

template <int KP16, bool MASK, int SEG = 0>
static int tc_launch(spcp_problem* p, int64_t k) {
  using C = TcCfg<KP16, MASK, SEG>;
  auto kern = tc_eval_kernel<KP16, MASK, SEG>;
  static DevFlags attr = {};  // per instantiation and device
  if (!attr[dev_slot(p->device)].load(std::memory_order_relaxed)) {
    SPCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr[dev_slot(p->device)].store(1, std::memory_order_relaxed);
  }
  TcParams tp{};
  tp.units = p->tc_units.as<TcUnit>();
  tp.cta_begin = p->tc_begin.as<int32_t>();
  tp.u_img = p->tc_uimg.as<unsigned char>();
  tp.v_img = p->tc_vimg.as<unsigned char>();
  tp.scales = p->tc_scales.as<TcScales>();
  tp.pleft = p->pleft.as<float>();
  tp.pright = p->pright.as<float>();
  tp.pphi = p->pphi.as<double>();
  // partial row stride: the K-concatenated drains write SEG columns
  tp.kstore = SEG > 0 ? SEG : int(round_up(k, 4));
#ifdef SPCP_TC_TIMESTAMPS
  static long long* dbg = nullptr;
  if (!dbg) SPCP_CUDA(cudaMalloc(&dbg, 64 * 32 * sizeof(long long)));
  SPCP_CUDA(cudaMemsetAsync(dbg, 0, 64 * 32 * sizeof(long long), p->stream));
  tp.dbg_ts = dbg;
#endif
  if (p->prof && prof_begin(p)) return SPCP_ERR_CUDA;
  SPCP_CUDA(launch_pdl(kern, dim3(p->tc_grid), dim3(C::NTHREADS), C::SMEM, p->stream, p->tc_xmap,
                       p->tc_mmap, tp));
  SPCP_CHECK_LAUNCH("tc_eval_kernel");
  if (p->prof && prof_end(p)) return SPCP_ERR_CUDA;
  p->launches++;
  return SPCP_OK;
}

template <int KP16>
static int tc_images(spcp_problem* p, int64_t k, const double* z, const double* dz,
                     double alpha) {
  constexpr int RB = KP16 * 2;
  int rc;
  if ((rc = p->tc_uimg.ensure(size_t(p->tc_nsb) * 2 * 128 * RB))) return rc;
  if ((rc = p->tc_vimg.ensure(size_t(p->tc_ntc) * 2 * 64 * RB))) return rc;
  const int64_t total = (p->m_pad + p->n_pad) * KP16;
  tc_images_kernel<KP16><<<grid_for(total), 256, 0, p->stream>>>(
      z, dz, alpha, p->m, p->n, k, p->m_pad, p->n_pad, p->tc_scales.as<TcScales>(),
      p->lambda_s, p->tc_uimg.as<unsigned char>(), p->tc_vimg.as<unsigned char>(),
      p->tc_bmax.as<unsigned long long>(), p->tc_nbmax);
  SPCP_CHECK_LAUNCH("tc_images");
  p->launches++;
  return SPCP_OK;
}

template <int SEG>
static int tc_images_kc(spcp_problem* p, int64_t k, const double* z, const double* dz,
                        double alpha) {
  using C = TcCfg<16, false, SEG>;
  int rc;
  if ((rc = p->tc_uimg.ensure(size_t(p->tc_nsb) * C::U_BYTES))) return rc;
  if ((rc = p->tc_vimg.ensure(size_t(p->tc_ntc) * C::V_BYTES))) return rc;
  const int64_t total = (p->m_pad + p->n_pad) * SEG;
  SPCP_CUDA(launch_pdl(tc_images_kc_kernel<SEG>, dim3(grid_for(total)), dim3(256), 0, p->stream,
                       z, dz, alpha, p->m, p->n, k, p->m_pad, p->n_pad,
                       p->tc_scales.as<TcScales>(), p->lambda_s, p->tc_uimg.as<unsigned char>(),
                       p->tc_vimg.as<unsigned char>(), p->tc_bmax.as<unsigned long long>(),
                       p->tc_nbmax));
  SPCP_CHECK_LAUNCH("tc_images_kc");
  p->launches++;
  return SPCP_OK;
}

// 1: max + scales + images in one launch (tc_prep_kc); 0: tc_max + tc_images_kc.
// Measured same-box: no gain at C2 (0.415 ms steps either way), C1 steps
// 0.032 -> 0.038 ms (the grid barrier), so 0.
#ifndef SPCP_TC_PREP_FUSED
#define SPCP_TC_PREP_FUSED 0
#endif
// max + scales + images in one launch (tc_prep_kc_kernel: grid barrier, so
// the grid is sized to be fully resident)
template <int SEG>
static int tc_prep_kc(spcp_problem* p, int64_t k, const double* z, const double* dz,
                      double alpha) {
  using C = TcCfg<16, false, SEG>;
  int rc;
  if ((rc = ensure_common(p))) return rc;
  if ((rc = p->tc_uimg.ensure(size_t(p->tc_nsb) * C::U_BYTES))) return rc;
  if ((rc = p->tc_vimg.ensure(size_t(p->tc_ntc) * C::V_BYTES))) return rc;
  static DevFlags occ_dev = {};
  int per_sm = occ_dev[dev_slot(p->device)].load(std::memory_order_relaxed);
  if (per_sm == 0) {
    SPCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tc_prep_kc_kernel<SEG>, 256,
                                                            0));
    per_sm = std::max(1, std::min(per_sm, 4));
    occ_dev[dev_slot(p->device)].store(per_sm, std::memory_order_relaxed);
  }
  unsigned* ctr = p->counter.as<unsigned>();
  SPCP_CUDA(launch_pdl(tc_prep_kc_kernel<SEG>, dim3(kSMs * per_sm), dim3(256), 0, p->stream, z,
                       dz, alpha, p->m, p->n, k, p->m_pad, p->n_pad, p->tc_scales.as<TcScales>(),
                       p->lambda_s, p->tc_uimg.as<unsigned char>(),
                       p->tc_vimg.as<unsigned char>(), ctr + 4, ctr + 5));
  SPCP_CHECK_LAUNCH("tc_prep_kc");
  p->launches++;
  return SPCP_OK;
}

// K-concatenated layout (k <= 32): SEG = round_up(k, 4) up to 20; k = 21..32
// take SEG = 32 with one-atom rows (TcCfg::REUSE: the third K-segment re-reads
// the stored ones).  (Storing the third segment as a second atom left two X
// stages and one U buffer in shared memory: 0.68 vs 0.59 ms at C4.)
static bool tc_use_kc(int64_t k) {
  static const bool split = env_str("SPCP_TC_LAYOUT") == "split";
  return k <= 32 && !split;
}
static int kc_seg(int64_t k) { return k <= 20 ? int(round_up(k, 4)) : 32; }

#define SPCP_KC_SEGS(X) X(4) X(8) X(12) X(16) X(20) X(32)
template <bool MASK>
static int tc_launch_kc(spcp_problem* p, int64_t k) {
  switch (kc_seg(k)) {
#define SPCP_KC_CASE(S) \
    case S: return tc_launch<16, MASK, S>(p, k);
    SPCP_KC_SEGS(SPCP_KC_CASE)
#undef SPCP_KC_CASE
  }
  return fail(SPCP_ERR_UNSUPPORTED, "no K-concatenated kernel for this rank bound");
}

static int tc_eval(spcp_problem* p, int64_t k, const double* z, const double* dz, double alpha,
                   LaunchShape& sh) {
  int rc;
  if ((rc = tc_build(p))) return rc;
  if (tc_use_kc(k)) {
#if SPCP_TC_PREP_FUSED
    switch (kc_seg(k)) {
#define SPCP_KC_CASE(S) \
      case S: rc = tc_prep_kc<S>(p, k, z, dz, alpha); break;
      SPCP_KC_SEGS(SPCP_KC_CASE)
#undef SPCP_KC_CASE
      default: rc = fail(SPCP_ERR_UNSUPPORTED, "no K-concatenated image kernel");
    }
#else
    const int64_t nu = p->m * k, nv = p->n * k;
    p->tc_nbmax = int(grid_for(nu + nv, 1024, kTcMaxBlocks));
    SPCP_CUDA(launch_pdl(tc_max_kernel, dim3(p->tc_nbmax), dim3(256), 0, p->stream, z, dz, alpha,
                         nu, nv, p->tc_bmax.as<unsigned long long>()));
    SPCP_CHECK_LAUNCH("tc_max");
    p->launches += 1;
    switch (kc_seg(k)) {
#define SPCP_KC_CASE(S) \
      case S: rc = tc_images_kc<S>(p, k, z, dz, alpha); break;
      SPCP_KC_SEGS(SPCP_KC_CASE)
#undef SPCP_KC_CASE
      default: rc = fail(SPCP_ERR_UNSUPPORTED, "no K-concatenated image kernel");
    }
#endif
    if (rc) return rc;
    const int kst = kc_seg(k);  // slot row stride: the drains write SEG columns
    if ((rc = p->pleft.ensure(size_t(p->tc_runs) * 128 * kst * sizeof(float)))) return rc;
    const int gt_rows = (SPCP_TC_GT_FOLD || kc_seg(k) == 32) ? 64 : 128;  // TcCfg::GT_FOLD
    if ((rc = p->pright.ensure(size_t(p->tc_slots) * gt_rows * kst * sizeof(float)))) return rc;
    if ((rc = p->pphi.ensure(size_t(p->tc_grid) * sizeof(double)))) return rc;
    rc = p->masked ? tc_launch_kc<true>(p, k) : tc_launch_kc<false>(p, k);
    if (rc) return rc;
    sh.tc = 1;
    sh.kst = kst;
    sh.gt_rows = gt_rows;  // 64: gh + gl parts folded in the drain
    sh.chunked = 1;
    sh.nchunks = 1;
    sh.nrb = 1;
    sh.chunk_cols = p->tc_grid;
    return SPCP_OK;
  }
  const int kp16 = k <= 16 ? 16 : (k <= 32 ? 32 : 64);
  // operand scales (max |U|, |V| of the trial point -> powers of two)
  // the maxima are zero here: zeroed at build time and reset by every fused launch
  const int64_t nu = p->m * k, nv = p->n * k;
  p->tc_nbmax = int(grid_for(nu + nv, 1024, kTcMaxBlocks));
  tc_max_kernel<<<p->tc_nbmax, 256, 0, p->stream>>>(z, dz, alpha, nu, nv,
                                                    p->tc_bmax.as<unsigned long long>());
  SPCP_CHECK_LAUNCH("tc_max");
  p->launches += 1;
  rc = kp16 == 16 ? tc_images<16>(p, k, z, dz, alpha)
                  : (kp16 == 32 ? tc_images<32>(p, k, z, dz, alpha)
                                : tc_images<64>(p, k, z, dz, alpha));
  if (rc) return rc;
  const int kst = int(round_up(k, 4));  // partials store the real rank only
  if ((rc = p->pleft.ensure(size_t(p->tc_runs) * 128 * kst * sizeof(float)))) return rc;
  if ((rc = p->pright.ensure(size_t(p->tc_slots) * 64 * kst * sizeof(float)))) return rc;
  if ((rc = p->pphi.ensure(size_t(p->tc_grid) * sizeof(double)))) return rc;
  if (p->masked)
    rc = kp16 == 16 ? tc_launch<16, true>(p, k)
                    : (kp16 == 32 ? tc_launch<32, true>(p, k) : tc_launch<64, true>(p, k));
  else
    rc = kp16 == 16 ? tc_launch<16, false>(p, k)
                    : (kp16 == 32 ? tc_launch<32, false>(p, k) : tc_launch<64, false>(p, k));
  if (rc) return rc;
  sh.tc = 1;
  sh.kst = int(round_up(k, 4));
  sh.chunked = 1;
  sh.nchunks = 1;
  sh.nrb = 1;
  sh.chunk_cols = p->tc_grid;  // phi partial count
  return SPCP_OK;
}

// ---- sparse-observation evaluation (sddmm.cuh): CSR row pass + CSC column pass
template <typename T, typename TX, int KP>
static int sddmm_launch(spcp_problem* p, LaunchShape& sh) {
  // one wave of resident blocks, grid-stride over rows / columns
  static DevFlags occ_dev = {};
  int per_sm = occ_dev[dev_slot(p->device)].load(std::memory_order_relaxed);
  if (per_sm == 0) {
    SPCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sddmm_pass_kernel<T, TX, KP>,
                                                            256, 0));
    per_sm = std::max(1, std::min(per_sm, 8));
    occ_dev[dev_slot(p->device)].store(per_sm, std::memory_order_relaxed);
  }
  const int nb = kSMs * per_sm;
  int rc;
  if ((rc = p->pphi.ensure(size_t(nb) * sizeof(double)))) return rc;
  SddmmParams a{};
  a.tau = p->lambda_s;
  const bool x64 = std::is_same<TX, double>::value;
  a.ptr = p->csr_ptr.as<int64_t>();
  a.idx = p->csr_idx.as<int32_t>();
  a.val = x64 ? p->csr_v64.ptr : p->csr_v32.ptr;
  a.own = p->uc.ptr;
  a.other = p->vc.ptr;
  a.out = p->pleft.ptr;
  a.pphi = p->pphi.as<double>();
  a.rows = p->m;
  if (p->prof && prof_begin(p)) return SPCP_ERR_CUDA;
  sddmm_pass_kernel<T, TX, KP><<<nb, 256, 0, p->stream>>>(a);
  SPCP_CHECK_LAUNCH("sddmm_pass(rows)");
  SddmmParams b = a;
  b.ptr = p->csc_ptr.as<int64_t>();
  b.idx = p->csc_idx.as<int32_t>();
  b.val = x64 ? p->csc_v64.ptr : p->csc_v32.ptr;
  b.own = p->vc.ptr;
  b.other = p->uc.ptr;
  b.out = p->pright.ptr;
  b.pphi = nullptr;
  b.rows = p->n;
  sddmm_pass_kernel<T, TX, KP><<<nb, 256, 0, p->stream>>>(b);
  SPCP_CHECK_LAUNCH("sddmm_pass(cols)");
  if (p->prof && prof_end(p)) return SPCP_ERR_CUDA;
  p->launches += 2;
  sh.nchunks = 1;
  sh.nrb = 1;
  sh.nphi = nb;
  return SPCP_OK;
}

#define SPCP_SDDMM_KP(X) X(8) X(16) X(24) X(32) X(40) X(48) X(56) X(64)
template <typename T, typename TX>
static int sddmm_dispatch(spcp_problem* p, int kp, LaunchShape& sh) {
  switch (kp) {
#define SPCP_SD_CASE(K) \
    case K: return sddmm_launch<T, TX, K>(p, sh);
    SPCP_SDDMM_KP(SPCP_SD_CASE)
#undef SPCP_SD_CASE
  }
  return fail(SPCP_ERR_UNSUPPORTED, "no sparse-observation kernel for this rank bound");
}

static int sddmm_eval(spcp_problem* p, int64_t k, int dtype, const double* z, const double* dz,
                      double alpha, int& kp_used, LaunchShape& sh, int& part_dtype) {
  const int kp = int(round_up(k, 8));
  kp_used = kp;
  int rc;
  if (dtype == SPCP_F32 && p->csr_v32.ptr) {
    part_dtype = SPCP_F32;
    if ((rc = prep<float>(p, k, kp, z, dz, alpha))) return rc;
    if ((rc = p->pleft.ensure(size_t(p->m_pad) * kp * sizeof(float)))) return rc;
    if ((rc = p->pright.ensure(size_t(p->n_pad) * kp * sizeof(float)))) return rc;
    return sddmm_dispatch<float, float>(p, kp, sh);
  }
  part_dtype = SPCP_F64;
  if ((rc = prep<double>(p, k, kp, z, dz, alpha))) return rc;
  if ((rc = p->pleft.ensure(size_t(p->m_pad) * kp * sizeof(double)))) return rc;
  if ((rc = p->pright.ensure(size_t(p->n_pad) * kp * sizeof(double)))) return rc;
  return p->csr_v64.ptr ? sddmm_dispatch<double, double>(p, kp, sh)
                        : sddmm_dispatch<double, float>(p, kp, sh);
}

static int run_stream_eval(spcp_problem* p, int64_t k, int dtype, const double* z,
                           const double* dz, double alpha, int& kp_used, LaunchShape& sh,
                           int& part_dtype) {
  if (dtype == SPCP_F32 && !p->x32.ptr)
    return fail(SPCP_ERR_VALUE, "fp32 evaluation requested but no fp32 copy of X is stored");
  if (p->sddmm && k <= 64 && (dtype == SPCP_F64 || p->sddmm32))
    return sddmm_eval(p, k, dtype, z, dz, alpha, kp_used, sh, part_dtype);
  int kp = eval_kp(dtype, k);
  kp_used = kp;
  if (kp == 0) {
    part_dtype = SPCP_F64;
    return dense_fallback_eval(p, k, z, dz, alpha, sh);
  }
  int rc;
  if (dtype == SPCP_F32 && k <= 64 && tc_env_enabled()) {
    part_dtype = SPCP_F32;
    return tc_eval(p, k, z, dz, alpha, sh);
  }
  if (dtype == SPCP_F32) {
    part_dtype = SPCP_F32;
    if ((rc = prep<float>(p, k, kp, z, dz, alpha))) return rc;
    StreamParams sp = base_params(p, false);
    sp.uc = p->uc.ptr;
    sp.vc = p->vc.ptr;
    return p->masked ? dispatch_eval<float, float, true>(p, kp, sp, sh)
                     : dispatch_eval<float, float, false>(p, kp, sp, sh);
  }
  part_dtype = SPCP_F64;
  if ((rc = prep<double>(p, k, kp, z, dz, alpha))) return rc;
  StreamParams sp = base_params(p, true);
  sp.uc = p->uc.ptr;
  sp.vc = p->vc.ptr;
  if (p->x64.ptr)
    return p->masked ? dispatch_eval<double, double, true>(p, kp, sp, sh)
                     : dispatch_eval<double, double, false>(p, kp, sp, sh);
  return p->masked ? dispatch_eval<double, float, true>(p, kp, sp, sh)
                   : dispatch_eval<double, float, false>(p, kp, sp, sh);
}

// ---- dense fallback: G (float64, m_pad x ldx scratch) then RAW products
template <typename TX>
static int launch_dense(spcp_problem* p, int mode, int64_t k, const double* z, int64_t row0,
                        int64_t rows, double* l_out, double* s_out, int64_t ldo, double* pphi) {
  dim3 grid(unsigned(ceil_div(p->n, 64)), unsigned(ceil_div(rows, 64)));
  const TX* x = reinterpret_cast<const TX*>(sizeof(TX) == 8 ? p->x64.ptr : p->x32.ptr);
  const uint32_t* mb = p->masked ? p->mbits.as<uint32_t>() : nullptr;
  if (mode == 0)
    dense_kernel<TX, 0><<<grid, 256, 0, p->stream>>>(z, p->m, p->n, k, x, p->ldx, mb, p->ldm,
                                                    p->lambda_s, row0, rows, l_out, s_out, ldo,
                                                    pphi);
  else
    dense_kernel<TX, 1><<<grid, 256, 0, p->stream>>>(z, p->m, p->n, k, x, p->ldx, mb, p->ldm,
                                                    p->lambda_s, row0, rows, l_out, s_out, ldo,
                                                    pphi);
  SPCP_CHECK_LAUNCH("dense_kernel");
  p->launches++;
  return SPCP_OK;
}

static int dense_fallback_eval(spcp_problem* p, int64_t k, const double* z, const double* dz,
                               double alpha, LaunchShape& sh) {
  // trial point in float64
  int rc;
  const int64_t len = (p->m + p->n) * k;
  const int64_t len_al = round_up(len, 32);  // keep gmat 256B-aligned for cp.async16
  if ((rc = p->scratch.ensure(size_t(len_al) * sizeof(double) +
                              size_t(p->m_pad) * p->ldx * sizeof(double))))
    return rc;
  double* w = p->scratch.as<double>();
  double* gmat = w + len_al;
  {
    VecPtrs vp{};
    vp.a[0] = z;
    vp.coef[0] = 1.0;
    int cnt = 1;
    if (dz) {
      vp.a[1] = dz;
      vp.coef[1] = alpha;
      cnt = 2;
    }
    lincomb_kernel<<<grid_for(len), 256, 0, p->stream>>>(vp, cnt, len, w);
    SPCP_CHECK_LAUNCH("lincomb");
    p->launches++;
  }
  SPCP_CUDA(cudaMemsetAsync(gmat, 0, size_t(p->m_pad) * p->ldx * sizeof(double), p->stream));
  const int64_t nbx = ceil_div(p->n, 64), nby = ceil_div(p->m, 64);
  DevBuf& ph = p->pphi;
  if ((rc = ph.ensure(size_t(nbx * nby) * sizeof(double)))) return rc;
  rc = p->x64.ptr ? launch_dense<double>(p, 1, k, w, 0, p->m, gmat, nullptr, p->ldx,
                                         ph.as<double>())
                  : launch_dense<float>(p, 1, k, w, 0, p->m, gmat, nullptr, p->ldx,
                                        ph.as<double>());
  if (rc) return rc;
  // fold phi now: the RAW launches below reuse the pphi buffer
  if ((rc = p->scal.ensure(8 * sizeof(double)))) return rc;
  sum_partials_kernel<<<1, 256, 0, p->stream>>>(ph.as<double>(), int(nbx * nby),
                                                p->scal.as<double>());
  SPCP_CHECK_LAUNCH("sum_partials(phi)");
  p->launches++;
  // products G V and G^T U through the RAW streaming kernel over gmat, in
  // column blocks of 32 of the rank dimension
  const int64_t nrb = p->m_pad / 128;
  const int64_t ncb = ceil_div(k, 32);
  // partial outputs laid out as the fused kernel's: pleft [1][m_pad][kp], pright [nrb][n_pad][kp]
  const int kp = int(round_up(k, 2));
  if ((rc = p->gu_tmp.ensure(size_t(p->m_pad) * kp * sizeof(double) +
                             size_t(nrb) * p->n_pad * kp * sizeof(double))))
    return rc;
  double* pl = p->gu_tmp.as<double>();
  double* pr = pl + p->m_pad * kp;
  if ((rc = p->wr.ensure(size_t(p->n_pad) * 32 * sizeof(double)))) return rc;
  if ((rc = p->wl.ensure(size_t(p->m_pad) * 32 * sizeof(double)))) return rc;
  if ((rc = p->small.ensure(size_t(std::max(p->m_pad, p->n_pad)) * 32 * sizeof(double)))) return rc;
  for (int64_t cb = 0; cb < ncb; ++cb) {
    const int64_t c0 = cb * 32, bw = std::min<int64_t>(32, k - c0);
    // operands: columns c0..c0+bw of V (for G V) and of U (for G^T U)
    // gather via matmul_small with a selection matrix is overkill; use a strided copy
    SPCP_CUDA(cudaMemsetAsync(p->wr.ptr, 0, size_t(p->n_pad) * 32 * sizeof(double), p->stream));
    SPCP_CUDA(cudaMemsetAsync(p->wl.ptr, 0, size_t(p->m_pad) * 32 * sizeof(double), p->stream));
    SPCP_CUDA(cudaMemcpy2DAsync(p->wr.ptr, 32 * sizeof(double), w + p->m * k + c0,
                                k * sizeof(double), bw * sizeof(double), p->n,
                                cudaMemcpyDeviceToDevice, p->stream));
    SPCP_CUDA(cudaMemcpy2DAsync(p->wl.ptr, 32 * sizeof(double), w + c0, k * sizeof(double),
                                bw * sizeof(double), p->m, cudaMemcpyDeviceToDevice, p->stream));
    StreamParams sp{};
    sp.m_pad = p->m_pad;
    sp.n_pad = p->n_pad;
    sp.ldx = p->ldx;
    sp.x = gmat;
    sp.mbits = nullptr;
    sp.ldm = 0;
    sp.tau = p->lambda_s;
    sp.wr = p->wr.ptr;
    sp.wl = p->wl.ptr;
    sp.do_left = 1;
    sp.do_right = 1;
    LaunchShape s2;
    if ((rc = launch_stream<double, double, 0, 32, MODE_RAW, false>(p, sp, s2, false))) return rc;
    // fold partials of this column block into pl / pr column slots c0..c0+bw
    // (pl: one chunk; pr: per row band) — reduce chunks now into pl
    double* srcl = p->pleft.as<double>();
    double* srcr = p->pright.as<double>();
    // sum chunks of the left partial: use reduce_apply into small, then scatter
    reduce_apply_kernel<double><<<grid_for(p->m * bw), 256, 0, p->stream>>>(
        srcl, s2.nchunks, p->m, p->m_pad, 32, bw, p->small.as<double>());
    SPCP_CHECK_LAUNCH("reduce_apply");
    p->launches++;
    SPCP_CUDA(cudaMemcpy2DAsync(pl + c0, kp * sizeof(double), p->small.ptr, bw * sizeof(double),
                                bw * sizeof(double), p->m, cudaMemcpyDeviceToDevice, p->stream));
    reduce_apply_kernel<double><<<grid_for(p->n * bw), 256, 0, p->stream>>>(
        srcr, s2.nrb, p->n, p->n_pad, 32, bw, p->small.as<double>());
    SPCP_CHECK_LAUNCH("reduce_apply");
    p->launches++;
    SPCP_CUDA(cudaMemcpy2DAsync(pr + c0, kp * sizeof(double), p->small.ptr, bw * sizeof(double),
                                bw * sizeof(double), p->n, cudaMemcpyDeviceToDevice, p->stream));
  }
  // expose as a one-chunk / one-band partial set in pleft/pright
  int rc2;
  if ((rc2 = p->pleft.ensure(size_t(p->m_pad) * kp * sizeof(double)))) return rc2;
  if ((rc2 = p->pright.ensure(size_t(p->n_pad) * kp * sizeof(double)))) return rc2;
  SPCP_CUDA(cudaMemcpyAsync(p->pleft.ptr, pl, size_t(p->m_pad) * kp * sizeof(double),
                            cudaMemcpyDeviceToDevice, p->stream));
  SPCP_CUDA(cudaMemcpyAsync(p->pright.ptr, pr, size_t(p->n_pad) * kp * sizeof(double),
                            cudaMemcpyDeviceToDevice, p->stream));
  // one phi partial: the folded dense value
  if ((rc2 = p->pphi.ensure(sizeof(double)))) return rc2;
  SPCP_CUDA(cudaMemcpyAsync(p->pphi.ptr, p->scal.ptr, sizeof(double), cudaMemcpyDeviceToDevice,
                            p->stream));
  sh.nchunks = 1;
  sh.nrb = 1;
  sh.chunk_cols = 1;  // phi partial count seen by run_reduce (dense path)
  return SPCP_OK;
}

static int run_reduce(spcp_problem* p, int64_t k, int kp, int part_dtype, const LaunchShape& sh,
                      bool dense, const double* z, const double* dz, double alpha, int u_mode,
                      int v_mode, const void* gu_sum, void* gu_part, const double* scal_sum,
                      double* scal_out, double* g_out) {
  int rc;
  if ((rc = ensure_common(p))) return rc;
  const int64_t work = std::max(p->m, p->n) * k;
  const int nblk = grid_for(work, 256, 148 * 4);
  if ((rc = p->blk.ensure(size_t(nblk) * 6 * sizeof(double)))) return rc;
  ReduceParams rp{};
  rp.m = p->m;
  rp.n = p->n;
  rp.k = k;
  rp.m_pad = p->m_pad;
  rp.n_pad = p->n_pad;
  rp.kp = kp;
  rp.z = z;
  rp.dz = dz;
  rp.alpha = alpha;
  rp.lambda_l = p->lambda_l;
  rp.pleft = p->pleft.ptr;
  rp.nchunks = sh.nchunks;
  rp.pright = p->pright.ptr;
  rp.nrb = sh.nrb;
  rp.gu_sum = gu_sum;
  rp.gu_part = gu_part;
  rp.g_out = g_out;
  rp.u_mode = u_mode;
  rp.v_mode = v_mode;
  rp.blk = p->blk.as<double>();
  rp.counter = p->counter.as<unsigned>();
  rp.pphi = (u_mode == U_FROM_SUM) ? nullptr : p->pphi.as<double>();
  rp.nphi = (u_mode == U_FROM_SUM) ? 0
            : sh.nphi > 0 ? sh.nphi
                          : (dense ? int(sh.chunk_cols) : sh.nchunks * sh.nrb);
  rp.scal_sum = scal_sum;
  rp.scal_out = scal_out;
  rp.out = p->out_dev.as<double>();
  if (sh.tc) {
    const int32_t* csr = p->tc_csr.as<int32_t>();
    rp.nphi = (u_mode == U_FROM_SUM) ? 0 : int(sh.chunk_cols);
    rp.csr_u_off = csr + p->tc_csr_u_off;
    rp.csr_u_idx = csr + p->tc_csr_u_idx;
    rp.csr_v_off = csr + p->tc_csr_v_off;
    rp.csr_v_idx = csr + p->tc_csr_v_idx;
    rp.kst = sh.kst;
    rp.gt_rows = sh.gt_rows;
    rp.chunked = sh.chunked;
    rp.tc_unscale = &p->tc_scales.as<TcScales>()->gv_unscale;
  }
  // One block per sub-band / column tile (tc_fold_kernel) vs the LPI kernel.
  // First measured mid-round (C2 step 0.412 vs 0.415 ms, C4 0.678 vs 0.701, C3
  // k = 5 0.223 vs 0.213, C1 0.034 vs 0.032).
  // Re-measured with the final fused kernel (`gpurun_out/r2bf_configs.txt`,
  // same box, two rounds): C2 step 0.391 vs 0.395 ms, C4 0.620 vs 0.643, C3 and
  // C5 within noise, C1 0.034 vs 0.032 — on by default above 2^24 entries
  // (SPCP_TC_FOLD=0 / 1 forces it off / on).
  static const std::string fold_s = env_str("SPCP_TC_FOLD");
  const bool fold_env = fold_s == "1" || (fold_s != "0" && p->m * p->n >= (int64_t(1) << 24));
  if (sh.tc && sh.chunked && (u_mode == U_FULL || u_mode == U_PARTIAL) && v_mode && fold_env &&
      p->tc_max_u_src <= kFoldMaxSrc && p->tc_max_v_src <= kFoldMaxSrc) {
    // one block per sub-band / column tile (tc_fold_kernel)
    const int nb = int(p->tc_nsb + p->tc_ntc);
    if ((rc = p->blk.ensure(size_t(nb) * 6 * sizeof(double)))) return rc;
    rp.blk = p->blk.as<double>();
    SPCP_CUDA(launch_pdl(tc_fold_kernel, dim3(nb), dim3(256), 0, p->stream, rp, int(p->tc_nsb)));
  } else if (sh.tc && (u_mode == U_FULL || u_mode == U_PARTIAL) && v_mode) {
// lanes per output item from the largest source count of each side:
    // about four partial loads per lane, a power of two in [1, 32]
    auto lanes = [](int64_t loads) {
      int lp = 1;
      while (lp < 32 && loads > 4 * lp) lp <<= 1;
      return lp;
    };
    const int lp_u = lanes(p->tc_max_u_src);
    const int lp_v = lanes(p->tc_max_v_src * (sh.gt_rows == 128 ? 2 : 1));
    const int64_t items = (p->m + p->n) * (sh.kst / 4);
    const int lp = std::max(lp_u, lp_v);
    // balanced sources: one item space at 2 lanes per item (measured best for
    // C2); skewed sources (tall-skinny C3 / C5 shards): per-side lane counts
#ifdef SPCP_REDUCE_FORCE_LPI2
    const bool skewed = false;
#else
    const bool skewed = std::max(lp_u, lp_v) >= 8 * std::min(lp_u, lp_v);  // C3: 1 vs 32
#endif
    // balanced: SPCP_REDUCE_LPI = 2 (default) or 4 lanes per item
    static const int lpi_env = env_str("SPCP_REDUCE_LPI") == "4" ? 4 : 2;
    const int lanes_used = skewed ? lp : lpi_env;
    const int kind = skewed ? 2 : (lpi_env == 4 ? 1 : 0);
    // one wave of resident blocks (grid-stride over the items): a partial
    // second wave left ~1/3 of the SM time idle (ncu, C2)
    static std::atomic<int> resident[kMaxDevices][3] = {};
    int res = resident[dev_slot(p->device)][kind].load(std::memory_order_relaxed);
    if (!res) {
      int per_sm = 0;
      cudaError_t e = kind == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                      &per_sm, tc_reduce_kernel, 256, 0)
                    : kind == 1 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                      &per_sm, tc_reduce_lpi_kernel<4>, 256, 0)
                                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                      &per_sm, tc_reduce_lpi_kernel<2>, 256, 0);
      if (e != cudaSuccess || per_sm < 1) per_sm = 4;
      res = per_sm * kSMs;
      resident[dev_slot(p->device)][kind].store(res, std::memory_order_relaxed);
    }
    const int nb = int(std::min<int64_t>((items * lanes_used + 255) / 256, res));
    if ((rc = p->blk.ensure(size_t(nb) * 6 * sizeof(double)))) return rc;
    rp.blk = p->blk.as<double>();  // (ensure may have grown the buffer)
    if (kind == 2)
      SPCP_CUDA(launch_pdl(tc_reduce_kernel, dim3(nb), dim3(256), 0, p->stream, rp, lp_u, lp_v));
    else if (kind == 1)
      SPCP_CUDA(launch_pdl(tc_reduce_lpi_kernel<4>, dim3(nb), dim3(256), 0, p->stream, rp));
    else
      SPCP_CUDA(launch_pdl(tc_reduce_lpi_kernel<2>, dim3(nb), dim3(256), 0, p->stream, rp));
  }
  else if (part_dtype == SPCP_F32)
    reduce_kernel<float><<<nblk, 256, 0, p->stream>>>(rp);
  else
    reduce_kernel<double><<<nblk, 256, 0, p->stream>>>(rp);
  SPCP_CHECK_LAUNCH("reduce_kernel");
  p->launches++;
  return SPCP_OK;
}

static int fetch_out(spcp_problem* p, double* out) {
  SPCP_CUDA(cudaMemcpyAsync(p->host_out, p->out_dev.ptr, 8 * sizeof(double),
                            cudaMemcpyDeviceToHost, p->stream));
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  if (p->prof && p->ev_count) prof_collect(p);
  std::memcpy(out, p->host_out, 8 * sizeof(double));
  return SPCP_OK;
}

}  // namespace spcp

using namespace spcp;

// k = 0 fp64 products X W_right / X^T W_left of fp32-exact X on the FP64 tensor
// cores (f64_mma_kernel<KP, MASK, RAW0>), up to 64 columns per pass (the SIMT
// RAW pass takes 32): the randomized SVD's sketches (linalg.py:77-106).
static int apply0_f64mma(spcp_problem* p, int64_t b, const double* w_right, double* left_out,
                         const double* w_left, double* right_out) {
  int rc;
  for (int64_t c0 = 0; c0 < b; c0 += 64) {
    const int64_t bw = std::min<int64_t>(64, b - c0);
    const int kp = int(round_up(bw, 8));
    if (w_right) {
      if ((rc = p->wr.ensure(size_t(p->n_pad) * kp * sizeof(double)))) return rc;
      stage_cols_kernel<double><<<grid_for(p->n_pad * kp), 256, 0, p->stream>>>(
          w_right, b, c0, bw, p->n, p->n_pad, kp, p->wr.as<double>());
      SPCP_CHECK_LAUNCH("stage_cols");
    }
    if (w_left) {
      if ((rc = p->wl.ensure(size_t(p->m_pad) * kp * sizeof(double)))) return rc;
      stage_cols_kernel<double><<<grid_for(p->m_pad * kp), 256, 0, p->stream>>>(
          w_left, b, c0, bw, p->m, p->m_pad, kp, p->wl.as<double>());
      SPCP_CHECK_LAUNCH("stage_cols");
    }
    StreamParams sp{};
    sp.m_pad = p->m_pad;
    sp.n_pad = p->n_pad;
    sp.ldx = p->ldx;
    sp.ldm = p->ldm;
    sp.tau = p->lambda_s;
    sp.x = p->x32.ptr;
    sp.mbits = p->masked ? p->mbits.as<uint32_t>() : nullptr;
    sp.uc = p->wl.ptr;  // band operand of G^T W_left
    sp.vc = p->wr.ptr;  // tile operand of G W_right
    sp.do_left = w_right != nullptr;
    sp.do_right = w_left != nullptr;
    LaunchShape sh;
#define SPCP_CASE(K)                                                              \
  case K:                                                                         \
    rc = p->masked ? launch_f64mma<K, true, true>(p, sp, sh)                      \
                   : launch_f64mma<K, false, true>(p, sp, sh);                    \
    break;
    switch (kp) {
      SPCP_CASE(8) SPCP_CASE(16) SPCP_CASE(24) SPCP_CASE(32) SPCP_CASE(40) SPCP_CASE(48)
      SPCP_CASE(56) SPCP_CASE(64)
      default: return fail(SPCP_ERR_UNSUPPORTED, "apply width");
    }
#undef SPCP_CASE
    if (rc) return rc;
    if ((rc = p->small.ensure(size_t(std::max(p->m, p->n)) * 64 * sizeof(double)))) return rc;
    if (w_right) {
      reduce_apply_kernel<double><<<grid_for(p->m * bw), 256, 0, p->stream>>>(
          p->pleft.as<double>(), sh.nchunks, p->m, p->m_pad, kp, bw, p->small.as<double>());
      SPCP_CHECK_LAUNCH("reduce_apply");
      p->launches++;
      SPCP_CUDA(cudaMemcpy2DAsync(left_out + c0, b * sizeof(double), p->small.ptr,
                                  bw * sizeof(double), bw * sizeof(double), p->m,
                                  cudaMemcpyDeviceToDevice, p->stream));
    }
    if (w_left) {
      reduce_apply_kernel<double><<<grid_for(p->n * bw), 256, 0, p->stream>>>(
          p->pright.as<double>(), sh.nrb, p->n, p->n_pad, kp, bw, p->small.as<double>());
      SPCP_CHECK_LAUNCH("reduce_apply");
      p->launches++;
      SPCP_CUDA(cudaMemcpy2DAsync(right_out + c0, b * sizeof(double), p->small.ptr,
                                  bw * sizeof(double), bw * sizeof(double), p->n,
                                  cudaMemcpyDeviceToDevice, p->stream));
    }
  }
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  return SPCP_OK;
}

// gstored: products with a stored G (spcp_grad_store, element type T, the X
// layout, zeros off Omega) as RAW passes instead of G from X and the factors
template <typename T>
static int apply_impl(spcp_problem* p, int64_t k, const double* z, int64_t b,
                      const double* w_right, double* left_out, const double* w_left,
                      double* right_out, const void* gstored = nullptr) {
  int rc;
  if (k < 0 || b < 1) return fail(SPCP_ERR_DIMENSION, "bad apply shape");
  SPCP_CUDA(cudaSetDevice(p->device));
  const bool x64 = p->x64.ptr != nullptr;
  int kr = gstored ? 0 : (std::is_same<T, float>::value ? apply_kr32(k) : apply_kr64(k));
  // residual operands (T)
  if (kr > 0) {
    if ((rc = prep<T>(p, k, kr, z, nullptr, 0.0))) return rc;
  } else if (kr < 0) {
    // large rank bound: materialise G once, then RAW products over it
    const int64_t len = (p->m + p->n) * k;
    (void)len;
    if ((rc = p->gu_tmp.ensure(size_t(p->m_pad) * p->ldx * sizeof(double)))) return rc;
    double* gmat = p->gu_tmp.as<double>();
    SPCP_CUDA(cudaMemsetAsync(gmat, 0, size_t(p->m_pad) * p->ldx * sizeof(double), p->stream));
    const int64_t nbx = ceil_div(p->n, 64), nby = ceil_div(p->m, 64);
    if ((rc = p->pphi.ensure(size_t(nbx * nby) * sizeof(double)))) return rc;
    rc = x64 ? launch_dense<double>(p, 1, k, z, 0, p->m, gmat, nullptr, p->ldx, p->pphi.as<double>())
             : launch_dense<float>(p, 1, k, z, 0, p->m, gmat, nullptr, p->ldx, p->pphi.as<double>());
    if (rc) return rc;
  }
  if constexpr (sizeof(T) == 8) {
    if (!gstored && k == 0 && !x64 && p->x32.ptr && SPCP_F64_MMA)
      return apply0_f64mma(p, b, w_right, left_out, w_left, right_out);
  }
  for (int64_t c0 = 0; c0 < b; c0 += 32) {
    const int64_t bw = std::min<int64_t>(32, b - c0);
    int pw = bw <= 8 ? 8 : (bw <= 16 ? 16 : 32);
    if ((kr < 0 || (kr > 32 && sizeof(T) == 8)) && pw == 16)
      pw = 32;  // f64_stream_kernel / dense widths: 8, 32
    if (w_right) {
      if ((rc = p->wr.ensure(size_t(p->n_pad) * pw * sizeof(T)))) return rc;
      stage_cols_kernel<T><<<grid_for(p->n_pad * pw), 256, 0, p->stream>>>(
          w_right, b, c0, bw, p->n, p->n_pad, pw, p->wr.as<T>());
      SPCP_CHECK_LAUNCH("stage_cols");
    }
    if (w_left) {
      if ((rc = p->wl.ensure(size_t(p->m_pad) * pw * sizeof(T)))) return rc;
      stage_cols_kernel<T><<<grid_for(p->m_pad * pw), 256, 0, p->stream>>>(
          w_left, b, c0, bw, p->m, p->m_pad, pw, p->wl.as<T>());
      SPCP_CHECK_LAUNCH("stage_cols");
    }
    StreamParams sp{};
    sp.m_pad = p->m_pad;
    sp.n_pad = p->n_pad;
    sp.ldx = p->ldx;
    sp.ldm = p->ldm;
    sp.tau = p->lambda_s;
    sp.uc = p->uc.ptr;
    sp.vc = p->vc.ptr;
    sp.wr = p->wr.ptr;
    sp.wl = p->wl.ptr;
    sp.do_left = w_right != nullptr;
    sp.do_right = w_left != nullptr;
    LaunchShape sh;
    if (gstored) {
      sp.x = gstored;
      sp.mbits = nullptr;
      rc = dispatch_apply<T, T, false>(p, 0, pw, sp, sh);
    } else if (kr < 0) {
      sp.x = p->gu_tmp.ptr;
      sp.mbits = nullptr;
      rc = pw == 8 ? launch_stream<double, double, 0, 8, MODE_RAW, false>(p, sp, sh, false)
                   : launch_stream<double, double, 0, 32, MODE_RAW, false>(p, sp, sh, false);
    } else {
      sp.x = x64 ? p->x64.ptr : p->x32.ptr;
      sp.mbits = p->masked ? p->mbits.as<uint32_t>() : nullptr;
      if (std::is_same<T, float>::value) {
        sp.x = p->x32.ptr;
        rc = p->masked ? dispatch_apply<T, float, true>(p, kr, pw, sp, sh)
                       : dispatch_apply<T, float, false>(p, kr, pw, sp, sh);
      } else if (x64) {
        rc = p->masked ? dispatch_apply<T, double, true>(p, kr, pw, sp, sh)
                       : dispatch_apply<T, double, false>(p, kr, pw, sp, sh);
      } else {
        rc = p->masked ? dispatch_apply<T, float, true>(p, kr, pw, sp, sh)
                       : dispatch_apply<T, float, false>(p, kr, pw, sp, sh);
      }
    }
    if (rc) return rc;
    if ((rc = p->small.ensure(size_t(std::max(p->m, p->n)) * 32 * sizeof(double)))) return rc;
    if (w_right) {
      reduce_apply_kernel<T><<<grid_for(p->m * bw), 256, 0, p->stream>>>(
          p->pleft.as<T>(), sh.nchunks, p->m, p->m_pad, pw, bw, p->small.as<double>());
      SPCP_CHECK_LAUNCH("reduce_apply");
      p->launches++;
      SPCP_CUDA(cudaMemcpy2DAsync(left_out + c0, b * sizeof(double), p->small.ptr,
                                  bw * sizeof(double), bw * sizeof(double), p->m,
                                  cudaMemcpyDeviceToDevice, p->stream));
    }
    if (w_left) {
      reduce_apply_kernel<T><<<grid_for(p->n * bw), 256, 0, p->stream>>>(
          p->pright.as<T>(), sh.nrb, p->n, p->n_pad, pw, bw, p->small.as<double>());
      SPCP_CHECK_LAUNCH("reduce_apply");
      p->launches++;
      SPCP_CUDA(cudaMemcpy2DAsync(right_out + c0, b * sizeof(double), p->small.ptr,
                                  bw * sizeof(double), bw * sizeof(double), p->n,
                                  cudaMemcpyDeviceToDevice, p->stream));
    }
  }
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  return SPCP_OK;
}


// Sparse-observation storage (sddmm.cuh): CSR + CSC of the observed entries,
// values from the device copies of X.  Built at creation when the observed
// fraction is at most SPCP_SDDMM_DENSITY, or forced by SPCP_SDDMM=on|off (or
// the SPCP_STORE_SPARSE / SPCP_STORE_DENSE flags).  Measured crossovers against
// the dense passes at the C4 shape (tools/sddmm_probe.py,
// profiles/r02_sddmm_probe.txt): fp64 ~12% observed (the dense fp64 pass is
// FP64-bound), fp32 ~2.5% (the tensor-core pass is ~0.69 ms whatever the mask;
// the sparse passes are bound by the L2 gathers of the other factor's rows, one
// 4k-byte row per observed entry per pass).  fp64 evaluations take the sparse
// path whenever it is built, fp32 ones below kSddmmDensity32.
static constexpr double kSddmmDensity = 0.12;
static constexpr double kSddmmDensity32 = 0.025;

static int build_sddmm(spcp_problem* p) {
  int rc;
  const int64_t words = ceil_div(p->n, 32);
  DevBuf cnt;
  if ((rc = cnt.ensure(size_t(std::max(p->m, p->n)) * sizeof(int64_t)))) return rc;
  if ((rc = p->csr_ptr.ensure(size_t(p->m + 1) * sizeof(int64_t)))) return rc;
  if ((rc = p->csc_ptr.ensure(size_t(p->n + 1) * sizeof(int64_t)))) return rc;
  const uint32_t* mb = p->mbits.as<uint32_t>();
  sddmm_row_count_kernel<<<kSMs * 4, 256, 0, p->stream>>>(mb, p->ldm, p->m, words,
                                                          cnt.as<int64_t>());
  SPCP_CHECK_LAUNCH("sddmm_row_count");
  sddmm_scan_kernel<<<1, 1024, 0, p->stream>>>(cnt.as<int64_t>(), p->m, p->csr_ptr.as<int64_t>());
  SPCP_CHECK_LAUNCH("sddmm_scan(rows)");
  sddmm_col_count_kernel<<<kSMs * 4, 256, 0, p->stream>>>(mb, p->ldm, p->m, p->n,
                                                          cnt.as<int64_t>());
  SPCP_CHECK_LAUNCH("sddmm_col_count");
  sddmm_scan_kernel<<<1, 1024, 0, p->stream>>>(cnt.as<int64_t>(), p->n, p->csc_ptr.as<int64_t>());
  SPCP_CHECK_LAUNCH("sddmm_scan(cols)");
  int64_t nnz[2] = {0, 0};
  SPCP_CUDA(cudaMemcpyAsync(&nnz[0], p->csr_ptr.as<int64_t>() + p->m, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, p->stream));
  SPCP_CUDA(cudaMemcpyAsync(&nnz[1], p->csc_ptr.as<int64_t>() + p->n, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, p->stream));
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  if (nnz[0] != nnz[1]) return fail(SPCP_ERR_NUMERICAL, "sparse-observation index mismatch");
  if (nnz[0] >= (int64_t(1) << 40)) return fail(SPCP_ERR_UNSUPPORTED, "too many observations");
  const size_t nz = size_t(std::max<int64_t>(nnz[0], 1));
  if ((rc = p->csr_idx.ensure(nz * sizeof(int32_t)))) return rc;
  if ((rc = p->csc_idx.ensure(nz * sizeof(int32_t)))) return rc;
  const int g = kSMs * 4;
  if (p->x32.ptr) {
    if ((rc = p->csr_v32.ensure(nz * sizeof(float)))) return rc;
    if ((rc = p->csc_v32.ensure(nz * sizeof(float)))) return rc;
    sddmm_csr_fill_kernel<float><<<g, 256, 0, p->stream>>>(
        mb, p->ldm, p->m, p->n, p->x32.as<float>(), p->ldx, p->csr_ptr.as<int64_t>(),
        p->csr_idx.as<int32_t>(), p->csr_v32.as<float>());
    SPCP_CHECK_LAUNCH("sddmm_csr_fill");
    sddmm_csc_fill_kernel<float><<<g, 256, 0, p->stream>>>(
        mb, p->ldm, p->m, p->n, p->x32.as<float>(), p->ldx, p->csc_ptr.as<int64_t>(),
        p->csc_idx.as<int32_t>(), p->csc_v32.as<float>());
    SPCP_CHECK_LAUNCH("sddmm_csc_fill");
  }
  if (p->x64.ptr) {
    if ((rc = p->csr_v64.ensure(nz * sizeof(double)))) return rc;
    if ((rc = p->csc_v64.ensure(nz * sizeof(double)))) return rc;
    sddmm_csr_fill_kernel<double><<<g, 256, 0, p->stream>>>(
        mb, p->ldm, p->m, p->n, p->x64.as<double>(), p->ldx, p->csr_ptr.as<int64_t>(),
        p->csr_idx.as<int32_t>(), p->csr_v64.as<double>());
    SPCP_CHECK_LAUNCH("sddmm_csr_fill");
    sddmm_csc_fill_kernel<double><<<g, 256, 0, p->stream>>>(
        mb, p->ldm, p->m, p->n, p->x64.as<double>(), p->ldx, p->csc_ptr.as<int64_t>(),
        p->csc_idx.as<int32_t>(), p->csc_v64.as<double>());
    SPCP_CHECK_LAUNCH("sddmm_csc_fill");
  }
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  p->nnz = nnz[0];
  p->sddmm = true;
  return SPCP_OK;
}

// ====================================================================== ABI
template <int KP, bool MASK>
static int launch_line_mma(spcp_problem* p, dim3 grid, int64_t chunk_cols, int64_t k,
                           const double* z, const double* dz, const uint32_t* mb, double* r0,
                           size_t ld) {
  using G = LineGeom<KP, MASK>;
  auto kern = line_setup_mma_kernel<KP, MASK>;
  static DevFlags attr = {};
  if (!attr[dev_slot(p->device)].load(std::memory_order_relaxed)) {
    SPCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(G::SMEM)));
    attr[dev_slot(p->device)].store(1, std::memory_order_relaxed);
  }
  kern<<<grid, 256, G::SMEM, p->stream>>>(z, dz, p->m, p->n, p->n_pad, k, p->x32.as<float>(),
                                          p->ldx, mb, p->ldm, chunk_cols, r0, r0 + ld,
                                          r0 + 2 * ld);
  SPCP_CHECK_LAUNCH("line_setup_mma");
  p->launches++;
  return SPCP_OK;
}

extern "C" {

int spcp_abi_version(void) { return SPCP_ABI_VERSION; }
const char* spcp_last_error(void) { return g_last_error.c_str(); }

int spcp_device_count(int* out) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *out = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *out = c;
  return SPCP_OK;
}

int spcp_problem_create(spcp_problem** out, int device, int64_t m, int64_t n, const void* x,
                        int64_t ldx, int x_dtype, int x_on_device, const uint8_t* mask,
                        unsigned store, double lambda_l, double lambda_s, int64_t n_total,
                        int64_t col0, void* stream) {
  if (!out) return fail(SPCP_ERR_VALUE, "null output handle");
  *out = nullptr;
  if (m < 1 || n < 1) return fail(SPCP_ERR_DIMENSION, "X must be a non-empty 2-D matrix");
  if (ldx < n) return fail(SPCP_ERR_DIMENSION, "ldx < n");
  if (!(lambda_l > 0.0)) return fail(SPCP_ERR_VALUE, "lambda_l must be positive");
  if (!(lambda_s > 0.0)) return fail(SPCP_ERR_VALUE, "lambda_s must be positive");
  if (x_dtype != SPCP_F32 && x_dtype != SPCP_F64) return fail(SPCP_ERR_VALUE, "bad x dtype");
  if ((store & 3u) == 0) return fail(SPCP_ERR_VALUE, "store must keep fp32 and/or fp64 X");
  if (n_total < n || col0 < 0 || col0 + n > n_total)
    return fail(SPCP_ERR_DIMENSION, "bad column shard");
  SPCP_CUDA(cudaSetDevice(device));
  auto* p = new spcp_problem();
  p->device = device;
  p->m = m;
  p->n = n;
  p->n_total = n_total;
  p->col0 = col0;
  p->m_pad = round_up(m, 128);
  p->n_pad = round_up(n, 64);
  p->ldx = p->n_pad;
  p->ldm = round_up(ceil_div(p->n_pad, 32), 4);  // 16 B rows for TMA
  p->masked = mask != nullptr;
  p->lambda_l = lambda_l;
  p->lambda_s = lambda_s;
  p->stream = reinterpret_cast<cudaStream_t>(stream);
  p->stored = store & 3u;
  auto bail = [&](int rc) {
    spcp_problem_destroy(p);
    return rc;
  };
  int rc;
  const size_t xe = size_t(p->m_pad) * p->ldx;
  if (store & SPCP_STORE_F32) {
    if ((rc = p->x32.ensure(xe * sizeof(float)))) return bail(rc);
    if (cudaMemsetAsync(p->x32.ptr, 0, xe * sizeof(float), p->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "memset x32"));
  }
  if (store & SPCP_STORE_F64) {
    if ((rc = p->x64.ensure(xe * sizeof(double)))) return bail(rc);
    if (cudaMemsetAsync(p->x64.ptr, 0, xe * sizeof(double), p->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "memset x64"));
  }
  if (p->masked) {
    const size_t mb = size_t(p->m_pad) * p->ldm * sizeof(uint32_t);
    if ((rc = p->mbits.ensure(mb))) return bail(rc);
    if (cudaMemsetAsync(p->mbits.ptr, 0, mb, p->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "memset mask"));
  }
  // upload in row chunks of <= 256 MiB of source
  const size_t esz = x_dtype == SPCP_F64 ? 8 : 4;
  int64_t chunk_rows = std::max<int64_t>(1, int64_t((size_t(256) << 20) / (size_t(n) * esz)));
  chunk_rows = std::min(chunk_rows, m);
  DevBuf stage, mstage, parts;
  const int nblk = 296;
  if ((rc = parts.ensure(2 * nblk * sizeof(double)))) return bail(rc);
  if (cudaMemsetAsync(parts.ptr, 0, 2 * nblk * sizeof(double), p->stream) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "memset parts"));
  if (!x_on_device && (rc = stage.ensure(size_t(chunk_rows) * n * esz))) return bail(rc);
  if (p->masked && (rc = mstage.ensure(size_t(chunk_rows) * n))) return bail(rc);
  for (int64_t r0 = 0; r0 < m; r0 += chunk_rows) {
    const int64_t rows = std::min(chunk_rows, m - r0);
    const void* src;
    int64_t lds;
    if (x_on_device) {
      src = static_cast<const char*>(x) + size_t(r0) * ldx * esz;
      lds = ldx;
    } else {
      cudaError_t e = cudaMemcpy2DAsync(stage.ptr, n * esz,
                                        static_cast<const char*>(x) + size_t(r0) * ldx * esz,
                                        ldx * esz, n * esz, rows, cudaMemcpyHostToDevice,
                                        p->stream);
      if (e != cudaSuccess) return bail(cuda_fail(e, "upload X"));
      src = stage.ptr;
      lds = n;
    }
    const uint8_t* mrows = nullptr;
    if (p->masked) {
      cudaError_t e = cudaMemcpyAsync(mstage.ptr, mask + size_t(r0) * n, size_t(rows) * n,
                                      cudaMemcpyHostToDevice, p->stream);
      if (e != cudaSuccess) return bail(cuda_fail(e, "upload mask"));
      mrows = mstage.as<uint8_t>();
      pack_mask_kernel<<<grid_for(rows * ceil_div(n, 32)), 256, 0, p->stream>>>(
          mrows, rows, n, r0, p->mbits.as<uint32_t>(), p->ldm);
    }
    double* psq = parts.as<double>();
    if (x_dtype == SPCP_F64)
      convert_x_kernel<double><<<nblk, 256, 0, p->stream>>>(
          static_cast<const double*>(src), lds, rows, n, r0, p->x32.as<float>(),
          p->x64.as<double>(), p->ldx, mrows, psq, psq + nblk);
    else
      convert_x_kernel<float><<<nblk, 256, 0, p->stream>>>(
          static_cast<const float*>(src), lds, rows, n, r0, p->x32.as<float>(),
          p->x64.as<double>(), p->ldx, mrows, psq, psq + nblk);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && debug_sync()) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return bail(cuda_fail(e, "convert_x / pack_mask"));
    // stage buffers are reused next chunk: serialise
    e = cudaStreamSynchronize(p->stream);
    if (e != cudaSuccess) return bail(cuda_fail(e, "upload sync"));
  }
  {
    DevBuf res;
    if ((rc = res.ensure(2 * sizeof(double)))) return bail(rc);
    sum_partials_kernel<<<1, 256, 0, p->stream>>>(parts.as<double>(), nblk, res.as<double>());
    sum_partials_kernel<<<1, 256, 0, p->stream>>>(parts.as<double>() + nblk, nblk,
                                                  res.as<double>() + 1);
    double h[2];
    cudaError_t e = cudaMemcpyAsync(h, res.ptr, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                    p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    if (e != cudaSuccess) return bail(cuda_fail(e, "f_zero"));
    p->f_zero = h[0];
    p->n_obs = h[1];
  }
  if (p->masked) {
    static const std::string mode = env_str("SPCP_SDDMM");
    static const double thr = [] {
      const std::string v = env_str("SPCP_SDDMM_DENSITY");
      return v.empty() ? kSddmmDensity : atof(v.c_str());
    }();
    const double density = p->n_obs / (double(m) * double(n));
    const bool force_on = (store & SPCP_STORE_SPARSE) || (!(store & SPCP_STORE_DENSE) && mode == "on");
    const bool force_off = (store & SPCP_STORE_DENSE) || mode == "off";
    if (force_on || (!force_off && density <= thr)) {
      if ((rc = build_sddmm(p))) return bail(rc);
      p->sddmm32 = force_on || density <= kSddmmDensity32;
    }
  }
  for (int i = 0; i < spcp_problem::kEvRing; ++i) {
    SPCP_CUDA(cudaEventCreate(&p->ev0[i]));
    SPCP_CUDA(cudaEventCreate(&p->ev1[i]));
  }
  *out = p;
  return SPCP_OK;
}

int spcp_problem_destroy(spcp_problem* p) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  cudaSetDevice(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  for (DevBuf* b : {&p->x32, &p->x64, &p->mbits, &p->uc, &p->vc, &p->wr, &p->wl, &p->pleft,
                    &p->pright, &p->pphi, &p->blk, &p->out_dev, &p->counter, &p->scratch,
                    &p->scal, &p->gu_tmp, &p->vec_part, &p->small, &p->csr_ptr, &p->csr_idx,
                    &p->csr_v32, &p->csr_v64, &p->csc_ptr, &p->csc_idx, &p->csc_v32,
                    &p->csc_v64, &p->tc_units, &p->tc_begin, &p->tc_csr, &p->tc_uimg,
                    &p->tc_vimg, &p->tc_scales, &p->tc_bmax, &p->big, &p->line_part})
    b->release();
  if (p->host_out) cudaFreeHost(p->host_out);
  for (int i = 0; i < spcp_problem::kEvRing; ++i) {
    if (p->ev0[i]) cudaEventDestroy(p->ev0[i]);
    if (p->ev1[i]) cudaEventDestroy(p->ev1[i]);
  }
  delete p;
  return SPCP_OK;
}

int spcp_problem_set_stream(spcp_problem* p, void* stream) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  p->stream = reinterpret_cast<cudaStream_t>(stream);
  return SPCP_OK;
}

int spcp_problem_info(spcp_problem* p, double* info) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  info[0] = p->f_zero;
  info[1] = p->n_obs;
  info[2] = double(p->stored);
  info[3] = double(p->x32.bytes + p->x64.bytes + p->mbits.bytes);
  info[4] = p->sddmm ? double(p->nnz) : -1.0;  // observed entries on the sparse path
  return SPCP_OK;
}

static int eval_impl(spcp_problem* p, int64_t k, int dtype, const double* z, const double* dz,
                     double alpha, double* g_out, int u_mode, void* gu_part, double* scal) {
  int rc;
  if ((rc = check_k(p, k))) return rc;
  if (dtype != SPCP_F32 && dtype != SPCP_F64) return fail(SPCP_ERR_VALUE, "bad compute dtype");
  SPCP_CUDA(cudaSetDevice(p->device));
  int kp = 0, pdt = SPCP_F64;
  LaunchShape sh;
  if ((rc = run_stream_eval(p, k, dtype, z, dz, alpha, kp, sh, pdt))) return rc;
  const bool dense = (kp == 0);
  if (dense) kp = int(round_up(k, 2));
  return run_reduce(p, k, kp, pdt, sh, dense, z, dz, alpha, u_mode, 1, nullptr, gu_part,
                    nullptr, scal, g_out);
}

int spcp_eval(spcp_problem* p, int64_t k, int dtype, const double* z, const double* dz,
              double alpha, double* g_out, double* out) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc = eval_impl(p, k, dtype, z, dz, alpha, g_out, U_FULL, nullptr, nullptr);
  if (rc) return rc;
  return fetch_out(p, out);
}

int spcp_eval_async(spcp_problem* p, int64_t k, int dtype, const double* z, const double* dz,
                    double alpha, double* g_out, double* out_dev) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc = eval_impl(p, k, dtype, z, dz, alpha, g_out, U_FULL, nullptr, nullptr);
  if (rc) return rc;
  if (out_dev)
    SPCP_CUDA(cudaMemcpyAsync(out_dev, p->out_dev.ptr, 8 * sizeof(double),
                              cudaMemcpyDeviceToDevice, p->stream));
  return SPCP_OK;
}

int spcp_eval_partial(spcp_problem* p, int64_t k, int dtype, const double* z, const double* dz,
                      double alpha, void* gu_part, double* scal, double* g_out) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  return eval_impl(p, k, dtype, z, dz, alpha, g_out, U_PARTIAL, gu_part, scal);
}

int spcp_eval_finish(spcp_problem* p, int64_t k, int dtype, const double* z, const double* dz,
                     double alpha, const void* gu_sum, const double* scal_sum, double* g_out,
                     double* out) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc;
  if ((rc = check_k(p, k))) return rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  LaunchShape sh;
  const int pdt = (dtype == SPCP_F32 && eval_kp(SPCP_F32, k) != 0) ? SPCP_F32 : SPCP_F64;
  if ((rc = run_reduce(p, k, int(round_up(k, 2)), pdt, sh, false, z, dz, alpha, U_FROM_SUM, 0,
                       gu_sum, nullptr, scal_sum, nullptr, g_out)))
    return rc;
  return fetch_out(p, out);
}

int spcp_split_objective_host(spcp_problem* p, int64_t k, int dtype, const double* u,
                              const double* v, double* value, double* grad_u, double* grad_v) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc;
  if ((rc = check_k(p, k))) return rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  const int64_t nu = p->m * k, nv = p->n * k;
  if ((rc = p->scratch.ensure(size_t(nu + nv) * 2 * sizeof(double)))) return rc;
  double* z = p->scratch.as<double>();
  double* g = z + nu + nv;
  SPCP_CUDA(cudaMemcpyAsync(z, u, size_t(nu) * sizeof(double), cudaMemcpyHostToDevice, p->stream));
  SPCP_CUDA(cudaMemcpyAsync(z + nu, v, size_t(nv) * sizeof(double), cudaMemcpyHostToDevice,
                            p->stream));
  double out[8];
  if (eval_kp(dtype, k) == 0) {
    // dense fallback uses `scratch` itself: stage z elsewhere
    if ((rc = p->vec_part.ensure(size_t(nu + nv) * 2 * sizeof(double)))) return rc;
    double* z2 = p->vec_part.as<double>();
    SPCP_CUDA(cudaMemcpyAsync(z2, z, size_t(nu + nv) * sizeof(double), cudaMemcpyDeviceToDevice,
                              p->stream));
    z = z2;
    g = z2 + nu + nv;
  }
  // one stream synchronisation per call: the scalars and both gradient blocks
  // are queued behind the evaluation together (no host round trip between)
  if ((rc = eval_impl(p, k, dtype, z, nullptr, 0.0, g, U_FULL, nullptr, nullptr))) return rc;
  SPCP_CUDA(cudaMemcpyAsync(p->host_out, p->out_dev.ptr, 8 * sizeof(double),
                            cudaMemcpyDeviceToHost, p->stream));
  if (grad_u)
    SPCP_CUDA(cudaMemcpyAsync(grad_u, g, size_t(nu) * sizeof(double), cudaMemcpyDeviceToHost,
                              p->stream));
  if (grad_v)
    SPCP_CUDA(cudaMemcpyAsync(grad_v, g + nu, size_t(nv) * sizeof(double),
                              cudaMemcpyDeviceToHost, p->stream));
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  if (p->prof && p->ev_count && prof_collect(p)) return SPCP_ERR_CUDA;
  std::memcpy(out, p->host_out, 8 * sizeof(double));
  *value = out[0];
  return SPCP_OK;
}

int spcp_phi_dense_host(spcp_problem* p, const double* l, double* value, double* grad,
                        double* s_star) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  const int64_t mn = p->m * p->n;
  const int nblk = grid_for(mn, 256, 148 * 8);
  if ((rc = p->scratch.ensure(size_t(mn) * 3 * sizeof(double) + size_t(nblk) * sizeof(double))))
    return rc;
  double* dl = p->scratch.as<double>();
  double* dg = dl + mn;
  double* ds = dg + mn;
  double* part = ds + mn;
  SPCP_CUDA(cudaMemcpyAsync(dl, l, size_t(mn) * sizeof(double), cudaMemcpyHostToDevice, p->stream));
  const uint32_t* mb = p->masked ? p->mbits.as<uint32_t>() : nullptr;
  if (p->x64.ptr)
    phi_dense_kernel<double><<<nblk, 256, 0, p->stream>>>(dl, p->m, p->n, p->x64.as<double>(),
                                                          p->ldx, mb, p->ldm, p->lambda_s, dg,
                                                          ds, part);
  else
    phi_dense_kernel<float><<<nblk, 256, 0, p->stream>>>(dl, p->m, p->n, p->x32.as<float>(),
                                                         p->ldx, mb, p->ldm, p->lambda_s, dg, ds,
                                                         part);
  SPCP_CHECK_LAUNCH("phi_dense");
  p->launches++;
  if ((rc = ensure_common(p))) return rc;
  sum_partials_kernel<<<1, 256, 0, p->stream>>>(part, nblk, p->out_dev.as<double>());
  p->launches++;
  SPCP_CUDA(cudaMemcpyAsync(p->host_out, p->out_dev.ptr, sizeof(double), cudaMemcpyDeviceToHost,
                            p->stream));
  if (grad)
    SPCP_CUDA(cudaMemcpyAsync(grad, dg, size_t(mn) * sizeof(double), cudaMemcpyDeviceToHost,
                              p->stream));
  if (s_star)
    SPCP_CUDA(cudaMemcpyAsync(s_star, ds, size_t(mn) * sizeof(double), cudaMemcpyDeviceToHost,
                              p->stream));
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  *value = p->host_out[0];
  return SPCP_OK;
}

int spcp_apply(spcp_problem* p, int64_t k, const double* z, int64_t b, const double* w_right,
               double* left_out, const double* w_left, double* right_out) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  return apply_impl<double>(p, k, z, b, w_right, left_out, w_left, right_out);
}

int spcp_grad_store(spcp_problem* p, int64_t k, const double* z, int dtype) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  if (k < 1) return fail(SPCP_ERR_DIMENSION, "k must be >= 1");
  if (dtype != SPCP_F32 && dtype != SPCP_F64) return fail(SPCP_ERR_VALUE, "dtype");
  int rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  p->gstore_type = -1;
  if (!p->x64.ptr && !p->x32.ptr)
    return fail(SPCP_ERR_UNSUPPORTED, "grad_store: no dense X store (sparse-observation problem)");
  const size_t es = dtype == SPCP_F32 ? 4 : 8;
  const size_t need = size_t(p->m_pad) * size_t(p->ldx) * es;
  p->line_ready = false;  // the workspace is shared with the stored ray
  if (p->big.bytes < need) {
    p->big.release();
    size_t free_b = 0, total_b = 0;
    SPCP_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (need + (size_t(1) << 30) > free_b)
      return fail(SPCP_ERR_UNSUPPORTED, "grad_store: the m x n gradient does not fit");
    if ((rc = p->big.ensure(need))) return rc;
  }
  if (!p->x64.ptr && k <= 64 && SPCP_F64_MMA) {
    // fp32-exact X: G from the FP64 tensor-core pass's phase 1 (every entry of
    // the padded array written: pads and off-Omega entries are zeros)
    if ((rc = prep<double>(p, k, int(round_up(k, 8)), z, nullptr, 0.0))) return rc;
    StreamParams sp{};
    sp.m_pad = p->m_pad;
    sp.n_pad = p->n_pad;
    sp.ldx = p->ldx;
    sp.ldm = p->ldm;
    sp.tau = p->lambda_s;
    sp.x = p->x32.ptr;
    sp.mbits = p->masked ? p->mbits.as<uint32_t>() : nullptr;
    sp.uc = p->uc.ptr;
    sp.vc = p->vc.ptr;
    sp.pleft = p->big.ptr;
    LaunchShape sh;
    const int kp = int(round_up(k, 8));
#define SPCP_CASE(K)                                                                        \
  case K:                                                                                   \
    rc = dtype == SPCP_F32                                                                  \
             ? (p->masked ? launch_f64mma<K, true, false, 4>(p, sp, sh)                     \
                          : launch_f64mma<K, false, false, 4>(p, sp, sh))                   \
             : (p->masked ? launch_f64mma<K, true, false, 8>(p, sp, sh)                     \
                          : launch_f64mma<K, false, false, 8>(p, sp, sh));                  \
    break;
    switch (kp) {
      SPCP_CASE(8) SPCP_CASE(16) SPCP_CASE(24) SPCP_CASE(32) SPCP_CASE(40) SPCP_CASE(48)
      SPCP_CASE(56) SPCP_CASE(64)
      default: return fail(SPCP_ERR_UNSUPPORTED, "grad_store width");
    }
#undef SPCP_CASE
    if (rc) return rc;
    p->gstore_type = dtype;
    return SPCP_OK;
  }
  SPCP_CUDA(cudaMemsetAsync(p->big.ptr, 0, need, p->stream));  // pads and off-Omega rows
  const int64_t nbx = ceil_div(p->n, 64), nby = ceil_div(p->m, 64);
  if ((rc = p->pphi.ensure(size_t(nbx * nby) * sizeof(double)))) return rc;
  const dim3 grid{unsigned(nbx), unsigned(nby), 1u};
  const uint32_t* mb = p->masked ? p->mbits.as<uint32_t>() : nullptr;
#define SPCP_GS(TX, XP, TO)                                                                \
  dense_kernel<TX, 1, TO><<<grid, 256, 0, p->stream>>>(z, p->m, p->n, k, XP, p->ldx, mb,    \
                                                       p->ldm, p->lambda_s, 0, p->m,        \
                                                       p->big.as<TO>(), nullptr, p->ldx,     \
                                                       p->pphi.as<double>())
  if (p->x64.ptr) {
    if (dtype == SPCP_F32) SPCP_GS(double, p->x64.as<double>(), float);
    else SPCP_GS(double, p->x64.as<double>(), double);
  } else {
    if (dtype == SPCP_F32) SPCP_GS(float, p->x32.as<float>(), float);
    else SPCP_GS(float, p->x32.as<float>(), double);
  }
#undef SPCP_GS
  SPCP_CHECK_LAUNCH("grad_store");
  p->launches++;
  p->gstore_type = dtype;
  return SPCP_OK;
}

int spcp_apply_stored(spcp_problem* p, int64_t b, const double* w_right, double* left_out,
                      const double* w_left, double* right_out) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  if (p->gstore_type < 0) return fail(SPCP_ERR_VALUE, "apply_stored before grad_store");
  return p->gstore_type == SPCP_F32
             ? apply_impl<float>(p, 0, nullptr, b, w_right, left_out, w_left, right_out,
                                 p->big.ptr)
             : apply_impl<double>(p, 0, nullptr, b, w_right, left_out, w_left, right_out,
                                  p->big.ptr);
}

int spcp_grad_release(spcp_problem* p) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  p->gstore_type = -1;  // the memory stays with the problem (spcp_workspace_trim)
  return SPCP_OK;
}

int spcp_workspace_trim(spcp_problem* p) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  SPCP_CUDA(cudaSetDevice(p->device));
  if (p->stream) SPCP_CUDA(cudaStreamSynchronize(p->stream));
  p->big.release();
  p->gstore_type = -1;
  p->line_ready = false;
  return SPCP_OK;
}

int spcp_apply_f32(spcp_problem* p, int64_t k, const double* z, int64_t b,
                   const double* w_right, double* left_out, const double* w_left,
                   double* right_out) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  // fp32 streaming products need the fp32 copy of X and the fused widths
  if (!p->x32.ptr || apply_kr32(k) < 0)
    return apply_impl<double>(p, k, z, b, w_right, left_out, w_left, right_out);
  return apply_impl<float>(p, k, z, b, w_right, left_out, w_left, right_out);
}

int spcp_materialize(spcp_problem* p, int64_t k, const double* z, int64_t row0, int64_t rows,
                     double* l_out, double* s_out, int out_on_host) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc;
  if (row0 < 0 || rows < 0 || row0 + rows > p->m) return fail(SPCP_ERR_DIMENSION, "bad row range");
  SPCP_CUDA(cudaSetDevice(p->device));
  const bool x64 = p->x64.ptr != nullptr;
  int64_t step = rows;
  if (out_on_host) {
    step = std::max<int64_t>(1, int64_t((size_t(128) << 20) / (size_t(p->n) * 8)));
    if ((rc = p->gu_tmp.ensure(size_t(step) * p->n * 2 * sizeof(double)))) return rc;
  }
  for (int64_t r = row0; r < row0 + rows; r += step) {
    const int64_t nr = std::min(step, row0 + rows - r);
    double* lo = l_out ? (out_on_host ? p->gu_tmp.as<double>() : l_out + (r - row0) * p->n) : nullptr;
    double* so = s_out ? (out_on_host ? p->gu_tmp.as<double>() + step * p->n
                                      : s_out + (r - row0) * p->n)
                       : nullptr;
    rc = x64 ? launch_dense<double>(p, 0, k, z, r, nr, lo, so, p->n, nullptr)
             : launch_dense<float>(p, 0, k, z, r, nr, lo, so, p->n, nullptr);
    if (rc) return rc;
    if (out_on_host) {
      if (l_out)
        SPCP_CUDA(cudaMemcpyAsync(l_out + (r - row0) * p->n, lo, size_t(nr) * p->n * 8,
                                  cudaMemcpyDeviceToHost, p->stream));
      if (s_out)
        SPCP_CUDA(cudaMemcpyAsync(s_out + (r - row0) * p->n, so, size_t(nr) * p->n * 8,
                                  cudaMemcpyDeviceToHost, p->stream));
      SPCP_CUDA(cudaStreamSynchronize(p->stream));
    }
  }
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  return SPCP_OK;
}

int spcp_materialize_grad(spcp_problem* p, int64_t k, const double* z, double* g_out,
                          int64_t ldo) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc;
  if (k < 1) return fail(SPCP_ERR_DIMENSION, "k must be >= 1");
  if (ldo < p->n) return fail(SPCP_ERR_DIMENSION, "ldo < n");
  SPCP_CUDA(cudaSetDevice(p->device));
  const int64_t nbx = ceil_div(p->n, 64), nby = ceil_div(p->m, 64);
  if ((rc = p->pphi.ensure(size_t(nbx * nby) * sizeof(double)))) return rc;
  rc = p->x64.ptr ? launch_dense<double>(p, 1, k, z, 0, p->m, g_out, nullptr, ldo,
                                         p->pphi.as<double>())
                  : launch_dense<float>(p, 1, k, z, 0, p->m, g_out, nullptr, ldo,
                                        p->pphi.as<double>());
  if (rc) return rc;
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  return SPCP_OK;
}

// ---- line-restricted evaluation (line.cuh) ----------------------------------
int spcp_line_setup(spcp_problem* p, int64_t k, const double* z, const double* dz) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  if (k < 1) return fail(SPCP_ERR_DIMENSION, "k must be >= 1");
  if (!z || !dz) return fail(SPCP_ERR_VALUE, "line_setup needs z and dz");
  int rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  p->line_ready = false;
  if (!p->x64.ptr && !p->x32.ptr)
    return fail(SPCP_ERR_UNSUPPORTED, "line_setup: no dense X store (sparse-observation problem)");
  // rows of n_pad entries (zero pads): aligned double2 pairs for the probe
  const size_t per = size_t(p->m) * size_t(p->n_pad);
  const size_t ld = size_t(round_up(int64_t(per), 32));  // 256-byte aligned matrices
  const size_t need = 3 * ld * sizeof(double);
  p->gstore_type = -1;  // the workspace is shared with the stored gradient
  if (p->big.bytes < need) {
    p->big.release();
    size_t free_b = 0, total_b = 0;
    SPCP_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (need + (size_t(1) << 30) > free_b)
      return fail(SPCP_ERR_UNSUPPORTED, "line_setup: the three m x n float64 matrices do not fit");
    if ((rc = p->big.ensure(need))) return rc;
  }
  double* r0 = p->big.as<double>();
  const uint32_t* mb = p->masked ? p->mbits.as<uint32_t>() : nullptr;
  if (!p->x64.ptr && k <= 64 && SPCP_F64_MMA) {
    // fp32-exact X: the three products on the FP64 tensor cores
    const int kp = int(round_up(k, 8));
    const int64_t nrb = p->m_pad / 128, ntiles = p->n_pad / 64;
    int64_t nch = pick_chunks(nrb, ntiles, 1, 2);
    const int64_t tiles_per = ceil_div(ntiles, nch);
    nch = ceil_div(ntiles, tiles_per);
    const dim3 grid{unsigned(nch), unsigned(nrb), 1u};
#define SPCP_CASE(K)                                                                          \
  case K:                                                                                     \
    rc = p->masked ? launch_line_mma<K, true>(p, grid, tiles_per * 64, k, z, dz, mb, r0, ld) \
                   : launch_line_mma<K, false>(p, grid, tiles_per * 64, k, z, dz, mb, r0, ld); \
    break;
    switch (kp) {
      SPCP_CASE(8) SPCP_CASE(16) SPCP_CASE(24) SPCP_CASE(32) SPCP_CASE(40) SPCP_CASE(48)
      SPCP_CASE(56) SPCP_CASE(64)
      default: return fail(SPCP_ERR_UNSUPPORTED, "line_setup width");
    }
#undef SPCP_CASE
    if (rc) return rc;
  } else {
    dim3 grid(unsigned(p->n_pad / 64), unsigned(ceil_div(p->m, 64)));
    if (p->x64.ptr)
      line_setup_kernel<double><<<grid, 256, 0, p->stream>>>(
          z, dz, p->m, p->n, p->n_pad, k, p->x64.as<double>(), p->ldx, mb, p->ldm, r0, r0 + ld,
          r0 + 2 * ld);
    else
      line_setup_kernel<float><<<grid, 256, 0, p->stream>>>(
          z, dz, p->m, p->n, p->n_pad, k, p->x32.as<float>(), p->ldx, mb, p->ldm, r0, r0 + ld,
          r0 + 2 * ld);
    SPCP_CHECK_LAUNCH("line_setup");
  }
  p->launches++;
  // regulariser on the ray: |z + a dz|^2 = zz + 2 a zd + a^2 dd
  const int64_t len = (p->m + p->n) * k;
  const double* a[3] = {z, z, dz};
  const double* b[3] = {z, dz, dz};
  double dots[3];
  if ((rc = spcp_vec_multidot(p, len, 3, a, b, dots))) return rc;
  p->line_zz = dots[0];
  p->line_zd = dots[1];
  p->line_dd = dots[2];
  p->line_ready = true;
  return SPCP_OK;
}

int spcp_line_probe(spcp_problem* p, double alpha, double* out_host) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  if (!p->line_ready) return fail(SPCP_ERR_VALUE, "line_probe before line_setup");
  int rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  if ((rc = ensure_common(p))) return rc;
  const int nb = kSMs * 4;
  if ((rc = p->line_part.ensure(size_t(2 * nb) * sizeof(double)))) return rc;
  const size_t per = size_t(p->m) * size_t(p->n_pad);
  const size_t ld = size_t(round_up(int64_t(per), 32));
  const double* r0 = p->big.as<double>();
  line_probe_kernel<<<nb, 256, 0, p->stream>>>(r0, r0 + ld, r0 + 2 * ld, int64_t(per), alpha,
                                               p->lambda_s, p->line_part.as<double>());
  SPCP_CHECK_LAUNCH("line_probe");
  line_fold_kernel<<<1, 256, 0, p->stream>>>(p->line_part.as<double>(), nb,
                                             p->out_dev.as<double>());
  SPCP_CHECK_LAUNCH("line_fold");
  p->launches += 2;
  SPCP_CUDA(cudaMemcpyAsync(p->host_out, p->out_dev.ptr, 2 * sizeof(double),
                            cudaMemcpyDeviceToHost, p->stream));
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  const double phi = p->host_out[0], dphi = p->host_out[1];
  const double reg = 0.5 * p->lambda_l * (p->line_zz + alpha * (2.0 * p->line_zd + alpha * p->line_dd));
  const double dreg = p->lambda_l * (p->line_zd + alpha * p->line_dd);
  out_host[0] = phi + reg;
  out_host[1] = phi;
  out_host[2] = reg;
  out_host[3] = dphi + dreg;
  for (int i = 4; i < 8; ++i) out_host[i] = 0.0;
  return SPCP_OK;
}

int spcp_line_release(spcp_problem* p) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  SPCP_CUDA(cudaSetDevice(p->device));
  p->line_ready = false;  // the memory stays with the problem (spcp_workspace_trim)
  return SPCP_OK;
}

int spcp_vec_multidot(spcp_problem* p, int64_t len, int count, const double* const* a,
                      const double* const* b, double* out_host) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  if ((rc = ensure_common(p))) return rc;
  const int nblk = grid_for(len, 256, 148 * 2);
  for (int c0 = 0; c0 < count; c0 += kMaxVec) {
    const int cnt = std::min(kMaxVec, count - c0);
    VecPtrs vp{};
    for (int i = 0; i < cnt; ++i) {
      vp.a[i] = a[c0 + i];
      vp.b[i] = b[c0 + i];
    }
    if ((rc = p->vec_part.ensure(size_t(cnt) * nblk * sizeof(double) + 64 * sizeof(double))))
      return rc;
    double* part = p->vec_part.as<double>();
    multidot_kernel<<<dim3(nblk, cnt), 256, 0, p->stream>>>(vp, len, part, nblk);
    SPCP_CHECK_LAUNCH("multidot");
    fold_kernel<<<cnt, 256, 0, p->stream>>>(part, nblk, p->out_dev.as<double>());
    SPCP_CHECK_LAUNCH("fold");
    p->launches += 2;
    SPCP_CUDA(cudaMemcpyAsync(p->host_out, p->out_dev.ptr, cnt * sizeof(double),
                              cudaMemcpyDeviceToHost, p->stream));
    SPCP_CUDA(cudaStreamSynchronize(p->stream));
    std::memcpy(out_host + c0, p->host_out, cnt * sizeof(double));
  }
  return SPCP_OK;
}

int spcp_vec_lincomb(spcp_problem* p, int64_t len, int count, const double* coef,
                     const double* const* v, double* out) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  SPCP_CUDA(cudaSetDevice(p->device));
  if (count < 1) return fail(SPCP_ERR_VALUE, "lincomb needs >= 1 vector");
  if (count > kMaxVec) return fail(SPCP_ERR_VALUE, "lincomb: too many vectors");
  VecPtrs vp{};
  for (int i = 0; i < count; ++i) {
    vp.a[i] = v[i];
    vp.coef[i] = coef[i];
  }
  lincomb_kernel<<<grid_for(len), 256, 0, p->stream>>>(vp, count, len, out);
  SPCP_CHECK_LAUNCH("lincomb");
  p->launches++;
  return SPCP_OK;
}

static int vec_gram_impl(spcp_problem* p, int64_t len, int na, const double* const* a, int nb,
                         const double* const* b, double* out_host, double* out_dev) {
  int rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  if (nb < 1 || nb > 4 || na < 1) return fail(SPCP_ERR_VALUE, "vec_gram: need 1<=nb<=4, na>=1");
  if ((rc = ensure_common(p))) return rc;
  // one wave: the (column block x a-group) grid fills the resident slots of
  // the kernel's register budget (more blocks only add a partial second wave)
  static DevFlags occ[4] = {};
  int per_sm = occ[nb - 1][dev_slot(p->device)].load(std::memory_order_relaxed);
  if (!per_sm) {
    cudaError_t e = nb == 1 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vec_gram_kernel<1>, 256, 0)
                  : nb == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vec_gram_kernel<2>, 256, 0)
                  : nb == 3 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vec_gram_kernel<3>, 256, 0)
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vec_gram_kernel<4>, 256, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 2;
    occ[nb - 1][dev_slot(p->device)].store(per_sm, std::memory_order_relaxed);
  }
  for (int a0 = 0; a0 < na; a0 += kGramNA) {
    const int cnt = std::min(kGramNA, na - a0);
    const int ngroups = int(ceil_div(cnt, kGramGA));
    const int nblk = grid_for(len, 256, std::max<int64_t>(kSMs, int64_t(kSMs) * per_sm / ngroups));
    GramPtrs gp{};
    for (int i = 0; i < cnt; ++i) gp.a[i] = a[a0 + i];
    for (int j = 0; j < nb; ++j) gp.b[j] = b[j];
    if ((rc = p->vec_part.ensure(size_t(nblk) * kGramNA * 4 * sizeof(double)))) return rc;
    double* part = p->vec_part.as<double>();
    const dim3 grid{unsigned(nblk), unsigned(ceil_div(cnt, kGramGA)), 1u};
    switch (nb) {
      case 1: vec_gram_kernel<1><<<grid, 256, 0, p->stream>>>(gp, cnt, len, part); break;
      case 2: vec_gram_kernel<2><<<grid, 256, 0, p->stream>>>(gp, cnt, len, part); break;
      case 3: vec_gram_kernel<3><<<grid, 256, 0, p->stream>>>(gp, cnt, len, part); break;
      default: vec_gram_kernel<4><<<grid, 256, 0, p->stream>>>(gp, cnt, len, part); break;
    }
    SPCP_CHECK_LAUNCH("vec_gram");
    double* dst = out_dev ? out_dev + size_t(a0) * nb : p->out_dev.as<double>();
    vec_gram_fold_kernel<<<1, 256, 0, p->stream>>>(part, nblk, cnt, nb, dst);
    SPCP_CHECK_LAUNCH("vec_gram_fold");
    p->launches += 2;
    if (out_host) {
      SPCP_CUDA(cudaMemcpyAsync(p->host_out, p->out_dev.ptr, size_t(cnt) * nb * sizeof(double),
                                cudaMemcpyDeviceToHost, p->stream));
      SPCP_CUDA(cudaStreamSynchronize(p->stream));
      std::memcpy(out_host + size_t(a0) * nb, p->host_out, size_t(cnt) * nb * sizeof(double));
    }
  }
  return SPCP_OK;
}

int spcp_vec_gram(spcp_problem* p, int64_t len, int na, const double* const* a, int nb,
                  const double* const* b, double* out_host) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  return vec_gram_impl(p, len, na, a, nb, b, out_host, nullptr);
}

int spcp_vec_gram_dev(spcp_problem* p, int64_t len, int na, const double* const* a, int nb,
                      const double* const* b, double* out_dev) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  if (!out_dev) return fail(SPCP_ERR_VALUE, "vec_gram_dev: null output");
  return vec_gram_impl(p, len, na, a, nb, b, nullptr, out_dev);
}

int spcp_gram(spcp_problem* p, int64_t rows, int64_t pa, const double* a, int64_t qb,
              const double* b, double* out_host) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  const int64_t rpb = std::max<int64_t>(256, round_up(ceil_div(rows, 296), 32));
  const int64_t nrb = std::max<int64_t>(1, ceil_div(rows, rpb));
  const int64_t pq = pa * qb;
  if ((rc = p->vec_part.ensure(size_t(nrb * pq + pq) * sizeof(double)))) return rc;
  double* part = p->vec_part.as<double>();
  double* res = part + nrb * pq;
  dim3 grid(unsigned(nrb), unsigned(ceil_div(pa, 32)), unsigned(ceil_div(qb, 32)));
  gram_kernel<<<grid, 256, 0, p->stream>>>(a, pa, b, qb, rows, rpb, part);
  SPCP_CHECK_LAUNCH("gram");
  gram_fold_kernel<<<grid_for(pq), 256, 0, p->stream>>>(part, int(nrb), pq, res);
  SPCP_CHECK_LAUNCH("gram_fold");
  p->launches += 2;
  SPCP_CUDA(cudaMemcpyAsync(out_host, res, size_t(pq) * sizeof(double), cudaMemcpyDeviceToHost,
                            p->stream));
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  return SPCP_OK;
}

int spcp_matmul_small(spcp_problem* p, int64_t rows, int64_t pa, const double* a, int64_t qb,
                      const double* m_host, double* c) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  int rc;
  SPCP_CUDA(cudaSetDevice(p->device));
  if ((rc = p->small.ensure(std::max(p->small.bytes, size_t(pa * qb) * sizeof(double))))) return rc;
  DevBuf mm;
  if ((rc = mm.ensure(size_t(pa * qb) * sizeof(double)))) return rc;
  SPCP_CUDA(cudaMemcpyAsync(mm.ptr, m_host, size_t(pa * qb) * sizeof(double),
                            cudaMemcpyHostToDevice, p->stream));
  matmul_small_kernel<<<grid_for(rows * qb), 256, 0, p->stream>>>(a, rows, pa, mm.as<double>(), qb,
                                                                   c);
  SPCP_CHECK_LAUNCH("matmul_small");
  p->launches++;
  SPCP_CUDA(cudaStreamSynchronize(p->stream));
  mm.release();
  return SPCP_OK;
}

int spcp_prof_enable(spcp_problem* p, int on) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  if (p->ev_count) cudaStreamSynchronize(p->stream);
  p->prof = on != 0;
  p->prof_ms = 0.0;
  p->prof_count = 0;
  p->ev_count = 0;
  return SPCP_OK;
}

int spcp_prof_read(spcp_problem* p, double* ms_total, int64_t* launches, int64_t* kernels) {
  if (!p) return fail(SPCP_ERR_VALUE, "null problem handle");
  if (p->ev_count && prof_collect(p)) return SPCP_ERR_CUDA;
  *ms_total = p->prof_ms;
  *launches = p->prof_count;
  *kernels = p->launches;
  p->prof_ms = 0.0;
  p->prof_count = 0;
  p->launches = 0;
  return SPCP_OK;
}

}  // extern "C"
#include "slrm_io.cuh"
