/*
 * spcp_b200.h — C ABI of the B200-native Split-SPCP hot path.
 *
 * The reference (arXiv:1702.02241, /root/reference/pkg/src/spcp) is a pure
 * Python/numpy package, so its "FFI" for this path is the set of Python
 * entry points listed below; each C entry point replaces the numpy/BLAS work
 * behind one of them.  The Python host layer (paper_1702_02241_b200/) binds
 * these symbols with ctypes and keeps the reference's Python signatures,
 * argument meaning and exceptions.
 *
 *   spcp_problem_create      <- ProblemSpec(x, lambda_l, lambda_s, mask)
 *                               objective.py:20-59 (+ validation.py:10-34)
 *   spcp_eval / _partial /
 *   spcp_eval_finish         <- split_objective(fp, spec)      solver.py:105-123
 *                               via _flat_split_objective      solver.py:219-225
 *                               called per line-search trial   lbfgs.py:55-61
 *   spcp_split_objective_host<- split_objective with host (numpy) buffers
 *   spcp_phi_dense_host      <- phi_value_grad(l, spec)        objective.py:90-117
 *   spcp_apply               <- the m x n products of certificate.py:93-103,
 *                               rand_svd linalg.py:97-105 and the growth
 *                               power iteration solver.py:237-241
 *   spcp_materialize         <- FactorPair.compose + phi_value_grad S*
 *                               solver.py:313-320 (final L, S)
 *   spcp_vec_*               <- the L-BFGS vector algebra  lbfgs.py:152-188
 *   spcp_gram / spcp_matmul_small  <- thin_qr/factor_svd factor-space algebra
 *                               linalg.py:43-59, certificate.py:50-67
 *   spcp_slrm_header /
 *   spcp_slrm_read_device    <- read_matrix (binary)        matrixio.py:94-126
 *   spcp_slrm_write_device /
 *   spcp_slrm_write_product  <- write_matrix (binary)       matrixio.py:53-71
 *                               of the decompose outputs    cli.py:256-270
 *
 * Conventions:
 *   - every function returns an int status; 0 = SPCP_OK.  The Python layer
 *     maps SPCP_ERR_VALUE -> ValueError, SPCP_ERR_DIMENSION -> DimensionError,
 *     SPCP_ERR_NUMERICAL / SPCP_ERR_CUDA -> NumericalError (DeviceError);
 *     spcp_last_error() holds the message (thread-local).
 *   - matrices are row-major; the flat iterate is concat(U.ravel(), V.ravel())
 *     in float64 exactly as FactorPair.flatten (solver.py:65-66).
 *   - "dev" pointers are CUDA device pointers on the problem's device; work is
 *     stream-ordered on the problem's stream; nothing allocates inside eval
 *     once the workspace for a rank bound k has been created.
 *   - inputs are never mutated; outputs are caller-owned buffers.
 */
#ifndef SPCP_B200_H
#define SPCP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPCP_ABI_VERSION 1

enum spcp_status {
  SPCP_OK = 0,
  SPCP_ERR_VALUE = 1,       /* ValueError        (validation.py:19-20, objective.py:40-43) */
  SPCP_ERR_DIMENSION = 2,   /* DimensionError    (errors.py:8-9) */
  SPCP_ERR_NUMERICAL = 3,   /* NumericalError    (errors.py:12-13) */
  SPCP_ERR_CUDA = 4,        /* NumericalError subclass DeviceError: CUDA failure */
  SPCP_ERR_UNSUPPORTED = 5, /* ValueError: option not built into this library */
  /* matrix files (matrixio.py:94-125, errors.py:29-44) */
  SPCP_ERR_IO = 6,               /* MatrixIOError, code "io_error" (OS error) */
  SPCP_ERR_MALFORMED_HEADER = 7, /* MalformedHeaderError "malformed_header" */
  SPCP_ERR_TRUNCATED = 8,        /* TruncatedPayloadError "truncated_payload" */
  SPCP_ERR_NONFINITE = 9,        /* NonFiniteDataError "non_finite_data" */
  SPCP_ERR_NOT_FOUND = 10,       /* FileNotFoundError (open / mkstemp ENOENT) */
};

enum spcp_dtype { SPCP_F32 = 0, SPCP_F64 = 1, SPCP_U8 = 2 /* mask bytes, SLRM reads only */ };

/* storage flags for spcp_problem_create */
#define SPCP_STORE_F32 1u
#define SPCP_STORE_F64 2u
#define SPCP_STORE_SPARSE 4u /* masked X: force the sparse-observation (CSR + CSC) path */
#define SPCP_STORE_DENSE 8u  /* masked X: force the dense streaming pass */

typedef struct spcp_problem spcp_problem;

int spcp_abi_version(void);
const char* spcp_last_error(void);
int spcp_device_count(int* out);

/* ---- ProblemSpec upload (objective.py:20-59) ------------------------------
 * x: m x n row-major with leading dimension ldx (elements), float64 or
 *    float32 (x_dtype), on the host (x_on_device = 0) or the device.
 * mask: optional m x n bool bytes on the host (non-zero = observed), or NULL.
 * store: SPCP_STORE_F32 | SPCP_STORE_F64 — which device copies of X to keep
 *    (fp32 copy feeds the fp32 kernels, fp64 copy the fp64 kernels; an fp32
 *    copy is also read exactly by the fp64 kernels when X is fp32-exact).
 * n_total / col0: column-sharded mode; this problem holds
 *    columns [col0, col0+n) of an m x n_total matrix.  Single GPU: n_total = n,
 *    col0 = 0.
 * stream: cudaStream_t to order all work on (NULL = legacy default stream).
 */
int spcp_problem_create(spcp_problem** out, int device, int64_t m, int64_t n,
                        const void* x, int64_t ldx, int x_dtype, int x_on_device,
                        const uint8_t* mask, unsigned store, double lambda_l,
                        double lambda_s, int64_t n_total, int64_t col0, void* stream);
int spcp_problem_destroy(spcp_problem* p);
int spcp_problem_set_stream(spcp_problem* p, void* stream);
/* info (8 doubles): [0] = 0.5*||P_Omega X||_F^2 (local shard), [1] = #observed
 * entries, [2] = stored dtypes mask, [3] = device bytes held, [4] = observed
 * entries stored for the sparse-observation evaluation (CSR + CSC, built at
 * creation for masks at most 12% observed and used by fp64 evaluations, and by
 * fp32 ones below 2.5%; SPCP_STORE_SPARSE / SPCP_SDDMM=on use it for both),
 * -1 if only the dense streaming passes are used. */
int spcp_problem_info(spcp_problem* p, double* info);

/* ---- objective + gradient (solver.py:105-123) ------------------------------
 * Evaluates F and grad F at the trial point w = z + alpha*dz (dz may be NULL),
 * z, dz, g_out: device float64 vectors of length (m + n)*k, flat [U | V].
 * dtype: SPCP_F32 runs the fused fp32 streaming kernel (fp64 accumulation of
 * the objective, fp64 regulariser and trial point); SPCP_F64 runs it in fp64.
 * out (host, 8 doubles): [0] f, [1] phi, [2] lambda/2(|U|^2+|V|^2),
 *   [3] g . dz (0 when dz == NULL), [4] |g|^2, [5] |g_U|^2, [6] g_U . dz_U,
 *   [7] reserved.  The call synchronises the problem's stream. */
int spcp_eval(spcp_problem* p, int64_t k, int dtype, const double* z, const double* dz,
              double alpha, double* g_out, double* out);

/* Stream-ordered spcp_eval: the same evaluation, but the 8 scalars stay on the
 * device (copied into out_dev, device float64[8], when it is not NULL) and the
 * call does not synchronise — for callers that keep the control flow on the
 * device or batch several evaluations (the throughput bench).  Same reference
 * function (split_objective solver.py:105-123). */
int spcp_eval_async(spcp_problem* p, int64_t k, int dtype, const double* z, const double* dz,
                    double alpha, double* g_out, double* out_dev);

/* Sharded evaluation split around the grad_U all-reduce:
 * _partial writes the shard's G_p V_p (m x k, `dtype` elements) into gu_part
 * (device), 4 shard scalars [phi_p, lambda/2|V_p|^2, g_V.dz_V, |g_V|^2] into
 * scal (device float64) and the shard-local grad_V into g_out's V block.
 * The caller all-reduces gu_part and scal across ranks, then _finish adds
 * lambda*U, writes g_out's U block and fills out[8] as spcp_eval (synchronous). */
int spcp_eval_partial(spcp_problem* p, int64_t k, int dtype, const double* z,
                      const double* dz, double alpha, void* gu_part, double* scal,
                      double* g_out);
int spcp_eval_finish(spcp_problem* p, int64_t k, int dtype, const double* z,
                     const double* dz, double alpha, const void* gu_sum,
                     const double* scal_sum, double* g_out, double* out);

/* Host-buffer drop-in for split_objective (the e2e path): u (m x k), v (n x k)
 * float64 host arrays in, value and grad_u / grad_v float64 host arrays out. */
int spcp_split_objective_host(spcp_problem* p, int64_t k, int dtype, const double* u,
                              const double* v, double* value, double* grad_u,
                              double* grad_v);

/* Host-buffer drop-in for phi_value_grad(l, spec) (objective.py:90-117):
 * l is m x n float64; grad / s_star outputs may be NULL. */
int spcp_phi_dense_host(spcp_problem* p, const double* l, double* value, double* grad,
                        double* s_star);

/* ---- streaming operator products (certificate / rSVD / growth) -------------
 * With G = grad phi(U V^T) (k >= 1, z = flat [U|V] float64 device) or, when
 * k == 0, G = P_Omega(X) (the zero-filled observed matrix, ProblemSpec.observed
 * objective.py:49-53), computes
 *   left_out  (m x b) = G  @ w_right   (w_right: n x b)   if w_right != NULL
 *   right_out (n x b) = G^T @ w_left   (w_left:  m x b)   if w_left  != NULL
 * in float64 (all pointers device float64, row-major).  In sharded mode the
 * left product is the shard's partial sum (caller all-reduces). */
int spcp_apply(spcp_problem* p, int64_t k, const double* z, int64_t b,
               const double* w_right, double* left_out, const double* w_left,
               double* right_out);

/* spcp_apply with fp32 streaming products (fp32 X copy, fp32 operands, fp64
 * outputs): for the certificate's subspace iteration, which only compares
 * sigma(P) against 1.  Falls back to spcp_apply when no fp32 copy of X is
 * stored or k exceeds the fused widths. */
int spcp_apply_f32(spcp_problem* p, int64_t k, const double* z, int64_t b,
                   const double* w_right, double* left_out, const double* w_left,
                   double* right_out);

/* ---- stored gradient (the certificate's repeated products, certificate.py:119)
 * spcp_grad_store materialises G = grad phi(U V^T) on Omega (zeros elsewhere)
 * once, float32 (dtype SPCP_F32) or float64, in device memory (m x n elements;
 * SPCP_ERR_UNSUPPORTED when it does not fit — keep calling spcp_apply);
 * spcp_apply_stored then gives G W_right / G^T W_left like spcp_apply from one
 * pass over the stored G, without recomputing the rank-k residual;
 * spcp_grad_release ends its use.  The stored G and the stored ray below share
 * one workspace that stays with the problem between uses (allocating and
 * freeing tens of GB costs 25-500 ms per call); spcp_workspace_trim frees it,
 * spcp_problem_destroy too. */
int spcp_grad_store(spcp_problem* p, int64_t k, const double* z, int dtype);
int spcp_apply_stored(spcp_problem* p, int64_t b, const double* w_right, double* left_out,
                      const double* w_left, double* right_out);
int spcp_grad_release(spcp_problem* p);
int spcp_workspace_trim(spcp_problem* p);

/* ---- final L and S (solver.py:313-320) --------------------------------------
 * Rows [row0, row0+rows) of L = U V^T and S* = shrink(X - L) on Omega, float64,
 * written to device or host buffers (row-major, n columns); either may be NULL. */
int spcp_materialize(spcp_problem* p, int64_t k, const double* z, int64_t row0,
                     int64_t rows, double* l_out, double* s_out, int out_on_host);

/* Dense grad phi(U V^T) (m x n float64, device, row stride ldo) — the
 * materialised D = -G/lambda of certificate.py:93-95, used only for small
 * problems where the complement SVD is done densely like the reference. */
int spcp_materialize_grad(spcp_problem* p, int64_t k, const double* z, double* g_out,
                          int64_t ldo);

/* ---- line-restricted evaluation (the probes of one line search, lbfgs.py:64-99)
 * On the ray z + a dz the residual is quadratic in a: R(a) = R0 - a D1 - a^2 D2
 * on Omega with R0 = X - U V^T, D1 = dU V^T + U dV^T, D2 = dU dV^T.
 * spcp_line_setup stores the three m x n float64 matrices (24 bytes per entry
 * of device memory; SPCP_ERR_UNSUPPORTED when they do not fit or X is held
 * only as sparse observations — the caller then keeps probing with
 * spcp_eval).  spcp_line_probe(a) returns out_host[8] = [F, phi, reg,
 * grad F . dz, 0, 0, 0, 0] at z + a dz (float64, fixed-order sums) from one
 * pass over the stored matrices, without the gradient; spcp_line_release
 * ends their use (the memory stays for the next search: spcp_workspace_trim).
 * Replaces the per-probe fun(x) calls of the reference's strong-Wolfe search
 * (spcp/lbfgs.py:64-99) for the probes that are not accepted; the accepted
 * point is re-evaluated with spcp_eval. */
int spcp_line_setup(spcp_problem* p, int64_t k, const double* z, const double* dz);
int spcp_line_probe(spcp_problem* p, double alpha, double* out_host);
int spcp_line_release(spcp_problem* p);

/* ---- L-BFGS vector algebra (lbfgs.py:152-188, compact form) -----------------
 * All device float64, length len.  Deterministic (fixed-order) reductions.
 * multidot: out_host[i] = <a[i], b[i]> for i < count (a, b: host arrays of
 *   device pointers).  lincomb: out = sum_i coef[i] * v[i] (out may alias v[0]).
 */
int spcp_vec_multidot(spcp_problem* p, int64_t len, int count, const double* const* a,
                      const double* const* b, double* out_host);
int spcp_vec_lincomb(spcp_problem* p, int64_t len, int count, const double* coef,
                     const double* const* v, double* out);
/* vec_gram: out_host[i*nb + j] = <a[i], b[j]>, i < na, j < nb (nb <= 4); every
 * vector is read once (one pass for all dots of an L-BFGS iteration). */
int spcp_vec_gram(spcp_problem* p, int64_t len, int na, const double* const* a, int nb,
                  const double* const* b, double* out_host);
/* vec_gram_dev: the same dots into a device buffer (na * nb float64), stream
 * ordered, no synchronisation: the column-sharded path all-reduces them on the
 * device before one copy to the host (dist.py). */
int spcp_vec_gram_dev(spcp_problem* p, int64_t len, int na, const double* const* a, int nb,
                      const double* const* b, double* out_dev);

/* ---- tall-skinny factor algebra (linalg.py:43-59, certificate.py:50-67) ----
 * gram: out_host (p x q, float64) = A^T B, A: rows x p, B: rows x q (device).
 * matmul_small: C (rows x q) = A (rows x p) @ M (p x q, host float64). */
int spcp_gram(spcp_problem* p, int64_t rows, int64_t pa, const double* a, int64_t qb,
              const double* b, double* out_host);
int spcp_matmul_small(spcp_problem* p, int64_t rows, int64_t pa, const double* a,
                      int64_t qb, const double* m_host, double* c);

/* ---- profiling: CUDA-event time of the fused streaming kernel --------------
 * When enabled, every eval records events around its main kernel; read
 * returns the accumulated milliseconds and launch count, then resets. */
int spcp_prof_enable(spcp_problem* p, int on);
int spcp_prof_read(spcp_problem* p, double* ms_total, int64_t* launches,
                   int64_t* kernels_launched);

/* ---- SLRM matrix files straight to / from HBM (matrixio.py:25-113) --------
 * Format: "SLRM", version u32 = 1, rows u64, cols u64 (little endian), then
 * the row-major float64 payload.  The reader validates the header and the
 * payload length before touching data (matrixio.py:94-109) and rejects NaN /
 * Inf after the read (matrixio.py:124-125); writes go to a temp file in the
 * target directory and are renamed into place (matrixio.py:40-50).
 *
 * header: rows / cols of an SLRM file (read_matrix's shape, matrixio.py:98).
 * read_device: the window [row0, row0+rows) x [col0, col0+cols) (rows / cols
 *   < 0 = to the end) into a device matrix dst (row stride ld elements) as
 *   SPCP_F32, SPCP_F64 or SPCP_U8 (1 where the entry is non-zero: the CLI's
 *   mask semantics, cli.py:165-167).  Row chunks are double-buffered through
 *   pinned memory; a column window is how a rank reads its shard (§8(e)).
 * write_device: a device matrix (SPCP_F32 widened, or SPCP_F64) to a file.
 * write_product: L = U V^T and S* = shrink(X - L) on Omega (solver.py:313-320,
 *   the decompose command's --output-l / --output-s, cli.py:256-259) streamed
 *   from the problem to files (either path may be NULL); nnz_s (may be NULL)
 *   receives the trace's "nnz_s" (cli.py:268). */
int spcp_slrm_header(const char* path, int64_t* rows, int64_t* cols);
int spcp_slrm_read_device(const char* path, int device, int64_t row0, int64_t rows,
                          int64_t col0, int64_t cols, void* dst, int dst_dtype, int64_t ld,
                          void* stream);
int spcp_slrm_write_device(const char* path, int device, const void* src, int src_dtype,
                           int64_t rows, int64_t cols, int64_t ld, void* stream);
int spcp_slrm_write_product(spcp_problem* p, int64_t k, const double* z, const char* l_path,
                            const char* s_path, int64_t* nnz_s);

#ifdef __cplusplus
}
#endif
#endif /* SPCP_B200_H */
