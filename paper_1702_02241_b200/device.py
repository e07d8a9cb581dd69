"""Device-resident problem (the GPU side of ProblemSpec, objective.py:20-59).

`DeviceProblem` owns one `spcp_problem` handle of libspcp_b200.so: the padded
fp32/fp64 copies of X in HBM, the bit-packed observation mask and the
workspaces of the fused streaming kernel.  Device vectors are torch CUDA
tensors (torch is plumbing here: allocation, streams, torch.distributed); all
arithmetic on m x n data runs in this repo's sm_100a kernels.
"""

import ctypes

import numpy as np

from ._lib import (SPCP_ERR_UNSUPPORTED, SPCP_F32, SPCP_F64, STORE_DENSE, STORE_F32, STORE_F64,
                   STORE_SPARSE, check, lib)

__all__ = ["DeviceProblem", "torch_mod", "cuda_device", "dptr", "PRECISIONS", "nvtx_range"]

PRECISIONS = ("fp32", "fp64", "mixed")

_torch = None


def torch_mod():
    global _torch
    if _torch is None:
        import torch

        _torch = torch
    return _torch


class nvtx_range:
    """NVTX range around a solver phase (rSVD init, L-BFGS, certificate), so
    an nsys / ncu timeline of a solve shows where the time goes."""

    def __init__(self, name):
        self.name = name
        self.on = False

    def __enter__(self):
        torch = torch_mod()
        if torch.cuda.is_available():
            torch.cuda.nvtx.range_push(self.name)
            self.on = True
        return self

    def __exit__(self, *exc):
        if self.on:
            torch_mod().cuda.nvtx.range_pop()
        return False


def cuda_device():
    torch = torch_mod()
    if not torch.cuda.is_available():
        from .errors import DeviceError

        raise DeviceError("no CUDA device: the Split-SPCP compute path runs only on the GPU "
                          "(sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def dptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _ptr_array(ts):
    arr = (ctypes.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return arr


class DeviceProblem:
    """One column shard (or the whole matrix) of X resident on a GPU.

    x: host numpy array (float64 or float32) or a CUDA tensor, m x n.
    store: iterable of "f32" / "f64": which device copies to keep; "sparse" /
      "dense" force the masked evaluation path (default: the sparse copy is
      built at <= 12% observed and used by fp64 evaluations, and by fp32 ones
      below 2.5%, sddmm.cuh).
    n_total, col0: column-sharded mode.
    """

    def __init__(self, x, lambda_l, lambda_s, mask=None, store=("f32",), n_total=None,
                 col0=0):
        torch = torch_mod()
        self.device = cuda_device()
        self.stream = torch.cuda.current_stream(self.device)
        on_dev = isinstance(x, torch.Tensor)
        if on_dev:
            xt = x if x.is_contiguous() else x.contiguous()
            m, n = xt.shape
            dt = SPCP_F64 if xt.dtype == torch.float64 else SPCP_F32
            if xt.dtype not in (torch.float32, torch.float64):
                raise ValueError("device X must be float32 or float64")
            xptr, ldx = ctypes.c_void_p(xt.data_ptr()), n
        else:
            xa = np.asarray(x)
            if xa.dtype not in (np.float32, np.float64):
                xa = xa.astype(np.float64)
            xa = np.ascontiguousarray(xa)
            m, n = xa.shape
            dt = SPCP_F64 if xa.dtype == np.float64 else SPCP_F32
            xptr, ldx = ctypes.c_void_p(xa.ctypes.data), n
            self._keep = xa
        mptr = None
        if mask is not None:
            mk = np.ascontiguousarray(mask, dtype=np.bool_)
            mptr = ctypes.c_void_p(mk.ctypes.data)
            self._keep_mask = mk
        flags = 0
        codes = {"f32": STORE_F32, "f64": STORE_F64, "sparse": STORE_SPARSE, "dense": STORE_DENSE}
        for s in store:
            flags |= codes[s]
        self.m, self.n = int(m), int(n)
        self.n_total = int(n_total if n_total is not None else n)
        self.col0 = int(col0)
        self.lambda_l, self.lambda_s = float(lambda_l), float(lambda_s)
        self.masked = mask is not None
        self.store = frozenset(store)
        h = ctypes.c_void_p()
        check(lib.spcp_problem_create(ctypes.byref(h), self.device.index, self.m, self.n, xptr,
                                      ldx, dt, int(on_dev), mptr, flags, self.lambda_l,
                                      self.lambda_s, self.n_total, self.col0,
                                      ctypes.c_void_p(self.stream.cuda_stream)))
        self.handle = h
        self._keep = None
        self._keep_mask = None
        info = (ctypes.c_double * 8)()
        check(lib.spcp_problem_info(self.h, info))
        self.f_zero = float(info[0])
        self.n_obs = float(info[1])
        # observed entries held for the sparse-observation path (sddmm.cuh), or None
        self.sparse_nnz = int(info[4]) if info[4] >= 0 else None
        self._out = (ctypes.c_double * 8)()

    # ------------------------------------------------------------ lifecycle
    @property
    def h(self):
        if not self.handle:
            from .errors import DeviceError

            raise DeviceError("device problem already released")
        return self.handle

    def close(self):
        if getattr(self, "handle", None):
            lib.spcp_problem_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ helpers
    def empty(self, n, dtype=None):
        torch = torch_mod()
        return torch.empty(int(n), dtype=dtype or torch.float64, device=self.device)

    def zeros(self, n, dtype=None):
        torch = torch_mod()
        return torch.zeros(int(n), dtype=dtype or torch.float64, device=self.device)

    @staticmethod
    def dtype_code(precision):
        return SPCP_F32 if precision == "fp32" else SPCP_F64

    # ------------------------------------------------------------ evaluation
    def eval(self, k, dtype, z, dz, alpha, g_out):
        """F and grad F at z + alpha*dz -> np.array([f, phi, reg, g.dz, |g|^2, |gU|^2,
        gU.dzU, 0]); g_out (device float64) receives the gradient."""
        check(lib.spcp_eval(self.h, int(k), int(dtype), dptr(z), dptr(dz), float(alpha),
                            dptr(g_out), self._out))
        return np.frombuffer(self._out, dtype=np.float64).copy()

    def eval_async(self, k, dtype, z, dz, alpha, g_out, out_dev=None):
        """Stream-ordered eval: the scalars stay on the device (out_dev, float64[8])
        and nothing synchronises."""
        check(lib.spcp_eval_async(self.h, int(k), int(dtype), dptr(z), dptr(dz), float(alpha),
                                  dptr(g_out), dptr(out_dev)))

    def eval_partial(self, k, dtype, z, dz, alpha, gu_part, scal, g_out):
        check(lib.spcp_eval_partial(self.h, int(k), int(dtype), dptr(z), dptr(dz),
                                    float(alpha), dptr(gu_part), dptr(scal), dptr(g_out)))

    def eval_finish(self, k, dtype, z, dz, alpha, gu_sum, scal_sum, g_out):
        check(lib.spcp_eval_finish(self.h, int(k), int(dtype), dptr(z), dptr(dz),
                                   float(alpha), dptr(gu_sum), dptr(scal_sum), dptr(g_out),
                                   self._out))
        return np.frombuffer(self._out, dtype=np.float64).copy()

    def split_objective_host(self, u, v, dtype, out=None):
        """(f, grad_U, grad_V) for host float64 factors.  `out=(gu, gv)` reuses
        caller buffers (e.g. pinned memory) instead of allocating fresh arrays."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        k = u.shape[1]
        if out is not None:
            gu, gv = out
            if (gu.shape != u.shape or gv.shape != v.shape or gu.dtype != np.float64
                    or gv.dtype != np.float64 or not gu.flags.c_contiguous
                    or not gv.flags.c_contiguous):
                raise ValueError("out buffers must be C-contiguous float64 of the factor shapes")
        else:
            gu = np.empty_like(u)
            gv = np.empty_like(v)
        val = ctypes.c_double()
        check(lib.spcp_split_objective_host(self.h, k, int(dtype),
                                            ctypes.c_void_p(u.ctypes.data),
                                            ctypes.c_void_p(v.ctypes.data), ctypes.byref(val),
                                            ctypes.c_void_p(gu.ctypes.data),
                                            ctypes.c_void_p(gv.ctypes.data)))
        return float(val.value), gu, gv

    def phi_dense_host(self, l, want_grad=True, want_s=True):
        l = np.ascontiguousarray(l, dtype=np.float64)
        g = np.empty_like(l) if want_grad else None
        s = np.empty_like(l) if want_s else None
        val = ctypes.c_double()
        check(lib.spcp_phi_dense_host(self.h, ctypes.c_void_p(l.ctypes.data),
                                      ctypes.byref(val),
                                      None if g is None else ctypes.c_void_p(g.ctypes.data),
                                      None if s is None else ctypes.c_void_p(s.ctypes.data)))
        return float(val.value), g, s

    # ------------------------------------------------------------ operators
    def apply(self, k, z, w_right=None, w_left=None, precision="fp64"):
        """(G @ w_right, G^T @ w_left) as float64 device matrices; G = grad phi at
        U V^T (k >= 1) or the zero-filled observed X (k == 0).  precision="fp32"
        streams the fp32 copy of X with fp32 operands (spcp_apply_f32)."""
        torch = torch_mod()
        b = int((w_right if w_right is not None else w_left).shape[1])
        left = right = None
        if w_right is not None:
            w_right = w_right.contiguous()
            left = torch.empty((self.m, b), dtype=torch.float64, device=self.device)
        if w_left is not None:
            w_left = w_left.contiguous()
            right = torch.empty((self.n, b), dtype=torch.float64, device=self.device)
        fn = lib.spcp_apply_f32 if precision == "fp32" else lib.spcp_apply
        check(fn(self.h, int(k), dptr(z), b, dptr(w_right), dptr(left), dptr(w_left),
                 dptr(right)))
        return left, right

    # ------------------------------------------------------------ stored gradient
    def grad_store(self, k, z, precision="fp32"):
        """Materialise G = grad phi(U V^T) once (float32 or float64) for
        apply_stored; False when it does not fit (or X is sparse-only)."""
        rc = lib.spcp_grad_store(self.h, int(k), dptr(z), SPCP_F32 if precision == "fp32"
                                 else SPCP_F64)
        if rc == SPCP_ERR_UNSUPPORTED:
            return False
        check(rc)
        return True

    def apply_stored(self, w_right=None, w_left=None):
        """(G @ w_right, G^T @ w_left) from the stored G (float64 device matrices)."""
        torch = torch_mod()
        b = int((w_right if w_right is not None else w_left).shape[1])
        left = right = None
        if w_right is not None:
            w_right = w_right.contiguous()
            left = torch.empty((self.m, b), dtype=torch.float64, device=self.device)
        if w_left is not None:
            w_left = w_left.contiguous()
            right = torch.empty((self.n, b), dtype=torch.float64, device=self.device)
        check(lib.spcp_apply_stored(self.h, b, dptr(w_right), dptr(left), dptr(w_left),
                                    dptr(right)))
        return left, right

    def grad_release(self):
        check(lib.spcp_grad_release(self.h))

    def trim_workspace(self):
        """Free the large workspace shared by the stored ray and the stored
        gradient (kept between uses; also freed by close())."""
        check(lib.spcp_workspace_trim(self.h))

    # ------------------------------------------------------------ line probes
    def line_setup(self, k, z, dz):
        """Store R0, D1, D2 of the ray z + a dz (csrc/line.cuh).  False when the
        three m x n float64 matrices do not fit (or X is sparse-only): the
        caller keeps probing with eval()."""
        rc = lib.spcp_line_setup(self.h, int(k), dptr(z), dptr(dz))
        if rc == SPCP_ERR_UNSUPPORTED:
            return False
        check(rc)
        return True

    def line_probe(self, alpha):
        """[F, phi, reg, grad F . dz, 0, 0, 0, 0] at z + alpha dz of the stored ray."""
        check(lib.spcp_line_probe(self.h, float(alpha), self._out))
        return np.frombuffer(self._out, dtype=np.float64).copy()

    def line_release(self):
        check(lib.spcp_line_release(self.h))

    def materialize(self, k, z, row0=0, rows=None, want_l=True, want_s=True):
        rows = self.m - row0 if rows is None else rows
        l = np.empty((rows, self.n)) if want_l else None
        s = np.empty((rows, self.n)) if want_s else None
        check(lib.spcp_materialize(self.h, int(k), dptr(z), int(row0), int(rows),
                                   None if l is None else ctypes.c_void_p(l.ctypes.data),
                                   None if s is None else ctypes.c_void_p(s.ctypes.data), 1))
        return l, s

    def grad_dense(self, k, z):
        """Dense grad phi(U V^T) as an (m x n) float64 device matrix."""
        torch = torch_mod()
        g = torch.empty((self.m, self.n), dtype=torch.float64, device=self.device)
        check(lib.spcp_materialize_grad(self.h, int(k), dptr(z), dptr(g), self.n))
        return g

    # ------------------------------------------------------------ vector algebra
    def multidot(self, a_list, b_list):
        cnt = len(a_list)
        out = (ctypes.c_double * cnt)()
        length = a_list[0].numel()
        check(lib.spcp_vec_multidot(self.h, length, cnt, _ptr_array(a_list),
                                    _ptr_array(b_list), out))
        return np.frombuffer(out, dtype=np.float64).copy()

    def vec_gram(self, a_list, b_list):
        """Host (len(a) x len(b)) matrix of dots, each device vector read once."""
        na, nb = len(a_list), len(b_list)
        out = (ctypes.c_double * (na * nb))()
        check(lib.spcp_vec_gram(self.h, a_list[0].numel(), na, _ptr_array(a_list), nb,
                                _ptr_array(b_list), out))
        return np.frombuffer(out, dtype=np.float64).reshape(na, nb).copy()

    def vec_gram_dev(self, a_list, b_list, out=None):
        """The same dots into a device float64 tensor (na x nb), no host sync."""
        torch = torch_mod()
        na, nb = len(a_list), len(b_list)
        if out is None:
            out = torch.empty((na, nb), dtype=torch.float64, device=self.device)
        check(lib.spcp_vec_gram_dev(self.h, a_list[0].numel(), na, _ptr_array(a_list), nb,
                                    _ptr_array(b_list), dptr(out)))
        return out

    def lincomb(self, coefs, vecs, out):
        cnt = len(vecs)
        c = (ctypes.c_double * cnt)(*[float(x) for x in coefs])
        check(lib.spcp_vec_lincomb(self.h, out.numel(), cnt, c, _ptr_array(vecs),
                                   dptr(out)))
        return out

    def gram(self, a, b):
        """a^T b for tall float64 device matrices (rows x p), (rows x q) -> host p x q."""
        a = a.contiguous()
        b = b.contiguous()
        rows, pa = a.shape
        qb = b.shape[1]
        out = np.empty((pa, qb))
        check(lib.spcp_gram(self.h, rows, pa, dptr(a), qb, dptr(b),
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def matmul_small(self, a, mat):
        """a (rows x p, device) @ mat (p x q, host) -> device rows x q."""
        torch = torch_mod()
        a = a.contiguous()
        rows, pa = a.shape
        mat = np.ascontiguousarray(mat, dtype=np.float64)
        qb = mat.shape[1]
        c = torch.empty((rows, qb), dtype=torch.float64, device=self.device)
        check(lib.spcp_matmul_small(self.h, rows, pa, dptr(a), qb,
                                    mat.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), dptr(c)))
        return c

    # ------------------------------------------------------------ profiling
    def prof_enable(self, on=True):
        check(lib.spcp_prof_enable(self.h, int(bool(on))))

    def prof_read(self):
        ms = ctypes.c_double()
        cnt = ctypes.c_int64()
        kl = ctypes.c_int64()
        check(lib.spcp_prof_read(self.h, ctypes.byref(ms), ctypes.byref(cnt),
                                 ctypes.byref(kl)))
        return float(ms.value), int(cnt.value), int(kl.value)
