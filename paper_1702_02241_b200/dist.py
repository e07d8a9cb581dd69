"""Column-sharded multi-GPU Split-SPCP.

Rank p owns columns J_p = [col0, col0 + n_p) of X (and of the mask), the
matching rows V_p of V, and a replica of U.  Per evaluation:

  local fused kernel -> phi_p, G_p V_p (m x k), grad_V shard, V-part dots
  one all-reduce step: G_p V_p (fp32 in fp32 mode) and the 4 fp64 scalars
  travel in ONE fused NCCL launch (a coalesced group of the two buffers; the
  dtypes differ, so they cannot share one buffer without losing the scalars'
  fp64 sums) -> grad_U = sum_p G_p V_p + lambda U on every rank (identical bits).

L-BFGS vectors keep the [U | V_p] layout: U-part inner products are computed
redundantly (identical on all ranks), V-part ones are summed across ranks on
the device (`vec_gram_dev` + all-reduce, one copy to the host per iteration),
so the replicated U and the history stay bit-identical on every rank.  NCCL
over NVLink/NVSwitch is the transport on GPUs (torch.distributed, backend
"nccl"; `pin_nccl()` fixes the algorithm and protocol so repeated runs sum in
the same order); the host logic is exercised with backend "gloo" on CPU by the
tests (tests/test_dist_gloo.py).

The certificate over column shards (`certificate_sharded`, certificate.py:77-141)
is the single-GPU code with CertOps reductions: the m x b products D_p W_p of
the subspace iteration and D_p V1_p are all-reduced, Grams of row-sharded
n-side blocks (V, V1, D^T U1, the subspace block) are summed as host k x k /
b x b matrices.
"""

import os

import math

import numpy as np

from .lbfgs import DeviceLbfgs
from .report import IterateState, SolveReport, WorkTimer

__all__ = ["ShardedSpace", "solve_split_spcp_sharded", "certificate_sharded", "allreduce_host",
           "shard_bounds", "pin_nccl", "allreduce_fused"]


def pin_nccl():
    """Fix NCCL's algorithm and protocol (before the communicator is created)
    so the all-reduce order, hence the bits, repeat run to run."""
    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "Simple")


def shard_bounds(n_total, world, rank):
    """Contiguous near-equal column partition."""
    base, extra = divmod(int(n_total), int(world))
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist

    return dist


class _Collective:
    """Maps a failing collective (NCCL / gloo raise RuntimeError or
    DistBackendError) to the package's DeviceError, a NumericalError subclass
    like every CUDA failure of the C ABI (SURVEY §8(b) error conventions)."""

    def __init__(self, what):
        self.what = what

    def __enter__(self):
        return self

    def __exit__(self, et, ev, tb):
        if et is not None and issubclass(et, RuntimeError):
            from .errors import DeviceError

            raise DeviceError(f"collective {self.what} failed: {ev}") from ev
        return False


def allreduce_host(arr, device, group=None):
    """Sum a small host array across ranks (on `device` so NCCL can carry it)."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(device)
    with _Collective("all_reduce(host array)"):
        _dist().all_reduce(t, group=group)
    return t.cpu().numpy()


def allreduce_fused(tensors, group=None):
    """Sum several device buffers across ranks in one collective launch: an
    NCCL group (torch's coalescing manager) when the backend is NCCL, plain
    calls otherwise (gloo on CPU tests)."""
    dist = _dist()
    with _Collective("all_reduce(evaluation)"):
        if dist.get_backend(group) == "nccl" and hasattr(dist, "_coalescing_manager"):
            with dist._coalescing_manager(group=group, device=tensors[0].device,
                                          async_ops=True) as cm:
                for t in tensors:
                    dist.all_reduce(t, group=group)
            cm.wait()
            return
        for t in tensors:
            dist.all_reduce(t, group=group)


class ShardedSpace:
    """DeviceLbfgs vector space over [U (replicated) | V_p (shard)] vectors.

    `dp` is a DeviceProblem for the shard (or any object with the same
    eval_partial / eval_finish / vec_gram / lincomb / empty methods)."""

    def __init__(self, dp, k, m, n_local, group=None, comm_device=None, gu_dtype=None):
        import torch

        self.dp = dp
        self.k = int(k)
        self.m, self.n = int(m), int(n_local)
        self.mk = self.m * self.k
        self.length = (self.m + self.n) * self.k
        self.group = group
        self.comm_device = comm_device if comm_device is not None else dp.device
        self.gu32 = torch.empty(self.mk, dtype=torch.float32, device=dp.device)
        self.gu64 = torch.empty(self.mk, dtype=torch.float64, device=dp.device)
        self.scal = torch.empty(4, dtype=torch.float64, device=dp.device)
        self.comm_bytes = 0
        self.comm_calls = 0

    def empty(self):
        return self.dp.empty(self.length)

    def eval(self, z, d, alpha, g_out, precision):
        from ._lib import SPCP_F32, SPCP_F64

        dist = _dist()
        code = SPCP_F32 if precision == "fp32" else SPCP_F64
        gu = self.gu32 if (precision == "fp32" and self.k <= 64) else self.gu64
        self.dp.eval_partial(self.k, code, z, d, alpha, gu, self.scal, g_out)
        allreduce_fused([gu, self.scal], self.group)
        self.comm_bytes += gu.numel() * gu.element_size() + 32
        self.comm_calls += 1
        out = self.dp.eval_finish(self.k, code, z, d, alpha, gu, self.scal, g_out)
        return out[0], out[3], out[4]

    # stored-ray probes (DeviceLbfgs fp64 searches): every rank stores its
    # shard's R0, D1, D2; the replicated U part of the regulariser is counted once
    def line_setup(self, z, d):
        setup = getattr(self.dp, "line_setup", None)
        ok = bool(setup(self.k, z, d)) if setup is not None else False
        if setup is None:  # host-side test doubles: no rank has it
            return False
        # all ranks or none (device memory may differ between ranks)
        flag = allreduce_host(np.array([0.0 if ok else 1.0]), self.comm_device, self.group)
        if flag[0] > 0.0:
            if ok:
                self.dp.line_release()
            return False
        g = self.dp.vec_gram([z[: self.mk], d[: self.mk]], [z[: self.mk], d[: self.mk]])
        self._ureg = (float(g[0, 0]), float(g[0, 1]), float(g[1, 1]))
        return True

    def line_probe(self, alpha):
        out = self.dp.line_probe(alpha)
        uu, ud, dd = self._ureg
        lam = self.dp.lambda_l
        reg_u = 0.5 * lam * (uu + alpha * (2.0 * ud + alpha * dd))
        dreg_u = lam * (ud + alpha * dd)
        tot = allreduce_host(np.array([out[0] - reg_u, out[3] - dreg_u]), self.comm_device,
                             self.group)
        self.comm_calls += 1
        return float(tot[0]) + reg_u, float(tot[1]) + dreg_u

    def line_release(self):
        self.dp.line_release()

    def gram(self, a_list, b_list):
        ua = [a[: self.mk] for a in a_list]
        ub = [b[: self.mk] for b in b_list]
        va = [a[self.mk:] for a in a_list]
        vb = [b[self.mk:] for b in b_list]
        dev = getattr(self.dp, "vec_gram_dev", None)
        if dev is None:  # host-side test doubles
            u_part = self.dp.vec_gram(ua, ub)
            v_part = self.dp.vec_gram(va, vb) if self.n > 0 else np.zeros_like(u_part)
            return u_part + allreduce_host(v_part, self.comm_device, self.group)
        import torch

        u_part = dev(ua, ub)
        v_part = dev(va, vb) if self.n > 0 else torch.zeros_like(u_part)
        with _Collective("all_reduce(dots)"):
            _dist().all_reduce(v_part, group=self.group)
        return (u_part + v_part).cpu().numpy()

    def lincomb(self, coefs, vecs, out):
        return self.dp.lincomb(coefs, vecs, out)

    def to_host(self, z):
        return z.cpu().numpy()


def _sharded_rsvd(dp, k, n_total, col0, oversample, power_iters, seed, group, comm_device):
    """rand_svd (linalg.py:77-106) of the column-sharded observed matrix."""
    import torch

    from .linalg import device_thin_qr, svd_small

    dist = _dist()
    m, n = dp.m, dp.n
    width = k + min(int(oversample), min(m, n_total) - k)
    omega = np.random.default_rng(seed).standard_normal((n_total, width))
    om = torch.from_numpy(np.ascontiguousarray(omega[col0:col0 + n])).to(dp.device)

    def red(g):
        return allreduce_host(g, comm_device, group)

    y, _ = dp.apply(0, None, w_right=om)
    with _Collective("all_reduce(rsvd sketch)"):
        dist.all_reduce(y, group=group)
    q, _ = device_thin_qr(dp, y)
    for _ in range(int(power_iters)):
        _, zl = dp.apply(0, None, w_left=q)
        q2, _ = device_thin_qr(dp, zl, gram_reduce=red)
        y, _ = dp.apply(0, None, w_right=q2)
        with _Collective("all_reduce(rsvd sketch)"):
            dist.all_reduce(y, group=group)
        q, _ = device_thin_qr(dp, y)
    _, bt = dp.apply(0, None, w_left=q)  # (n_p x width) rows of B^T
    world = dist.get_world_size(group)
    nmax = max(shard_bounds(n_total, world, r)[1] for r in range(world))
    pad = torch.zeros((nmax, width), dtype=torch.float64, device=bt.device)
    pad[:n] = bt
    parts = [torch.empty_like(pad) for _ in range(world)]
    with _Collective("all_gather(rsvd core)"):
        dist.all_gather(parts, pad, group=group)
    full = torch.cat([parts[r][: shard_bounds(n_total, world, r)[1]] for r in range(world)])
    inner = svd_small(full.cpu().numpy().T)
    u = dp.matmul_small(q, inner.u[:, :k])
    v_loc = inner.v[col0:col0 + n, :k]
    return u, inner.sigma[:k].copy(), v_loc


def solve_split_spcp_sharded(x_local, lambda_l, lambda_s, k, n_total, col0, cfg=None,
                             mask_local=None, group=None, init="rsvd", iter_hook=None):
    """solve_split_spcp (solver.py:255-324) over a column shard on this rank.

    x_local: m x n_p host array or CUDA tensor of columns [col0, col0+n_p).
    Returns a SolveReport whose `factors` hold (U, V_p) and whose extra
    records the all-reduce volume.  (Rank growth is single-GPU only.)"""
    import torch

    from .device import DeviceProblem
    from .solver import SolverConfig, _effective_precision

    cfg = cfg or SolverConfig()
    m = int(x_local.shape[0])
    n = int(x_local.shape[1])
    precision = _effective_precision(cfg.precision, (m, n_total))
    store = ("f32",) if precision in ("fp32", "mixed") else ("f64",)
    if isinstance(x_local, torch.Tensor):
        exact = x_local.dtype == torch.float32 or bool(
            (x_local.float().double() == x_local).all())
    else:
        xa = np.asarray(x_local)
        exact = bool(np.array_equal(xa.astype(np.float32).astype(xa.dtype), xa))
    if precision != "fp32" and not exact:
        # the fp64 phase must stream the unrounded X (ProblemSpec.device does
        # the same check): keep an fp64 copy next to the fp32 one
        store = ("f32", "f64") if precision == "mixed" else ("f64",)
    dp = DeviceProblem(x_local, lambda_l, lambda_s, mask_local, store=store, n_total=n_total,
                       col0=col0)
    comm_device = dp.device
    timer = WorkTimer()
    if init != "rsvd":
        raise ValueError("sharded solve supports init='rsvd'")
    u, sig, v_loc = _sharded_rsvd(dp, k, n_total, col0, 10, 1, cfg.seed, group, comm_device)
    root = np.sqrt(sig)
    z = torch.cat([(u * torch.from_numpy(root).to(dp.device)).reshape(-1),
                   torch.from_numpy(np.ascontiguousarray(v_loc * root)).to(dp.device).reshape(-1)
                   ]).contiguous()
    space = ShardedSpace(dp, k, m, n, group=group, comm_device=comm_device)

    def hook(it, zz):
        extra = {"rank": k}
        if iter_hook is not None:
            extra.update(iter_hook(it, IterateState(factors=None)) or {})
        return extra

    eng = DeviceLbfgs(space, memory=cfg.memory, grad_tol=cfg.grad_tol, max_iter=cfg.max_iter,
                      c1=cfg.wolfe_c1, c2=cfg.wolfe_c2, precision=precision,
                      switch_tol=cfg.switch_tol, iter_hook=hook, timer=timer)
    res = eng.run(z)
    zh = z.cpu().numpy()
    from .solver import FactorPair

    factors = FactorPair(zh[: m * k].reshape(m, k), zh[m * k:].reshape(n, k))
    rep = SolveReport(solver="split", termination=res.termination, iterations=res.records,
                      l=None, s=None, objective=res.objective, factors=factors,
                      extra={"k_final": k, "columns_grown": 0, "n_evals": res.n_evals,
                             "precision": precision, "allreduce_bytes": space.comm_bytes,
                             "allreduce_calls": space.comm_calls, "col0": col0, "n_local": n,
                             "n_total": n_total, "problem": dp})
    rep.device_state = (dp, k, z)
    return rep


def certificate_sharded(report, lambda_l=None, f_bound_hint=None, rank_tol=1e-10, group=None):
    """certificate (certificate.py:77-141) of a column-sharded solve: every
    rank passes its own SolveReport from solve_split_spcp_sharded; all ranks
    return the same CertificateReport."""
    from .certificate import CertOps, certificate_core

    dp, k, z = report.device_state
    ex = report.extra
    lam = float(lambda_l if lambda_l is not None else dp.lambda_l)
    dist = _dist()

    def red_host(a):
        return allreduce_host(a, dp.device, group)

    def red_dev(t):
        with _Collective("all_reduce(certificate product)"):
            dist.all_reduce(t, group=group)

    ops = CertOps(host=red_host, dev=red_dev, n_total=ex["n_total"], col0=ex["col0"])
    f_zero = float(red_host(np.array([dp.f_zero]))[0])
    hint = report.best_objective if f_bound_hint is None else f_bound_hint
    return certificate_core(dp, z, dp.m, ex["n_total"], k, lam, rank_tol, f_zero, hint, ops)
