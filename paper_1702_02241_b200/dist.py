"""Column-sharded multi-GPU Split-SPCP.

Rank p owns columns J_p = [col0, col0 + n_p) of X (and of the mask), the
matching rows V_p of V, and a replica of U.  Per evaluation:

  local fused kernel -> phi_p, G_p V_p (m x k), grad_V shard, V-part dots
  ONE all-reduce of G_p V_p (fp32 in fp32 mode) + one of 4 fp64 scalars
  -> grad_U = sum_p G_p V_p + lambda U on every rank (identical bits).

L-BFGS vectors keep the [U | V_p] layout: U-part inner products are computed
redundantly (identical on all ranks), V-part ones are summed across ranks in
the same all-reduce call per iteration (`vec_gram`), so the replicated U and
the history stay bit-identical on every rank.  NCCL over NVLink/NVSwitch is
the transport on GPUs (torch.distributed, backend "nccl"); the host logic is
exercised with backend "gloo" on CPU by the tests (tests/test_dist_gloo.py).
"""

import math

import numpy as np

from .lbfgs import DeviceLbfgs
from .report import IterateState, SolveReport, WorkTimer

__all__ = ["ShardedSpace", "solve_split_spcp_sharded", "allreduce_host", "shard_bounds"]


def shard_bounds(n_total, world, rank):
    """Contiguous near-equal column partition."""
    base, extra = divmod(int(n_total), int(world))
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist

    return dist


def allreduce_host(arr, device, group=None):
    """Sum a small host array across ranks (on `device` so NCCL can carry it)."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(device)
    _dist().all_reduce(t, group=group)
    return t.cpu().numpy()


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

    def empty(self):
        return self.dp.empty(self.length)

    def eval(self, z, d, alpha, g_out, precision):
        from ._lib import SPCP_F32, SPCP_F64

        dist = _dist()
        code = SPCP_F32 if precision == "fp32" else SPCP_F64
        gu = self.gu32 if (precision == "fp32" and self.k <= 64) else self.gu64
        self.dp.eval_partial(self.k, code, z, d, alpha, gu, self.scal, g_out)
        dist.all_reduce(gu, group=self.group)
        dist.all_reduce(self.scal, group=self.group)
        self.comm_bytes += gu.numel() * gu.element_size() + 32
        out = self.dp.eval_finish(self.k, code, z, d, alpha, gu, self.scal, g_out)
        return out[0], out[3], out[4]

    def gram(self, a_list, b_list):
        ua = [a[: self.mk] for a in a_list]
        ub = [b[: self.mk] for b in b_list]
        va = [a[self.mk:] for a in a_list]
        vb = [b[self.mk:] for b in b_list]
        u_part = self.dp.vec_gram(ua, ub)
        v_part = self.dp.vec_gram(va, vb) if self.n > 0 else np.zeros_like(u_part)
        return u_part + allreduce_host(v_part, self.comm_device, self.group)

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
    dist.all_reduce(y, group=group)
    q, _ = device_thin_qr(dp, y)
    for _ in range(int(power_iters)):
        _, zl = dp.apply(0, None, w_left=q)
        q2, _ = device_thin_qr(dp, zl, gram_reduce=red)
        y, _ = dp.apply(0, None, w_right=q2)
        dist.all_reduce(y, group=group)
        q, _ = device_thin_qr(dp, y)
    _, bt = dp.apply(0, None, w_left=q)  # (n_p x width) rows of B^T
    world = dist.get_world_size(group)
    nmax = max(shard_bounds(n_total, world, r)[1] for r in range(world))
    pad = torch.zeros((nmax, width), dtype=torch.float64, device=bt.device)
    pad[:n] = bt
    parts = [torch.empty_like(pad) for _ in range(world)]
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
    if not isinstance(x_local, torch.Tensor):
        xa = np.asarray(x_local)
        if precision != "fp32" and not np.array_equal(xa.astype(np.float32).astype(xa.dtype),
                                                      xa):
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
    return SolveReport(solver="split", termination=res.termination, iterations=res.records,
                       l=None, s=None, objective=res.objective, factors=factors,
                       extra={"k_final": k, "columns_grown": 0, "n_evals": res.n_evals,
                              "precision": precision, "allreduce_bytes": space.comm_bytes,
                              "col0": col0, "n_local": n, "problem": dp})
