"""Factorised (SVD-free) Split-SPCP solver (spcp solver.py:1-324), on the GPU.

Minimises  lambda_l/2 (|U|^2 + |V|^2) + phi(U V^T)  with the device-resident
L-BFGS of lbfgs.py.  Every objective/gradient evaluation is one launch of the
fused streaming kernel over X in HBM (plus operand prep and a fixed-order
reduction); the host sees only the scalars the line search needs.

Public API kept from the reference: FactorPair, SolverConfig, split_objective,
init_factors, factors_from_dense, lbfgs_minimize, solve_split_spcp.  New,
defaulted config fields: `precision` ("mixed" | "fp32" | "fp64") and
`switch_tol`; they do not change the reference's semantics (mixed finishes in
fp64 with the reference's stopping rule; problems below MIXED_MIN_ELEMS run
in fp64 throughout).
"""

import math
from dataclasses import dataclass

import numpy as np

from .errors import DimensionError
from .lbfgs import DeviceLbfgs, minimize_lbfgs
from .linalg import rand_svd_device, svd_small
from .objective import ProblemSpec, get_default_precision
from .report import IterateState, SolveReport, WorkTimer
from .validation import as_matrix, check_rank_bound

__all__ = ["FactorPair", "SolverConfig", "split_objective", "init_factors",
           "factors_from_dense", "lbfgs_minimize", "solve_split_spcp", "MIXED_MIN_ELEMS",
           "SplitSpace"]

INIT_STRATEGIES = ("rsvd", "full_svd", "random")
# below this many entries the fp32 bulk phase buys nothing: run fp64 throughout
MIXED_MIN_ELEMS = 1 << 22


@dataclass(frozen=True)
class FactorPair:
    """The split iterate (U, V), L = U V^T (solver.py:36-71)."""

    u: np.ndarray
    v: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "u", as_matrix(self.u, "u"))
        object.__setattr__(self, "v", as_matrix(self.v, "v"))
        if self.u.shape[1] != self.v.shape[1]:
            raise DimensionError(
                f"u and v must share the rank dimension, got {self.u.shape} and {self.v.shape}")
        if self.k < 1:
            raise DimensionError("rank bound k must be >= 1")

    @property
    def k(self):
        return self.u.shape[1]

    @property
    def shape(self):
        return (self.u.shape[0], self.v.shape[0])

    def compose(self):
        return self.u @ self.v.T

    def flatten(self):
        return np.concatenate([self.u.ravel(), self.v.ravel()])

    @classmethod
    def from_flat(cls, z, m, n, k):
        z = np.asarray(z, dtype=np.float64)
        return cls(z[: m * k].reshape(m, k).copy(), z[m * k:].reshape(n, k).copy())


@dataclass(frozen=True)
class SolverConfig:
    """Solver knobs (solver.py:74-102) + device precision policy."""

    memory: int = 10
    grad_tol: float = 1e-8
    max_iter: int = 500
    wolfe_c1: float = 1e-4
    wolfe_c2: float = 0.9
    rank_growth: bool = False
    max_k: int | None = None
    growth_tol: float = 1e-6
    seed: int = 0
    precision: str = "mixed"
    switch_tol: float = 1e-5

    def __post_init__(self):
        if not 0.0 < self.wolfe_c1 < self.wolfe_c2 < 1.0:
            raise ValueError(
                f"need 0 < wolfe_c1 < wolfe_c2 < 1, got {self.wolfe_c1}, {self.wolfe_c2}")
        if self.memory < 1:
            raise ValueError(f"memory must be >= 1, got {self.memory}")
        if self.precision not in ("mixed", "fp32", "fp64"):
            raise ValueError(f"precision must be mixed/fp32/fp64, got {self.precision!r}")


def _dtype(precision):
    from ._lib import SPCP_F32, SPCP_F64

    return SPCP_F32 if precision == "fp32" else SPCP_F64


def split_objective(fp, spec, precision=None):
    """(value, grad_u, grad_v) of the split objective (solver.py:105-123),
    evaluated by the fused GPU kernel; host float64 arrays in and out."""
    if fp.shape != spec.shape:
        raise DimensionError(f"factor shapes {fp.shape} do not match data shape {spec.shape}")
    precision = precision or get_default_precision()
    dp = spec.device(precision)
    return dp.split_objective_host(fp.u, fp.v, _dtype(precision))


def _effective_precision(precision, shape):
    if precision == "mixed" and shape[0] * shape[1] < MIXED_MIN_ELEMS:
        return "fp64"
    return precision


def init_factors(spec, k, strategy="rsvd", seed=0, oversample=10, power_iters=1):
    """Starting factors (solver.py:126-154): balanced rank-k (randomized) SVD
    of the zero-filled observations, or i.i.d. N(0, 1/k) entries."""
    m, n = spec.shape
    k = check_rank_bound(k, spec.shape)
    if strategy == "random":
        gen = np.random.default_rng(seed)
        sc = 1.0 / np.sqrt(k)
        return FactorPair(sc * gen.standard_normal((m, k)), sc * gen.standard_normal((n, k)))
    if strategy == "full_svd":
        tri = svd_small(np.asarray(spec.observed())).truncate(k)
        root = np.sqrt(tri.sigma)
        return FactorPair(tri.u * root, tri.v * root)
    if strategy != "rsvd":
        raise ValueError(f"unknown init strategy {strategy!r}; expected one of {INIT_STRATEGIES}")
    dp = spec.device("fp64" if spec.fp32_exact() else "mixed")
    eff = min(int(oversample), min(m, n) - k)
    u, sig, v = rand_svd_device(dp, k, oversample=eff, power_iters=power_iters, seed=seed)
    root = np.sqrt(sig)
    return FactorPair(u.cpu().numpy() * root, v * root)


def factors_from_dense(l, rank_tol=0.0):
    """Balanced factors of a dense matrix (solver.py:157-172)."""
    l = as_matrix(l, "l")
    tri = svd_small(l)
    sig = tri.sigma
    if sig.size == 0 or sig[0] <= 0.0:
        return FactorPair(np.zeros((l.shape[0], 1)), np.zeros((l.shape[1], 1)))
    r = max(int(np.sum(sig > rank_tol * sig[0])), 1)
    root = np.sqrt(sig[:r])
    return FactorPair(tri.u[:, :r] * root, tri.v[:, :r] * root)


def lbfgs_minimize(fun, start, cfg, iter_hook=None, timer=None):
    """Plug-in L-BFGS over a host callable (solver.py:175-216)."""
    m, n = start.shape
    k = start.k
    timer = timer or WorkTimer()
    hook = None
    if iter_hook is not None:
        def hook(it, z):
            return iter_hook(it, IterateState(factors=FactorPair.from_flat(z, m, n, k)))
    res = minimize_lbfgs(fun, start.flatten(), memory=cfg.memory, grad_tol=cfg.grad_tol,
                         max_iter=cfg.max_iter, c1=cfg.wolfe_c1, c2=cfg.wolfe_c2,
                         iter_hook=hook, timer=timer)
    fp = FactorPair.from_flat(res.x, m, n, k)
    return SolveReport(solver="split", termination=res.termination, iterations=res.records,
                       l=fp.compose(), s=None, objective=res.objective, factors=fp,
                       extra={"n_evals": res.n_evals})


class SplitSpace:
    """Vector space of flat [U | V] iterates of one device problem for
    DeviceLbfgs (single GPU; dist.ShardedSpace is the column-sharded one)."""

    def __init__(self, dp, k):
        self.dp = dp
        self.k = int(k)
        self.length = (dp.m + dp.n) * self.k

    def empty(self):
        return self.dp.empty(self.length)

    def eval(self, z, d, alpha, g_out, precision):
        out = self.dp.eval(self.k, _dtype(precision), z, d, alpha, g_out)
        return out[0], out[3], out[4]

    def line_setup(self, z, d):
        """Store the ray z + a d for line_probe (DeviceLbfgs, fp64 searches)."""
        return self.dp.line_setup(self.k, z, d)

    def line_probe(self, alpha):
        out = self.dp.line_probe(alpha)
        return out[0], out[3]

    def line_release(self):
        self.dp.line_release()

    def gram(self, a_list, b_list):
        return self.dp.vec_gram(a_list, b_list)

    def lincomb(self, coefs, vecs, out):
        return self.dp.lincomb(coefs, vecs, out)

    def to_host(self, z):
        return z.cpu().numpy()


def _growth_column_device(space, z, seed):
    """Rank-1 escape direction (solver.py:228-252): leading singular triple of
    -grad phi by power iteration whose products are streaming-kernel passes
    (b = 1), then append sqrt(1e-3 s1)(u1, v1)."""
    import torch

    dp, k = space.dp, space.k
    m, n = dp.m, dp.n
    tol, max_iter = 1e-6, 1000
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    vd = torch.from_numpy(v).to(dp.device).reshape(n, 1)

    def mv(x):  # -(G x)
        left, _ = space.apply_left(z, x)
        return -left

    def rmv(y):  # -(G^T y)
        _, right = space.apply_right(z, y)
        return -right

    sigma = 0.0
    u = None
    conv = False
    for _ in range(max_iter):
        u = mv(vd)
        su = space.norm_left(u)
        if su == 0.0:
            return None
        u = u / su
        w = rmv(u)
        sv = space.norm_right(w)
        if sv == 0.0:
            sigma = su
            conv = True
            break
        vd = w / sv
        if abs(sv - sigma) <= tol * max(1.0, sv):
            u = mv(vd)
            sigma = space.norm_left(u)
            if sigma > 0.0:
                u = u / sigma
            conv = True
            break
        sigma = sv
    del conv  # a partially converged triple is accepted (solver.py:242-245)
    if not sigma > 0.0:
        return None
    root = math.sqrt(1e-3 * sigma)
    return u.reshape(-1) * root, vd.reshape(-1) * root


def _grow(space, z, u_col, v_col):
    """Flat [U | V] with one extra column appended to each factor."""
    import torch

    dp, k = space.dp, space.k
    m, n = dp.m, dp.n
    uu = z[: m * k].reshape(m, k)
    vv = z[m * k:].reshape(n, k)
    return torch.cat([torch.cat([uu, u_col.reshape(m, 1)], 1).reshape(-1),
                      torch.cat([vv, v_col.reshape(n, 1)], 1).reshape(-1)]).contiguous()


def _space_ops(space):
    """Attach the operator helpers the growth step uses to a single-GPU space."""
    import torch

    dp = space.dp

    def apply_left(z, x):
        return dp.apply(space.k, z, w_right=x)

    def apply_right(z, y):
        return dp.apply(space.k, z, w_left=y)

    def norm(t):
        return float(torch.linalg.vector_norm(t).item())

    space.apply_left = apply_left
    space.apply_right = apply_right
    space.norm_left = norm
    space.norm_right = norm
    return space


def solve_split_spcp(spec, k, cfg=None, init="rsvd", iter_hook=None, timer=None, space_factory=None):
    """Initialise, minimise, optionally grow the rank (solver.py:255-324).

    Returns a SolveReport with the reference's fields; `l` and `s` are dense
    float64 arrays materialised from the device factors on first access.
    """
    import torch

    cfg = cfg or SolverConfig()
    m, n = spec.shape
    k = check_rank_bound(k, spec.shape)
    timer = timer or WorkTimer()
    precision = _effective_precision(cfg.precision, spec.shape)
    make_space = space_factory or (lambda dpk, kk: _space_ops(SplitSpace(dpk, kk)))
    dp = spec.device(precision)
    from .device import nvtx_range

    with nvtx_range("spcp.init_factors"):
        fp = init_factors(spec, k, strategy=init, seed=cfg.seed)
    z = torch.from_numpy(fp.flatten()).to(dp.device)
    cap = cfg.max_k if cfg.max_k is not None else min(m, n)
    records, n_evals, offset, grown = [], 0, 0, 0
    best = None
    switches = []
    while True:
        kk = z.numel() // (m + n)
        space = make_space(dp, kk)

        def hook(it, zz, kk=kk, offset=offset, space=space):
            extra = {"rank": kk}
            if iter_hook is not None:
                st = IterateState(factors=FactorPair.from_flat(space.to_host(zz), m, n, kk))
                extra.update(iter_hook(offset + it, st) or {})
            return extra

        eng = DeviceLbfgs(space, memory=cfg.memory, grad_tol=cfg.grad_tol,
                          max_iter=cfg.max_iter, c1=cfg.wolfe_c1, c2=cfg.wolfe_c2,
                          precision=precision, switch_tol=cfg.switch_tol, iter_hook=hook,
                          timer=timer)
        with nvtx_range(f"spcp.lbfgs k={kk}"):
            res = eng.run(z)
        n_evals += res.n_evals
        if eng.switched_at is not None:
            switches.append(offset + eng.switched_at)
        for rec in res.records:
            rec.iteration += offset
        records.extend(res.records)
        offset = records[-1].iteration + 1 if records else 0
        prev = best["objective"] if best is not None else None
        if best is None or res.objective < best["objective"]:
            best = {"objective": res.objective, "termination": res.termination,
                    "z": z.clone(), "k": kk}
        stationary = res.termination in ("converged", "line_search_failed")
        if not (cfg.rank_growth and stationary and kk < cap):
            break
        if prev is not None and (prev - res.objective) / max(1.0, abs(prev)) < cfg.growth_tol:
            break
        col = _growth_column_device(space, z, seed=cfg.seed + grown + 1)
        if col is None:
            break
        z = _grow(space, z, *col)
        grown += 1
    kf = best["k"]
    zf = best["z"]
    zh = zf.cpu().numpy()
    factors = FactorPair.from_flat(zh, m, n, kf)
    cache = {}

    def dense(which):
        def get():
            if "ls" not in cache:
                cache["ls"] = dp.materialize(kf, zf)
            return cache["ls"][0 if which == "l" else 1]
        return get

    extra = {"k_final": kf, "columns_grown": grown, "n_evals": n_evals,
             "precision": precision}
    if switches:
        extra["fp64_switch_iter"] = switches
    report = SolveReport(solver="split", termination=best["termination"], iterations=records,
                         l=dense("l"), s=dense("s"), objective=best["objective"],
                         factors=factors, extra=extra)
    # the device iterate stays reachable so L and S can be streamed to files
    # without host m x n arrays (matrixio.write_decomposition)
    report.device_state = (dp, kf, zf)
    return report
