"""Computable optimality certificate (spcp certificate.py:1-141), on the GPU.

At L = U V^T with D = -grad phi(L) / lambda_l and the compact SVD
L = U1 S V1^T (from the factors: two tall QRs + a k x k SVD), the squared
distance from 0 to the subdifferential of lambda|L|_* + phi(L) is

    lambda^2 ( |I - U1^T D V1|^2 + |U1^T D P_V|^2 + |P_U D V1|^2
               + sum_i max(sigma_i(P) - 1, 0)^2 ),   P = P_U D P_V

(certificate.py:100-128).  Device mapping:
  * a^T = D^T U1 and b = D V1 come from ONE fused streaming pass over X
    (`spcp_apply` with both product operands), c = a V1 is a Gram;
  * t4 needs the singular values of P above 1.  The reference takes a dense
    SVD of the m x n P (certificate.py:70-74,119).  Here P is never formed: a
    block subspace iteration applies P and P^T through streaming passes (D W
    and D^T Y computed from X on the fly, then projected) and the Ritz values
    give sigma_i(P); the block grows until its smallest Ritz value is below 1
    so every sigma > 1 is captured.  Ritz values are lower bounds: t4 comes
    from converged values, or is proved to be exactly 0 by a probabilistic
    bound on sigma_max(P) (`_power_bound_iters`), and `info` says which.
  * Column-sharded problems run the same code with `CertOps`
    reductions: Grams of row-sharded n-side blocks and the m x b products
    D W are summed across ranks (dist.certificate_sharded).
"""

import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from .errors import NumericalError
from .linalg import SvdTriplet, device_thin_qr, svd_small, thin_qr

__all__ = ["CertificateReport", "factor_svd", "certificate", "CertOps", "certificate_core",
           "FP32_PRODUCTS_MIN_ELEMS"]

# above this many entries the subspace iteration's D products stream the fp32
# copy of X (they are compared against 1 only); below it they run in fp64
FP32_PRODUCTS_MIN_ELEMS = 1 << 22


@dataclass(frozen=True)
class CertificateReport:
    """certificate.py:22-47 (+ `info`: how t4 was obtained)."""

    e_norm: float
    terms: tuple
    f_bound: float
    gap_bound: float
    r: int
    l_norm: float
    info: dict = field(default_factory=dict, compare=False)

    def to_dict(self):
        return {"e_norm": self.e_norm, "terms": list(self.terms), "f_bound": self.f_bound,
                "gap_bound": self.gap_bound, "rank": self.r}


def factor_svd(fp, rank_tol=1e-10):
    """Compact SVD of U V^T from the factors (certificate.py:50-67); host
    float64 like the reference (k-space algebra on host arrays)."""
    qu, ru = thin_qr(fp.u)
    qv, rv = thin_qr(fp.v)
    core = svd_small(ru @ rv.T)
    sig = core.sigma
    r = 0 if (sig.size == 0 or sig[0] <= 0.0) else int(np.sum(sig > rank_tol * sig[0]))
    return SvdTriplet((qu @ core.u)[:, :r], sig[:r].copy(), (qv @ core.v)[:, :r])


class CertOps:
    """Cross-rank sums for a column-sharded problem (identities on one GPU).

    host(a): sum a small host array (Grams of row-sharded n-side blocks).
    dev(t):  sum a device tensor in place (the m x b products D_p W_p)."""

    def __init__(self, host=None, dev=None, n_total=None, col0=0):
        self._host = host
        self._dev = dev
        self.n_total = n_total
        self.col0 = int(col0)
        self.sharded = host is not None

    def host(self, a):
        return a if self._host is None else self._host(a)

    def dev(self, t):
        if self._dev is not None:
            self._dev(t)
        return t

    def gram_rows(self, dp, a, b):
        """a^T b for n-side (row-sharded) device matrices."""
        return self.host(dp.gram(a, b))


def _device_factor_svd(dp, u, v, rank_tol, ops):
    """factor_svd (certificate.py:50-67) on device factors u (m x k,
    replicated) and v (n_p x k, this rank's rows); returns (u1, sigma, v1,
    all singular values) with u1, v1 device matrices."""
    qu, ru = device_thin_qr(dp, u)
    qv, rv = device_thin_qr(dp, v, ops.host if ops.sharded else None)
    core = svd_small(ru @ rv.T)
    sig = core.sigma
    r = 0 if (sig.size == 0 or sig[0] <= 0.0) else int(np.sum(sig > rank_tol * sig[0]))
    if r == 0:
        return None, sig[:0], None, sig, None
    u1 = dp.matmul_small(qu, core.u[:, :r])
    v1 = dp.matmul_small(qv, core.v[:, :r])
    # U1 = U ru^-1 core.u, V1 = V rv^-1 core.v (full column rank): the maps from
    # the factors to the bases, for _gradient_products
    maps = None
    if r == u.shape[1] and ru.shape == rv.shape == (r, r):
        cu, cv = np.linalg.cond(ru), np.linalg.cond(rv)
        if max(cu, cv) <= GRADIENT_ROUTE_MAX_COND:
            maps = (np.linalg.solve(ru, core.u[:, :r]), np.linalg.solve(rv, core.v[:, :r]))
    return u1, sig[:r].copy(), v1, sig, maps


# t1-t3 need G V1 and G^T U1.  With full-rank factors V1 = V rv^-1 core.v, so
# G V1 = (G V) rv^-1 core.v, and G V = grad_U F - lambda U comes out of ONE fp64
# evaluation (the FP64 tensor-core pass for fp32-exact X) instead of a separate
# streaming product; used when the maps are this well conditioned (the products
# keep ~cond * 1e-16 relative accuracy)
GRADIENT_ROUTE_MAX_COND = 1e4


def _gradient_products(dp, z, k, lam, ops):
    """(G V, G^T U_p) at z (device, m x k and n_p x k) from one fp64
    evaluation, or None when dp has no fp64 evaluation for this k."""
    import torch

    from ._lib import SPCP_F64

    m, n = dp.m, dp.n
    mk = m * k
    if ops.sharded:
        if not hasattr(dp, "eval_partial"):
            return None
        g = torch.empty((m + n) * k, dtype=torch.float64, device=z.device)
        gu = torch.empty(mk, dtype=torch.float64, device=z.device)
        scal = torch.empty(4, dtype=torch.float64, device=z.device)
        dp.eval_partial(k, SPCP_F64, z, None, 0.0, gu, scal, g)
        ops.dev(gu)  # G V summed over the column shards
        gv = gu
    else:
        if not hasattr(dp, "eval"):
            return None
        g = torch.empty((m + n) * k, dtype=torch.float64, device=z.device)
        dp.eval(k, SPCP_F64, z, None, 0.0, g)
        gv = g[:mk] - lam * z[:mk]
    gtu = g[mk:] - lam * z[mk:]
    return gv.reshape(m, k), gtu.reshape(n, k)


class _ProjectedOperator:
    """x -> P x and y -> P^T y with P = (I - U1U1^T) D (I - V1V1^T), D = -G/lam,
    every D product a streaming pass over X (spcp_apply)."""

    def __init__(self, dp, z, k, lam, u1, v1, ops, precision):
        self.dp, self.z, self.k, self.lam, self.u1, self.v1 = dp, z, k, lam, u1, v1
        self.ops = ops
        self.precision = precision
        # every pass applies the same G: materialise it once (G from X and the
        # factors in fp64, stored in the product precision) and stream the
        # stored copy, instead of recomputing the rank-k residual per pass
        store = getattr(dp, "grad_store", None)
        self.stored = bool(store(k, z, precision)) if store is not None and STORE_GRADIENT \
            else False
        self.stored_used = self.stored

    def close(self):
        if self.stored:
            self.dp.grad_release()
            self.stored = False

    def _apply(self, w_right=None, w_left=None):
        if self.stored:
            return self.dp.apply_stored(w_right=w_right, w_left=w_left)
        return self.dp.apply(self.k, self.z, w_right=w_right, w_left=w_left,
                             precision=self.precision)

    def proj_u(self, w):  # replicated m-side
        if self.u1 is None:
            return w
        c = self.dp.gram(self.u1, w)
        return w - self.dp.matmul_small(self.u1, c)

    def proj_v(self, w):  # row-sharded n-side
        if self.v1 is None:
            return w
        c = self.ops.gram_rows(self.dp, self.v1, w)
        return w - self.dp.matmul_small(self.v1, c)

    def right(self, w):  # P w, w: n_p x b
        w = self.proj_v(w)
        y, _ = self._apply(w_right=w.contiguous())
        self.ops.dev(y)  # sum_p D_p W_p
        return self.proj_u(y.mul_(-1.0 / self.lam))

    def left(self, y):  # P^T y, y: m x b (replicated)
        y = self.proj_u(y)
        _, w = self._apply(w_left=y.contiguous())
        return self.proj_v(w.mul_(-1.0 / self.lam))


# the subspace iteration streams a stored copy of G when it fits (False: every
# pass recomputes G from X and the factors)
STORE_GRADIENT = True

# Ritz-value convergence tolerance by product precision: fp64 streaming
# products resolve sigma(P) to ~1e-15, the fp32 ones to ~1e-7
_SUBSPACE_TOL = {"fp64": 1e-9, "fp32": 1e-6}
_FAIL_PROB = 1e-6
# (1 - eps, certified factor): after the bound's iteration count, with
# probability >= 1 - fail, theta^2 >= (1 - eps) sigma_max^2, i.e.
# sigma_max <= theta / sqrt(1 - eps)
_TIERS = ((1.0 / 64.0, 8.0), (1.0 / 16.0, 4.0), (0.25, 2.0), (0.5, math.sqrt(2.0)))


def _power_bound_iters(dim, one_minus_eps, fail):
    """Iterations q after which a sqrt(theta) Ritz value of the block subspace
    iteration on P^T P certifies sigma_max(P) <= theta / sqrt(1 - eps) except
    with probability <= fail.

    Kuczynski & Wozniakowski (1992), power method from a random start on a
    dim x dim PSD matrix: P[xi_k < (1 - eps) lambda_1] <= 0.824 sqrt(dim)
    (1 - eps)^(k - 1/2), xi_k the Rayleigh quotient after k steps.  The block
    iteration's span after q passes contains the power iterate with k = q - 1
    steps of its first start vector, and its top Ritz value theta satisfies
    theta^2 >= xi_{q-1} (Cauchy-Schwarz), so the power-method bound applies
    with k = q - 1.  The iteration tests the bound at every step: a union bound
    over steps (geometric in q) and over the len(_TIERS) tiers gives the factor
    len(_TIERS) / eps on top of `fail`."""
    eps = 1.0 - one_minus_eps
    budget = fail * eps / len(_TIERS)
    k = math.log(0.824 * math.sqrt(max(dim, 1)) / budget) / -math.log(one_minus_eps) + 0.5
    return int(math.ceil(k)) + 1


# starting block of the subspace iteration (grows while its smallest Ritz
# value is >= 1, i.e. while it may miss a singular value above 1)
SUBSPACE_BLOCK = 8


def _subspace_sigmas(op, n_total, m, r, block=None, max_iter=400, tol=None, seed=0):
    """Top singular values of P by randomized block subspace iteration with
    Rayleigh-Ritz; the block doubles until its smallest Ritz value < 1.
    Returns (sigmas, info)."""
    import torch

    dp, ops = op.dp, op.ops
    block = SUBSPACE_BLOCK if block is None else block
    tol = _SUBSPACE_TOL[op.precision] if tol is None else tol
    cap = max(1, min(m, n_total) - r)
    b = min(block, cap)
    n_loc = dp.n
    iters_total = 0
    bounds = [(ome, fac, _power_bound_iters(n_total, ome, _FAIL_PROB)) for ome, fac in _TIERS]
    while True:
        # start block drawn over all n_total rows (the same on every rank and
        # the same as a single-GPU run), each rank keeps its own rows
        w_all = np.random.default_rng(seed).standard_normal((n_total, b))
        w = torch.from_numpy(np.ascontiguousarray(w_all[ops.col0:ops.col0 + n_loc])).to(dp.device)
        q, _ = device_thin_qr(dp, op.proj_v(w), ops.host if ops.sharded else None)
        prev = None
        sig = np.zeros(0)
        converged = False
        for it in range(max_iter):
            if q.shape[1] == 0:  # P vanishes on the start block: sigma(P) = 0
                return np.zeros(0), {"t4_method": "subspace", "block": b,
                                     "iters": iters_total, "sigma_p_max": 0.0,
                                     "converged": True}
            y = op.right(q)
            qy, _ = device_thin_qr(dp, y)
            if qy.shape[1] == 0:
                return np.zeros(0), {"t4_method": "subspace", "block": b,
                                     "iters": iters_total + 1, "sigma_p_max": 0.0,
                                     "converged": True}
            wz = op.left(qy)  # (Qy^T P)^T: its singular values are the Ritz values
            ev = np.linalg.eigvalsh(ops.gram_rows(dp, wz, wz))
            sig = np.sqrt(np.clip(ev[::-1], 0.0, None))
            iters_total += 1
            if sig.size == b and sig[-1] >= 1.0 and b < cap:
                # Ritz values are lower bounds of the top b singular values:
                # sigma_b(P) >= 1 already, so this block cannot hold every
                # sigma > 1 -- grow it now rather than converge a clustered tail
                break
            t4 = float(np.sum(np.maximum(sig - 1.0, 0.0) ** 2))
            if prev is not None and abs(sig[0] - prev[0]) <= tol * max(1.0, sig[0]) and \
                    abs(t4 - prev[1]) <= tol * max(1.0, t4):
                converged = True
                break
            # t4 only needs sigma(P) against 1: a certified sigma_max(P) < 1
            # makes t4 = 0 exactly (the reference's dense value)
            for ome, fac, q_need in bounds:
                if it + 1 >= q_need and fac * sig[0] < 1.0:
                    return sig, {"t4_method": "subspace", "block": b, "iters": iters_total,
                                 "sigma_p_max": float(sig[0]), "converged": True,
                                 "t4_bound": f"sigma_max(P) <= {fac:.4g} theta_max < 1 after "
                                             f"{it + 1} >= {q_need} passes (power-method "
                                             f"bound, failure prob < {_FAIL_PROB:g} over "
                                             f"the random start)"}
            prev = (sig[0], t4)
            q, _ = device_thin_qr(dp, wz, ops.host if ops.sharded else None)
        info = {"t4_method": "subspace", "block": b, "iters": iters_total,
                "sigma_p_max": float(sig[0]) if sig.size else 0.0, "converged": converged}
        if sig.size == b and sig[-1] >= 1.0 and b < cap:
            b = min(2 * b, cap)
            continue
        if not converged:
            warnings.warn(f"certificate: subspace iteration for sigma(P) did not converge in "
                          f"{max_iter} passes; t4 is a lower bound", RuntimeWarning)
            return sig, info
        if sig.size == 0 or sig[-1] < 1.0 or b >= cap:
            return sig, info
        b = min(2 * b, cap)


def certificate_core(dp, z, m, n_total, k, lam, rank_tol, f_zero, f_bound_hint, ops):
    """The certificate (certificate.py:77-141) of the device iterate z = [U | V_p]
    against the device problem dp (a column shard when `ops` is sharded)."""
    u = z[: m * k].reshape(m, k)
    v = z[m * k:].reshape(dp.n, k)
    u1, sig, v1, all_sig, maps = _device_factor_svd(dp, u, v, rank_tol, ops)
    r = sig.shape[0]
    l_norm = float(np.sqrt(np.sum(all_sig * all_sig)))  # |U V^T|_F = |R_U R_V^T|_F
    if r > 0:
        prods = _gradient_products(dp, z, k, lam, ops) if maps is not None else None
        if prods is not None:
            gv1 = dp.matmul_small(prods[0], maps[1])
            gtu1 = dp.matmul_small(prods[1], maps[0])
        else:
            gv1, gtu1 = dp.apply(k, z, w_right=v1, w_left=u1)
            ops.dev(gv1)
        b = gv1.mul_(-1.0 / lam)  # D V1            (m x r)
        at = gtu1.mul_(-1.0 / lam)  # (U1^T D)^T     (n_p x r)
        c = ops.gram_rows(dp, at, v1)  # U1^T D V1 (r x r)
        csq = float(np.sum(c * c))
        t1 = float(np.sum((np.eye(r) - c) ** 2))
        t2 = float(np.trace(ops.gram_rows(dp, at, at))) - csq
        t3 = float(np.trace(dp.gram(b, b))) - csq
        if t2 < -1e-9 or t3 < -1e-9:  # certificate.py:108-115
            a2 = at - dp.matmul_small(v1, c.T)
            b2 = b - dp.matmul_small(u1, c)
            t2 = float(np.trace(ops.gram_rows(dp, a2, a2)))
            t3 = float(np.trace(dp.gram(b2, b2)))
            if t2 < -1e-9 or t3 < -1e-9:
                raise NumericalError(
                    f"certificate cross terms negative after recompute: t2={t2}, t3={t3}")
        t2, t3 = max(t2, 0.0), max(t3, 0.0)
    else:
        t1 = t2 = t3 = 0.0
        u1 = v1 = None
    precision = "fp32" if (m * n_total > FP32_PRODUCTS_MIN_ELEMS and "f32" in dp.store) \
        else "fp64"
    op = _ProjectedOperator(dp, z, k, lam, u1, v1, ops, precision)
    try:
        sp, info = _subspace_sigmas(op, n_total, m, r)
    finally:
        op.close()
    info["products"] = precision
    info["stored_gradient"] = op.stored_used
    over = np.maximum(sp - 1.0, 0.0)
    t4 = float(np.sum(over * over))
    info["n_sigma_over_1"] = int(np.sum(sp > 1.0))
    lsq = lam * lam
    terms = (lsq * t1, lsq * t2, lsq * t3, lsq * t4)
    e_norm = math.sqrt(sum(terms))
    f_bound = f_zero if f_bound_hint is None else min(float(f_bound_hint), f_zero)
    gap = e_norm * (l_norm + f_bound / lam)
    return CertificateReport(e_norm=e_norm, terms=terms, f_bound=f_bound, gap_bound=gap, r=r,
                             l_norm=l_norm, info=info)


def certificate(l_factors, spec, f_bound_hint=None, rank_tol=1e-10):
    """Certify L = U V^T for the convex objective (certificate.py:77-141)."""
    import torch

    from .device import nvtx_range

    m, n = spec.shape
    dp = spec.device("fp64")
    z = torch.from_numpy(np.ascontiguousarray(l_factors.flatten())).to(dp.device)
    with nvtx_range("spcp.certificate"):
        return certificate_core(dp, z, m, n, l_factors.k, spec.lambda_l, rank_tol, dp.f_zero,
                                f_bound_hint, CertOps(n_total=n))
