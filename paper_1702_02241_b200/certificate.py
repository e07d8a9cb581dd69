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
    SVD of the m x n P.  Here P is never formed for large problems: a block
    subspace iteration applies P and P^T through streaming passes (D W and
    D^T Y computed from X on the fly, then projected) and the Ritz values
    give sigma_i(P); the block grows until its smallest Ritz value is below 1
    so every sigma > 1 is captured.  Small problems (dense_limit) take the
    reference's dense route on the device.
"""

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import NumericalError
from .linalg import SvdTriplet, device_thin_qr, svd_small, thin_qr

__all__ = ["CertificateReport", "factor_svd", "certificate", "DENSE_LIMIT"]

DENSE_LIMIT = 4096 * 4096  # entries of P below which t4 uses the dense SVD


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


def _device_factor_svd(dp, z, m, n, k, rank_tol, gram_reduce=None, v_rows=None):
    """factor_svd on device factors; returns (u1 dev m x r, sigma, v1 dev n x r,
    all singular values)."""
    uu = z[: m * k].reshape(m, k)
    vv = z[m * k:].reshape(v_rows if v_rows is not None else n, k)
    qu, ru = device_thin_qr(dp, uu)
    qv, rv = device_thin_qr(dp, vv, gram_reduce)
    core = svd_small(ru @ rv.T)
    sig = core.sigma
    r = 0 if (sig.size == 0 or sig[0] <= 0.0) else int(np.sum(sig > rank_tol * sig[0]))
    if r == 0:
        return None, sig[:0], None, sig
    u1 = dp.matmul_small(qu, core.u[:, :r])
    v1 = dp.matmul_small(qv, core.v[:, :r])
    return u1, sig[:r].copy(), v1, sig


def _sq(dp, a):
    return float(np.trace(dp.gram(a, a)))


def _dense_sigmas(dp, z, k, lam, u1, v1):
    """sigma(P) by the reference's dense route, computed on the device."""
    import torch

    g = dp.grad_dense(k, z)
    d = g.mul_(-1.0 / lam)
    if u1 is not None:
        d = d - u1 @ (u1.T @ d)
        d = d - (d @ v1) @ v1.T
    return torch.linalg.svdvals(d).cpu().numpy()


class _ProjectedOperator:
    """x -> P x and y -> P^T y with P = (I - U1U1^T) D (I - V1V1^T), D = -G/lam,
    every D product a streaming pass over X (spcp_apply)."""

    def __init__(self, dp, z, k, lam, u1, v1):
        self.dp, self.z, self.k, self.lam, self.u1, self.v1 = dp, z, k, lam, u1, v1

    def _proj(self, basis, w):
        if basis is None:
            return w
        c = self.dp.gram(basis, w)
        return w - self.dp.matmul_small(basis, c)

    # The subspace iteration only compares sigma(P) against 1, so its D
    # products stream X in fp32 (spcp_apply_f32; fp64 when no fp32 copy of X is
    # stored).  The cross terms t1..t3 keep the fp64 products.
    def right(self, w):  # P w, w: n x b
        w = self._proj(self.v1, w)
        y, _ = self.dp.apply(self.k, self.z, w_right=w.contiguous(), precision="fp32")
        return self._proj(self.u1, y.mul_(-1.0 / self.lam))

    def left(self, y):  # P^T y, y: m x b
        y = self._proj(self.u1, y)
        _, w = self.dp.apply(self.k, self.z, w_left=y.contiguous(), precision="fp32")
        return self._proj(self.v1, w.mul_(-1.0 / self.lam))


_SUBSPACE_TOL = 1e-9


def _q_bound(n, eps=0.5, fail=1e-6):
    """Iterations after which 1.648 sqrt(n) e^(-eps (2q - 1)) <= fail."""
    return int(math.ceil((math.log(1.648 * math.sqrt(max(n, 1)) / fail) / eps + 1.0) / 2.0))


def _subspace_sigmas(op, n, m, r, block=16, max_iter=60, tol=None, seed=0):
    """Top singular values of P by randomized block subspace iteration with
    Rayleigh-Ritz; the block doubles until its smallest Ritz value < 1."""
    import torch

    dp = op.dp
    tol = _SUBSPACE_TOL if tol is None else tol
    cap = max(1, min(m, n) - r)
    b = min(block, cap)
    iters_total = 0
    while True:
        w = torch.from_numpy(np.random.default_rng(seed).standard_normal((n, b))).to(dp.device)
        q, _ = device_thin_qr(dp, op._proj(op.v1, w))
        prev = None
        sig = None
        for it in range(max_iter):
            y = op.right(q)
            qy, _ = device_thin_qr(dp, y)
            wz = op.left(qy)  # (Qy^T P)^T: its singular values are the Ritz values
            ev = np.linalg.eigvalsh(dp.gram(wz, wz))
            sig = np.sqrt(np.clip(ev[::-1], 0.0, None))
            iters_total += 1
            t4 = float(np.sum(np.maximum(sig - 1.0, 0.0) ** 2))
            if prev is not None and abs(sig[0] - prev[0]) <= tol * max(1.0, sig[0]) and \
                    abs(t4 - prev[1]) <= tol * max(1.0, t4):
                break
            # t4 only needs sigma(P) against 1.  After q steps from a Gaussian start
            # the top Ritz value theta of the subspace (power) iteration on P^T P
            # satisfies P[theta^2 < (1 - eps) sigma_max^2] <= 1.648 sqrt(n)
            # e^(-eps (2q - 1)) (Kuczynski & Wozniakowski 1992).  With eps = 1/2 and
            # q >= _Q_BOUND(n) that is < 1e-6, so sqrt(2) theta < 1 proves every
            # sigma(P) < 1 and t4 = 0 exactly (the reference's dense SVD value).
            if it + 1 >= _q_bound(n) and math.sqrt(2.0) * sig[0] < 1.0:
                return sig, {"t4_method": "subspace", "block": b, "iters": iters_total,
                             "sigma_p_max": float(sig[0]),
                             "t4_bound": "sigma_max(P) < sqrt(2) theta_max < 1 "
                                         "(failure prob < 1e-6)"}
            prev = (sig[0], t4)
            q, _ = device_thin_qr(dp, wz)
        if sig[-1] < 1.0 or b >= cap:
            return sig, {"t4_method": "subspace", "block": b, "iters": iters_total,
                         "sigma_p_max": float(sig[0])}
        b = min(2 * b, cap)


def certificate(l_factors, spec, f_bound_hint=None, rank_tol=1e-10, dense_limit=DENSE_LIMIT):
    """Certify L = U V^T for the convex objective (certificate.py:77-141)."""
    import torch

    lam = spec.lambda_l
    m, n = spec.shape
    k = l_factors.k
    dp = spec.device("fp64")
    z = torch.from_numpy(np.ascontiguousarray(l_factors.flatten())).to(dp.device)
    u1, sig, v1, all_sig = _device_factor_svd(dp, z, m, n, k, rank_tol)
    r = sig.shape[0]
    l_norm = float(np.sqrt(np.sum(all_sig * all_sig)))  # |U V^T|_F = |R_U R_V^T|_F
    info = {}
    if r > 0:
        gv1, gtu1 = dp.apply(k, z, w_right=v1, w_left=u1)
        b = gv1.mul_(-1.0 / lam)  # D V1            (m x r)
        at = gtu1.mul_(-1.0 / lam)  # (U1^T D)^T     (n x r)
        c = dp.gram(at, v1)  # U1^T D V1 (r x r)
        csq = float(np.sum(c * c))
        t1 = float(np.sum((np.eye(r) - c) ** 2))
        t2 = _sq(dp, at) - csq
        t3 = _sq(dp, b) - csq
        if t2 < -1e-9 or t3 < -1e-9:  # certificate.py:108-115
            t2 = _sq(dp, at - dp.matmul_small(v1, c.T))
            t3 = _sq(dp, b - dp.matmul_small(u1, c))
            if t2 < -1e-9 or t3 < -1e-9:
                raise NumericalError(
                    f"certificate cross terms negative after recompute: t2={t2}, t3={t3}")
        t2, t3 = max(t2, 0.0), max(t3, 0.0)
    else:
        t1 = t2 = t3 = 0.0
        u1 = v1 = None
    if m * n <= dense_limit:
        sp = _dense_sigmas(dp, z, k, lam, u1, v1)
        info = {"t4_method": "dense", "sigma_p_max": float(sp[0]) if sp.size else 0.0}
    else:
        op = _ProjectedOperator(dp, z, k, lam, u1, v1)
        sp, info = _subspace_sigmas(op, n, m, r)
    over = np.maximum(sp - 1.0, 0.0)
    t4 = float(np.sum(over * over))
    info["n_sigma_over_1"] = int(np.sum(sp > 1.0))
    lsq = lam * lam
    terms = (lsq * t1, lsq * t2, lsq * t3, lsq * t4)
    e_norm = math.sqrt(sum(terms))
    f_zero = dp.f_zero
    f_bound = f_zero if f_bound_hint is None else min(float(f_bound_hint), f_zero)
    gap = e_norm * (l_norm + f_bound / lam)
    return CertificateReport(e_norm=e_norm, terms=terms, f_bound=f_bound, gap_bound=gap, r=r,
                             l_norm=l_norm, info=info)
