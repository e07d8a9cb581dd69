"""Dense factorisation primitives (spcp linalg.py:18-164).

Host functions keep the reference API for small dense inputs (k x k cores,
test matrices): `thin_qr`, `svd_small`, `leading_triple`.  The m x n work of
the solve path runs on the GPU:

* `rand_svd_device` — randomized SVD of the zero-filled observed matrix
  held in HBM (linalg.py:77-106): the four sketch passes are the RAW mode of
  the fused streaming kernel (`spcp_apply`, k = 0), the tall QRs are
  CholeskyQR2 on the device (Gram + small host Cholesky + device triangular
  multiply), the w x n core SVD is LAPACK on the host as in the reference.
  The Gaussian test matrix is drawn on the host with the reference's PCG64
  stream so the starting point is the reference's.
* `rand_svd` — the reference signature for a dense numpy matrix (uploads it).
"""

from dataclasses import dataclass

import numpy as np

from .errors import DimensionError, NumericalError, PowerIterationError
from .validation import as_matrix

__all__ = ["SvdTriplet", "thin_qr", "svd_small", "rand_svd", "leading_triple",
           "rand_svd_device", "device_thin_qr"]


@dataclass(frozen=True)
class SvdTriplet:
    """a = u diag(sigma) v^T, sigma non-increasing (linalg.py:18-40)."""

    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray

    @property
    def rank(self):
        return self.sigma.shape[0]

    def compose(self):
        return (self.u * self.sigma) @ self.v.T

    def truncate(self, r):
        return SvdTriplet(self.u[:, :r].copy(), self.sigma[:r].copy(), self.v[:, :r].copy())


def thin_qr(a):
    """Reduced QR with non-negative diag(R) (linalg.py:43-59)."""
    a = as_matrix(a, "a")
    if a.shape[0] < a.shape[1]:
        raise DimensionError(f"thin_qr requires m >= k, got shape {a.shape}")
    q, r = np.linalg.qr(a, mode="reduced")
    sgn = np.where(np.diagonal(r) < 0.0, -1.0, 1.0)
    return q * sgn, r * sgn[:, None]


def svd_small(a):
    """Compact SVD of a small dense matrix (linalg.py:62-74)."""
    a = as_matrix(a, "a")
    try:
        u, s, vt = np.linalg.svd(a, full_matrices=False)
    except np.linalg.LinAlgError as exc:
        raise NumericalError(f"SVD did not converge for shape {a.shape}: {exc}") from exc
    return SvdTriplet(u, s, vt.T.copy())


def leading_triple(matvec, rmatvec, m, n, tol=1e-9, max_iter=1000, seed=0, v0=None):
    """Alternating power iteration for the leading singular triple
    (linalg.py:109-164).  matvec / rmatvec may act on numpy arrays (host
    operators) — the solver's growth step uses the device variant in
    solver.py, which feeds the same recurrence with streaming-kernel products."""
    m, n = int(m), int(n)
    v = None
    if v0 is not None:
        v = np.asarray(v0, dtype=np.float64).reshape(n).copy()
        nv = float(np.linalg.norm(v))
        v = v / nv if nv != 0.0 else None
    if v is None:
        v = np.random.default_rng(seed).standard_normal(n)
        v /= np.linalg.norm(v)
    u = np.zeros(m)
    sigma = 0.0
    for _ in range(int(max_iter)):
        u = np.asarray(matvec(v), dtype=np.float64).reshape(m)
        su = float(np.linalg.norm(u))
        if su == 0.0:
            u = np.zeros(m)
            u[0] = 1.0
            return u, 0.0, v
        u /= su
        w = np.asarray(rmatvec(u), dtype=np.float64).reshape(n)
        sv = float(np.linalg.norm(w))
        if sv == 0.0:
            return u, su, v
        v = w / sv
        if abs(sv - sigma) <= tol * max(1.0, sv):
            u = np.asarray(matvec(v), dtype=np.float64).reshape(m)
            sigma = float(np.linalg.norm(u))
            if sigma > 0.0:
                u /= sigma
            return u, sigma, v
        sigma = sv
    raise PowerIterationError(
        f"power iteration did not converge in {max_iter} iterations (last sigma = {sigma:.6e})",
        u=u, sigma=sigma, v=v)


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------


def _chol_upper(g):
    """Upper R with R^T R = g, or None when g is not numerically PD."""
    try:
        low = np.linalg.cholesky(g)
    except np.linalg.LinAlgError:
        return None
    d = np.abs(np.diagonal(low))
    if d.min() <= 1e-7 * d.max():
        return None
    return low.T


def device_thin_qr(dp, a, gram_reduce=None):
    """Q, R (R host) of a tall float64 device matrix a (rows x w), A = Q R.

    CholeskyQR2: R1 = chol(a^T a), Q1 = a R1^-1, R2 = chol(Q1^T Q1),
    Q = Q1 R2^-1, R = R2 R1 (unique for full column rank with diag(R) > 0, so
    Q matches the reference's Householder QR with the diag(R) >= 0 convention,
    linalg.py:43-59).  `gram_reduce` sums Grams across column-sharded ranks
    (row-sharded a).

    Numerically rank-deficient input (the certificate's factor QRs of a
    rank-deficient product, a subspace block P W with rank(P) < w) takes an
    eigenbasis route on the same device Grams: Q = A W_r diag(l_r)^-1/2 over
    the r eigenpairs above the noise floor, re-orthonormalised by one
    CholeskyQR pass, R = Q^T A (r x w, not triangular).  Q then has r <= w
    columns; every caller only needs A = Q R with orthonormal Q (the factor
    SVD uses R_U R_V^T, the subspace iteration only span(Q)).
    """
    red = gram_reduce or (lambda x: x)
    g1 = red(dp.gram(a, a))
    r1 = _chol_upper(g1)
    if r1 is not None:
        q1 = dp.matmul_small(a, np.linalg.inv(r1))
        g2 = red(dp.gram(q1, q1))
        r2 = _chol_upper(g2)
        if r2 is not None:
            q = dp.matmul_small(q1, np.linalg.inv(r2))
            return q, r2 @ r1
    lam, wv = np.linalg.eigh(0.5 * (g1 + g1.T))
    lam, wv = lam[::-1], wv[:, ::-1]
    top = float(lam[0]) if lam.size else 0.0
    keep = lam > max(top, 0.0) * 1e-13 if top > 0.0 else np.zeros(lam.shape, bool)
    w = a.shape[1]
    if not keep.any():
        return a[:, :0].contiguous(), np.zeros((0, w))
    q1 = dp.matmul_small(a, wv[:, keep] / np.sqrt(lam[keep]))
    r2 = _chol_upper(red(dp.gram(q1, q1)))
    if r2 is None:
        raise NumericalError("device_thin_qr: re-orthonormalisation of the eigenbasis failed")
    q = dp.matmul_small(q1, np.linalg.inv(r2))
    return q, red(dp.gram(q, a))


def rand_svd_device(dp, k, oversample=10, power_iters=1, seed=0, omega=None):
    """Randomized rank-k SVD of P_Omega(X) resident in `dp` (linalg.py:77-106).

    Returns (u device m x k, sigma host, v host n x k)."""
    import torch

    m, n = dp.m, dp.n
    k = int(k)
    width = k + int(oversample)
    if k < 1:
        raise DimensionError(f"rand_svd requires k >= 1, got {k}")
    if width > min(m, n):
        raise DimensionError(
            f"sketch width k + oversample = {width} exceeds min(m, n) = {min(m, n)}")
    if omega is None:
        omega = np.random.default_rng(seed).standard_normal((n, width))
    om = torch.from_numpy(np.ascontiguousarray(omega)).to(dp.device)
    y, _ = dp.apply(0, None, w_right=om)
    q, _ = device_thin_qr(dp, y)
    for _ in range(int(power_iters)):
        _, z = dp.apply(0, None, w_left=q)
        q2, _ = device_thin_qr(dp, z)
        y, _ = dp.apply(0, None, w_right=q2)
        q, _ = device_thin_qr(dp, y)
    _, bt = dp.apply(0, None, w_left=q)  # B^T = X^T Q  (n x width)
    inner = svd_small(bt.cpu().numpy().T)  # B = Q^T X  (width x n), LAPACK as the reference
    u = dp.matmul_small(q, inner.u[:, :k])
    return u, inner.sigma[:k].copy(), inner.v[:, :k].copy()


def rand_svd(a, k, oversample=10, power_iters=1, seed=0):
    """Reference signature (linalg.py:77-106) for a dense host matrix."""
    from .objective import ProblemSpec

    a = as_matrix(a, "a")
    m, n = a.shape
    if int(k) < 1:
        raise DimensionError(f"rand_svd requires k >= 1, got {k}")
    if int(k) + int(oversample) > min(m, n):
        raise DimensionError(
            f"sketch width k + oversample = {int(k) + int(oversample)} exceeds min(m, n) = "
            f"{min(m, n)}")
    spec = ProblemSpec(x=a, lambda_l=1.0, lambda_s=1.0)
    dp = spec.device("fp64")
    u, s, v = rand_svd_device(dp, k, oversample, power_iters, seed)
    out = SvdTriplet(u.cpu().numpy(), s, v)
    spec.release_device()
    return out
