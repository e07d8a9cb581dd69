"""CPU oracle for the Split-SPCP hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference package's algorithm
(`/root/reference/pkg/src/spcp`, arXiv:1702.02241) for the one path this repo
accelerates: the marginalised Burer-Monteiro objective + gradient, the L-BFGS
driver with its strong-Wolfe line search, the rSVD initialisation and the
convergence certificate.  Every function cites the reference file:line it
restates.

Who may use it: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py`, and only as the
checker or the timed CPU baseline.  The product package
(`paper_1702_02241_b200`) never imports it; its compute path is CUDA only.

Parity pinning: `tests/golden/make_golden.py` imports the real reference (in
the build container, where `/root/reference` exists) and stores its outputs
as `.npz` fixtures; `tests/test_oracle_golden.py` checks this restatement
against those fixtures (bit-for-bit where the arithmetic order is the same,
to 1e-12 relative otherwise).

Numerics: float64 throughout, numpy + LAPACK, like the reference.
"""

from __future__ import annotations

import math
from collections import deque

import numpy as np

# --------------------------------------------------------------------------
# marginal function phi  (objective.py:62-117)
# --------------------------------------------------------------------------


def shrink(z, tau):
    """Soft threshold, objective.py:62-72."""
    if tau <= 0.0:
        raise ValueError("tau must be positive")
    z = np.asarray(z, dtype=np.float64)
    res = np.sign(z) * np.maximum(np.abs(z) - tau, 0.0)
    return res if res.ndim else float(res)


def huber(z, tau):
    """Huber envelope, ties take the quadratic branch; objective.py:75-87."""
    if tau <= 0.0:
        raise ValueError("tau must be positive")
    z = np.asarray(z, dtype=np.float64)
    mag = np.abs(z)
    res = np.where(mag <= tau, 0.5 * z * z, tau * mag - 0.5 * tau * tau)
    return res if res.ndim else float(res)


def phi_value_grad(l, x, lambda_s, mask=None):
    """(value, G, S*) of phi at dense L; objective.py:90-117.

    r = x - l (zeroed off the mask, :108-110); S* = shrink(r) (:111);
    G = -clip(r, +-lambda_s) (:112); value = sum huber(r) (:113-116).
    """
    tau = float(lambda_s)
    res = np.asarray(x, np.float64) - np.asarray(l, np.float64)
    if mask is not None:
        res = np.where(mask, res, 0.0)
    s_star = np.sign(res) * np.maximum(np.abs(res) - tau, 0.0)
    g = -np.clip(res, -tau, tau)
    mag = np.abs(res)
    val = float(np.sum(np.where(mag <= tau, 0.5 * res * res, tau * mag - 0.5 * tau * tau)))
    return val, g, s_star


def split_objective(u, v, x, lambda_l, lambda_s, mask=None):
    """F(U,V) and its factor gradients; solver.py:105-123.

    value = lam/2 (|U|^2 + |V|^2) + phi(U V^T) (:118-120);
    grad_u = G V + lam U (:121); grad_v = G^T U + lam V (:122).
    """
    u = np.asarray(u, np.float64)
    v = np.asarray(v, np.float64)
    phi, g, _ = phi_value_grad(u @ v.T, x, lambda_s, mask)
    lam = float(lambda_l)
    value = 0.5 * lam * (float(np.sum(u * u)) + float(np.sum(v * v))) + phi
    return value, g @ v + lam * u, g.T @ u + lam * v


def split_raw_products(u, v, x, lambda_s, mask=None):
    """(phi, G V, G^T U) without the regulariser: the raw reductions the
    survey asks to compare separately."""
    phi, g, _ = phi_value_grad(np.asarray(u) @ np.asarray(v).T, x, lambda_s, mask)
    return phi, g @ v, g.T @ u


def flat_objective(x, lambda_l, lambda_s, mask, m, n, k):
    """z -> (f, grad) adapter over concat(U.ravel(), V.ravel());
    solver.py:219-225 with FactorPair.from_flat solver.py:185-188."""

    def fun(z):
        z = np.asarray(z, np.float64)
        u = z[: m * k].reshape(m, k).copy()
        v = z[m * k:].reshape(n, k).copy()
        f, gu, gv = split_objective(u, v, x, lambda_l, lambda_s, mask)
        return f, np.concatenate([gu.ravel(), gv.ravel()])

    return fun


# --------------------------------------------------------------------------
# dense linear algebra primitives  (linalg.py:43-164)
# --------------------------------------------------------------------------


def thin_qr(a):
    """Reduced QR with diag(R) >= 0; linalg.py:43-59."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.shape[0] < a.shape[1]:
        raise ValueError("thin_qr requires m >= k")
    q, r = np.linalg.qr(a, mode="reduced")
    flip = np.where(np.diagonal(r) < 0.0, -1.0, 1.0)
    return q * flip, r * flip[:, None]


def svd_small(a):
    """Compact SVD (u, sigma, v) with v = Vt^T; linalg.py:62-74."""
    u, s, vt = np.linalg.svd(np.ascontiguousarray(a, np.float64), full_matrices=False)
    return u, s, vt.T.copy()


def rand_svd(a, k, oversample=10, power_iters=1, seed=0):
    """Gaussian-sketch randomized SVD with subspace power iteration;
    linalg.py:77-106 (sketch :97-99, power loop :100-103, core SVD :104-106)."""
    a = np.ascontiguousarray(a, np.float64)
    m, n = a.shape
    width = int(k) + int(oversample)
    if width > min(m, n):
        raise ValueError("sketch width exceeds min(m, n)")
    omega = np.random.default_rng(seed).standard_normal((n, width))
    q = thin_qr(a @ omega)[0]
    for _ in range(int(power_iters)):
        q = thin_qr(a.T @ q)[0]
        q = thin_qr(a @ q)[0]
    ub, s, vb = svd_small(q.T @ a)
    return (q @ ub)[:, :k], s[:k].copy(), vb[:, :k].copy()


def leading_triple(matvec, rmatvec, m, n, tol=1e-9, max_iter=1000, seed=0):
    """Alternating power iteration for (u, sigma_1, v); linalg.py:109-164.

    Returns (u, sigma, v, converged).  The reference raises
    PowerIterationError carrying the last iterate on cap exhaustion
    (:158-164); here that case returns converged=False with the iterate.
    """
    v = np.random.default_rng(seed).standard_normal(int(n))
    v /= np.linalg.norm(v)
    u = np.zeros(int(m))
    sig = 0.0
    for _ in range(int(max_iter)):
        u = np.asarray(matvec(v), np.float64).reshape(int(m))
        su = float(np.linalg.norm(u))
        if su == 0.0:
            u = np.zeros(int(m))
            u[0] = 1.0
            return u, 0.0, v, True
        u /= su
        w = np.asarray(rmatvec(u), np.float64).reshape(int(n))
        sv = float(np.linalg.norm(w))
        if sv == 0.0:
            return u, su, v, True
        v = w / sv
        if abs(sv - sig) <= tol * max(1.0, sv):
            u = np.asarray(matvec(v), np.float64).reshape(int(m))
            sig = float(np.linalg.norm(u))
            if sig > 0.0:
                u /= sig
            return u, sig, v, True
        sig = sv
    return u, sig, v, False


# --------------------------------------------------------------------------
# initialisation  (solver.py:126-154)
# --------------------------------------------------------------------------


def init_factors(x, k, strategy="rsvd", seed=0, mask=None, oversample=10, power_iters=1):
    """Balanced spectral (or random) starting factors; solver.py:126-154."""
    x = np.asarray(x, np.float64)
    m, n = x.shape
    if strategy == "random":
        gen = np.random.default_rng(seed)
        sc = 1.0 / math.sqrt(k)
        return sc * gen.standard_normal((m, k)), sc * gen.standard_normal((n, k))
    obs = x if mask is None else np.where(mask, x, 0.0)
    if strategy == "full_svd":
        uu, ss, vv = svd_small(obs)
        uu, ss, vv = uu[:, :k], ss[:k], vv[:, :k]
    elif strategy == "rsvd":
        uu, ss, vv = rand_svd(obs, k, oversample=min(int(oversample), min(m, n) - k),
                              power_iters=power_iters, seed=seed)
    else:
        raise ValueError(f"unknown init strategy {strategy!r}")
    root = np.sqrt(ss)
    return uu * root, vv * root


# --------------------------------------------------------------------------
# L-BFGS with strong Wolfe line search  (lbfgs.py:32-194)
# --------------------------------------------------------------------------

MAX_BRACKET = 30  # lbfgs.py:18
MAX_ZOOM = 40  # lbfgs.py:19


def cubic_min(a, fa, da, b, fb, db):
    """Minimiser of the interpolating cubic, NaN when undefined; lbfgs.py:32-42."""
    t1 = da + db - 3.0 * (fa - fb) / (a - b)
    disc = t1 * t1 - da * db
    if disc < 0.0:
        return math.nan
    t2 = math.copysign(math.sqrt(disc), b - a) if b != a else 0.0
    den = db - da + 2.0 * t2
    if den == 0.0:
        return math.nan
    return b - (b - a) * (db + t2 - t1) / den


def strong_wolfe(phi, f0, df0, alpha0, c1, c2):
    """Bracket (<=30 doublings) then zoom (<=40 cubic/bisection trials);
    lbfgs.py:64-99.  `phi(alpha) -> (f, df, g)`; returns (alpha, f, g) or None."""

    def zoom(lo, flo, dlo, hi, fhi, dhi):
        for _ in range(MAX_ZOOM):  # lbfgs.py:68
            a_, b_ = min(lo, hi), max(lo, hi)
            width = b_ - a_
            if width <= 1e-16 * max(1.0, abs(lo)):  # :71-72
                return None
            al = cubic_min(lo, flo, dlo, hi, fhi, dhi)
            if not math.isfinite(al) or al <= a_ + 0.1 * width or al >= b_ - 0.1 * width:
                al = 0.5 * (a_ + b_)  # :74-75
            f, df, g = phi(al)
            if f > f0 + c1 * al * df0 or f >= flo:  # :77-78
                hi, fhi, dhi = al, f, df
                continue
            if abs(df) <= -c2 * df0:  # :80-81
                return al, f, g
            if df * (hi - lo) >= 0.0:  # :82-83
                hi, fhi, dhi = lo, flo, dlo
            lo, flo, dlo = al, f, df  # :84
        return None

    a_prev, f_prev, d_prev = 0.0, f0, df0
    al = alpha0
    for i in range(MAX_BRACKET):  # :89
        f, df, g = phi(al)
        if f > f0 + c1 * al * df0 or (i > 0 and f >= f_prev):  # :91-92
            return zoom(a_prev, f_prev, d_prev, al, f, df)
        if abs(df) <= -c2 * df0:  # :93-94
            return al, f, g
        if df >= 0.0:  # :95-96
            return zoom(al, f, df, a_prev, f_prev, d_prev)
        a_prev, f_prev, d_prev = al, f, df
        al = 2.0 * al  # :98
    return None


def minimize_lbfgs(fun, x0, memory=10, grad_tol=1e-9, max_iter=500, c1=1e-4, c2=0.9,
                   iter_hook=None):
    """Two-loop L-BFGS; lbfgs.py:102-194.

    Returns dict(x, objective, grad_norm, termination, records, n_evals) where
    records is a list of (iteration, objective, grad_norm, extra-dict).
    """
    if not 0.0 < c1 < c2 < 1.0:
        raise ValueError("need 0 < c1 < c2 < 1")
    if memory < 1:
        raise ValueError("memory must be >= 1")
    x = np.array(x0, dtype=np.float64, copy=True)
    f, g = fun(x)
    evals = 1
    gn = float(np.linalg.norm(g))
    stop = grad_tol * max(1.0, gn)  # lbfgs.py:133
    recs = []

    def log(it):
        ex = iter_hook(it, x) if iter_hook is not None else None
        recs.append((it, float(f), gn, dict(ex or {})))

    log(0)
    if gn <= stop:
        return dict(x=x, objective=float(f), grad_norm=gn, termination="converged",
                    records=recs, n_evals=evals)
    pairs = deque(maxlen=int(memory))  # lbfgs.py:148
    term = "max_iter"
    for it in range(1, int(max_iter) + 1):
        q = g.copy()  # two-loop recursion lbfgs.py:152-163
        coef = []
        for s, y, rho in reversed(pairs):
            a = rho * (s @ q)
            coef.append(a)
            q -= a * y
        if pairs:
            s, y, _ = pairs[-1]
            q *= (s @ y) / (y @ y)
        for (s, y, rho), a in zip(pairs, reversed(coef)):
            q += (a - rho * (y @ q)) * s
        d = -q
        dg = float(d @ g)
        if dg >= 0.0:  # lbfgs.py:165-171
            pairs.clear()
            d = -g
            dg = -(gn ** 2)
        a0 = 1.0 if pairs else min(1.0, 1.0 / max(gn, 1e-12))  # :173
        n_here = [0]

        def phi(al, x=x, d=d):
            fv, gv = fun(x + al * d)
            n_here[0] += 1
            if not np.isfinite(fv):  # lbfgs.py:58-59
                fv = math.inf
            return fv, float(gv @ d), gv

        hit = strong_wolfe(phi, f, dg, a0, c1, c2)
        evals += n_here[0]
        if hit is None:
            term = "line_search_failed"
            break
        al, f_new, g_new = hit
        s_vec = al * d
        y_vec = g_new - g
        sy = float(s_vec @ y_vec)
        if sy > 1e-12 * float(np.linalg.norm(s_vec)) * float(np.linalg.norm(y_vec)):  # :184
            pairs.append((s_vec, y_vec, 1.0 / sy))
        x = x + s_vec
        f, g = f_new, g_new
        gn = float(np.linalg.norm(g))
        log(it)
        if gn <= stop:
            term = "converged"
            break
    return dict(x=x, objective=float(f), grad_norm=gn, termination=term, records=recs,
                n_evals=evals)


# --------------------------------------------------------------------------
# end-to-end split solve  (solver.py:228-324)
# --------------------------------------------------------------------------


def growth_column(u, v, x, lambda_s, mask, seed):
    """Append sqrt(1e-3 s1)(u1, v1) from the leading triple of -G;
    solver.py:228-252."""
    _, g, _ = phi_value_grad(u @ v.T, x, lambda_s, mask)
    m, n = g.shape
    u1, s1, v1, _ = leading_triple(lambda z: -(g @ z), lambda y: -(g.T @ y), m, n,
                                   tol=1e-6, seed=seed)
    if not s1 > 0.0:
        return None
    root = math.sqrt(1e-3 * s1)
    return np.hstack([u, root * u1[:, None]]), np.hstack([v, root * v1[:, None]])


def solve_split_spcp(x, lambda_l, lambda_s, k, mask=None, memory=10, grad_tol=1e-8,
                     max_iter=500, c1=1e-4, c2=0.9, rank_growth=False, max_k=None,
                     growth_tol=1e-6, seed=0, init="rsvd", iter_hook=None):
    """solver.py:255-324.  Returns a dict mirroring SolveReport fields."""
    x = np.asarray(x, np.float64)
    m, n = x.shape
    if not 1 <= k <= min(m, n):
        raise ValueError("k out of range")
    u, v = init_factors(x, k, strategy=init, seed=seed, mask=mask)
    cap = max_k if max_k is not None else min(m, n)
    recs, evals, offset, grown = [], 0, 0, 0
    best = None
    while True:
        kk = u.shape[1]
        hook = None
        if iter_hook is not None:
            def hook(it, z, kk=kk, offset=offset):
                return iter_hook(offset + it, z[: m * kk].reshape(m, kk),
                                 z[m * kk:].reshape(n, kk))
        res = minimize_lbfgs(flat_objective(x, lambda_l, lambda_s, mask, m, n, kk),
                             np.concatenate([u.ravel(), v.ravel()]), memory=memory,
                             grad_tol=grad_tol, max_iter=max_iter, c1=c1, c2=c2,
                             iter_hook=hook)
        evals += res["n_evals"]
        for (it, fo, gn, ex) in res["records"]:
            ex = dict(ex)
            ex.setdefault("rank", kk)
            recs.append((it + offset, fo, gn, ex))
        offset = recs[-1][0] + 1 if recs else 0
        z = res["x"]
        u, v = z[: m * kk].reshape(m, kk).copy(), z[m * kk:].reshape(n, kk).copy()
        prev = best["objective"] if best is not None else None
        if best is None or res["objective"] < best["objective"]:
            best = dict(objective=res["objective"], termination=res["termination"],
                        u=u, v=v)
        stationary = res["termination"] in ("converged", "line_search_failed")
        if not (rank_growth and stationary and kk < cap):
            break
        if prev is not None and (prev - res["objective"]) / max(1.0, abs(prev)) < growth_tol:
            break
        nxt = growth_column(u, v, x, lambda_s, mask, seed + grown + 1)
        if nxt is None:
            break
        u, v = nxt
        grown += 1
    lf = best["u"] @ best["v"].T
    _, _, s_star = phi_value_grad(lf, x, lambda_s, mask)
    return dict(termination=best["termination"], records=recs, l=lf, s=s_star,
                objective=best["objective"], u=best["u"], v=best["v"],
                k_final=best["u"].shape[1], columns_grown=grown, n_evals=evals)


# --------------------------------------------------------------------------
# certificate  (certificate.py:50-141)
# --------------------------------------------------------------------------


def factor_svd(u, v, rank_tol=1e-10):
    """Compact SVD of U V^T via two thin QRs and a k x k SVD;
    certificate.py:50-67."""
    qu, ru = thin_qr(u)
    qv, rv = thin_qr(v)
    cu, cs, cv = svd_small(ru @ rv.T)
    r = 0 if (cs.size == 0 or cs[0] <= 0.0) else int(np.sum(cs > rank_tol * cs[0]))
    return (qu @ cu)[:, :r], cs[:r].copy(), (qv @ cv)[:, :r]


def complement_term(p):
    """sum max(sigma(P) - 1, 0)^2 by dense SVD; certificate.py:70-74."""
    sig = np.linalg.svd(np.asarray(p, np.float64), compute_uv=False)
    over = np.maximum(sig - 1.0, 0.0)
    return float(np.sum(over * over))


def certificate(u, v, x, lambda_l, lambda_s, mask=None, f_bound_hint=None, rank_tol=1e-10):
    """Four-term subgradient distance, f_bound and gap bound;
    certificate.py:77-141.  Returns a dict mirroring CertificateReport."""
    lam = float(lambda_l)
    lmat = np.asarray(u) @ np.asarray(v).T
    _, g, _ = phi_value_grad(lmat, x, lambda_s, mask)
    dmat = -g / lam  # :95
    u1, sig, v1 = factor_svd(u, v, rank_tol=rank_tol)
    r = sig.shape[0]
    if r > 0:
        a = u1.T @ dmat
        b = dmat @ v1
        c = a @ v1
        csq = float(np.sum(c * c))
        t1 = float(np.sum((np.eye(r) - c) ** 2))
        t2 = float(np.sum(a * a)) - csq
        t3 = float(np.sum(b * b)) - csq
        if t2 < -1e-9 or t3 < -1e-9:  # :108-115
            t2 = float(np.sum((a - c @ v1.T) ** 2))
            t3 = float(np.sum((b - u1 @ c) ** 2))
        t2, t3 = max(t2, 0.0), max(t3, 0.0)
        p = dmat - u1 @ a - b @ v1.T + u1 @ (c @ v1.T)  # :118
        t4 = complement_term(p)
    else:
        t1 = t2 = t3 = 0.0
        t4 = complement_term(dmat)
    lsq = lam * lam
    terms = (lsq * t1, lsq * t2, lsq * t3, lsq * t4)
    e_norm = math.sqrt(sum(terms))
    obs = x if mask is None else np.where(mask, x, 0.0)
    f_zero = 0.5 * float(np.sum(np.asarray(obs, np.float64) ** 2))
    f_bound = f_zero if f_bound_hint is None else min(float(f_bound_hint), f_zero)
    l_norm = float(np.linalg.norm(lmat))
    return dict(e_norm=e_norm, terms=terms, f_bound=f_bound,
                gap_bound=e_norm * (l_norm + f_bound / lam), r=r, l_norm=l_norm)


def certificate_warns(cert, objective):
    """CLI under-rank warning predicate; cli.py:27,246-251."""
    return cert["gap_bound"] > 1e-2 * max(1.0, abs(objective))


# --------------------------------------------------------------------------
# synthetic inputs  (synth.py:13-73)
# --------------------------------------------------------------------------


def gen_low_rank_plus_sparse(m, n, rank, sparse_frac, noise_rel, seed=0):
    """x = A B^T + S + a z with exact outlier count and noise ratio;
    synth.py:13-57 (same PCG64 draw order so outputs are bit-identical)."""
    gen = np.random.default_rng(seed)
    a = gen.standard_normal((m, rank))
    b = gen.standard_normal((n, rank))
    l_ref = a @ b.T
    s_ref = np.zeros((m, n))
    cnt = int(round(sparse_frac * m * n))
    if cnt > 0:
        pos = gen.choice(m * n, size=cnt, replace=False)
        s_ref.flat[pos] = gen.standard_normal(cnt)
    clean = l_ref + s_ref
    if noise_rel == 0.0:
        return clean.copy(), l_ref, s_ref
    z = gen.standard_normal((m, n))
    rho2 = noise_rel * noise_rel
    zz = float(np.sum(z * z))
    cz = float(np.sum(clean * z))
    cc = float(np.sum(clean * clean))
    qa, qb, qc = zz * (1.0 - rho2), -2.0 * rho2 * cz, -rho2 * cc
    scale = (-qb + math.sqrt(qb * qb - 4.0 * qa * qc)) / (2.0 * qa)
    return clean + scale * z, l_ref, s_ref


def gen_mask(m, n, observe_frac, seed=0):
    """Exactly round(frac m n) observed entries; synth.py:60-73."""
    cnt = int(round(observe_frac * m * n))
    out = np.zeros((m, n), dtype=bool)
    out.flat[np.random.default_rng(seed).choice(m * n, size=cnt, replace=False)] = True
    return out
