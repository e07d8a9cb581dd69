"""Limited-memory BFGS with a strong-Wolfe line search (spcp lbfgs.py:1-194).

Two drivers share one line search (`strong_wolfe`, lbfgs.py:64-99):

* `minimize_lbfgs(fun, x0, ...)` — the reference's plug-in API: `fun(z) ->
  (value, gradient)` on float64 numpy vectors (any user callable).  Same
  control flow, constants, termination reasons and trace records.
* `DeviceLbfgs` — the same iteration with every (m+n)k-length vector resident
  in HBM.  The two-loop recursion is evaluated from inner products gathered
  in ONE pass over the history per iteration (`spcp_vec_gram`): with
  q_i = g - sum_{j newer} a_j y_j and r_i = gamma q_0 + sum_{j older}
  (a_j - b_j) s_j, every s_i.q_i and y_i.r_i is a combination of the cached
  dots S^T g, Y^T g, S^T Y, Y^T Y, so the host computes the coefficients and
  one kernel forms d = -(gamma g - gamma sum a_j y_j + sum (a_i - b_i) s_i).
  The host only ever sees scalars.
"""

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .report import IterationRecord, WorkTimer

__all__ = ["LbfgsResult", "minimize_lbfgs", "strong_wolfe", "DeviceLbfgs"]

BRACKET_LIMIT = 30  # lbfgs.py:18
ZOOM_LIMIT = 40  # lbfgs.py:19


@dataclass
class LbfgsResult:
    """lbfgs.py:22-29."""

    x: object
    objective: float
    grad_norm: float
    termination: str
    records: list = field(default_factory=list)
    n_evals: int = 0


def _cubic_minimizer(a, fa, da, b, fb, db):
    """Minimiser of the Hermite cubic on (a, fa, da), (b, fb, db); NaN if none
    (lbfgs.py:32-42)."""
    theta = da + db - 3.0 * (fa - fb) / (a - b)
    disc = theta * theta - da * db
    if disc < 0.0:
        return math.nan
    root = math.sqrt(disc)
    if b < a:
        root = -root
    elif b == a:
        root = 0.0
    den = db - da + 2.0 * root
    if den == 0.0:
        return math.nan
    return b - (b - a) * (db + root - theta) / den


def strong_wolfe(probe, f0, slope0, alpha0, c1, c2):
    """Bracketing + zoom strong-Wolfe search (lbfgs.py:64-99).

    probe(alpha) -> (f, slope) evaluates the objective on the ray (the caller
    keeps the gradient of the most recent probe, which is the accepted one on
    success).  Returns (alpha, f) or None when no acceptable step is found.
    """

    def zoom(lo, f_lo, s_lo, hi, f_hi, s_hi):
        for _ in range(ZOOM_LIMIT):
            left, right = (lo, hi) if lo <= hi else (hi, lo)
            width = right - left
            if width <= 1e-16 * max(1.0, abs(lo)):  # lbfgs.py:71-72
                return None
            trial = _cubic_minimizer(lo, f_lo, s_lo, hi, f_hi, s_hi)
            if not math.isfinite(trial) or trial <= left + 0.1 * width or \
                    trial >= right - 0.1 * width:
                trial = 0.5 * (left + right)  # safeguard (lbfgs.py:74-75)
            f, s = probe(trial)
            if f > f0 + c1 * trial * slope0 or f >= f_lo:
                hi, f_hi, s_hi = trial, f, s
            else:
                if abs(s) <= -c2 * slope0:
                    return trial, f
                if s * (hi - lo) >= 0.0:
                    hi, f_hi, s_hi = lo, f_lo, s_lo
                lo, f_lo, s_lo = trial, f, s
        return None

    prev_a, prev_f, prev_s = 0.0, f0, slope0
    a = alpha0
    for i in range(BRACKET_LIMIT):
        f, s = probe(a)
        if f > f0 + c1 * a * slope0 or (i > 0 and f >= prev_f):
            return zoom(prev_a, prev_f, prev_s, a, f, s)
        if abs(s) <= -c2 * slope0:
            return a, f
        if s >= 0.0:
            return zoom(a, f, s, prev_a, prev_f, prev_s)
        prev_a, prev_f, prev_s = a, f, s
        a *= 2.0
    return None


class _ProbeBudget(Exception):
    """An fp32 line search of the mixed solver ran out of probes."""


# mixed precision: probes one fp32 line search may spend before it is treated
# as failed (the fp32 noise floor) and the solver switches to fp64.  A failed
# search leaves the iterate where it was, so the cap only saves evaluations
# (a zoom at the fp32 floor otherwise runs ~40 probes until its interval
# collapses); the fp64 phase then runs the reference's search unchanged.
FP32_PROBE_CAP = 10

# fp64 searches: after this many probes of one search the space stores the ray
# (space.line_setup: R0, D1, D2 with R(a) = R0 - a D1 - a^2 D2) and answers
# the remaining probes from it at a fraction of an evaluation (no rank-k
# products, no gradient); the accepted point is re-evaluated in full.  Most
# searches accept their first probe and never get here; the long ones (the
# final search that ends in line_search_failed runs ~30 probes) do.  None
# disables.
LINE_PROBES_AFTER = 3


def _check_wolfe(c1, c2, memory):
    if not 0.0 < c1 < c2 < 1.0:
        raise ValueError(f"need 0 < c1 < c2 < 1, got c1={c1}, c2={c2}")
    if memory < 1:
        raise ValueError(f"memory must be >= 1, got {memory}")


def minimize_lbfgs(fun, x0, memory=10, grad_tol=1e-9, max_iter=500, c1=1e-4, c2=0.9,
                   iter_hook=None, timer=None):
    """Minimise fun(x) -> (value, gradient) from x0 (lbfgs.py:102-194).

    Plug-in API for arbitrary host callables.  The SPCP solve itself runs the
    device-resident `DeviceLbfgs` through `solver.lbfgs_minimize`.
    """
    _check_wolfe(c1, c2, memory)
    timer = timer or WorkTimer()
    x = np.array(x0, dtype=np.float64, copy=True)
    f, g = fun(x)
    g = np.asarray(g, dtype=np.float64)
    evals = 1
    gnorm = float(np.linalg.norm(g))
    target = grad_tol * max(1.0, gnorm)
    trace = []

    def log(it):
        timer.pause()
        extra = iter_hook(it, x) if iter_hook is not None else None
        trace.append(IterationRecord(it, float(f), gnorm, timer.elapsed(), dict(extra or {})))
        timer.resume()

    log(0)
    if gnorm <= target:
        return LbfgsResult(x, float(f), gnorm, "converged", trace, evals)
    pairs = deque(maxlen=int(memory))
    reason = "max_iter"
    for it in range(1, int(max_iter) + 1):
        q = g.copy()
        alphas = []
        for s_v, y_v, rho in reversed(pairs):
            a = rho * (s_v @ q)
            alphas.append(a)
            q -= a * y_v
        if pairs:
            s_n, y_n, _ = pairs[-1]
            q *= (s_n @ y_n) / (y_n @ y_n)
        for (s_v, y_v, rho), a in zip(pairs, reversed(alphas)):
            q += (a - rho * (y_v @ q)) * s_v
        d = -q
        slope = float(d @ g)
        if slope >= 0.0:  # lbfgs.py:165-171
            pairs.clear()
            d = -g
            slope = -(gnorm ** 2)
        a0 = 1.0 if pairs else min(1.0, 1.0 / max(gnorm, 1e-12))
        last = {}

        def probe(alpha, x=x, d=d):
            fv, gv = fun(x + alpha * d)
            gv = np.asarray(gv, dtype=np.float64)
            last["g"] = gv
            last["n"] = last.get("n", 0) + 1
            if not np.isfinite(fv):
                fv = math.inf
            return fv, float(gv @ d)

        hit = strong_wolfe(probe, f, slope, a0, c1, c2)
        evals += last.get("n", 0)
        if hit is None:
            reason = "line_search_failed"
            break
        alpha, f_new = hit
        g_new = last["g"]
        s_v = alpha * d
        y_v = g_new - g
        sy = float(s_v @ y_v)
        if sy > 1e-12 * float(np.linalg.norm(s_v)) * float(np.linalg.norm(y_v)):
            pairs.append((s_v, y_v, 1.0 / sy))
        x = x + s_v
        f, g = f_new, g_new
        gnorm = float(np.linalg.norm(g))
        log(it)
        if gnorm <= target:
            reason = "converged"
            break
    return LbfgsResult(x, float(f), gnorm, reason, trace, evals)


# ---------------------------------------------------------------------------
# device-resident driver
# ---------------------------------------------------------------------------


class DeviceLbfgs:
    """L-BFGS over device vectors for the split objective.

    space: object with
      length, empty(), eval(z, d, alpha, g_out, precision) -> (f, g.d, |g|^2),
      gram(A, B) -> host dots, lincomb(coefs, vecs, out), on_switch(precision)
    The iteration is the reference's (lbfgs.py:102-194); `precision` "mixed"
    runs fp32 evaluations until the gradient reaches `switch_tol` relative
    (or an fp32 line search stalls at the fp32 noise floor) and then finishes
    in fp64 so the termination test is the reference's.
    """

    def __init__(self, space, memory=10, grad_tol=1e-8, max_iter=500, c1=1e-4, c2=0.9,
                 precision="fp64", switch_tol=1e-5, iter_hook=None, timer=None):
        _check_wolfe(c1, c2, memory)
        self.sp = space
        self.memory = int(memory)
        self.grad_tol = grad_tol
        self.max_iter = int(max_iter)
        self.c1, self.c2 = c1, c2
        self.precision = precision
        self.cur = "fp32" if precision in ("fp32", "mixed") else "fp64"
        self.switch_tol = switch_tol
        self.hook = iter_hook
        self.timer = timer or WorkTimer()
        n = space.length
        slots = self.memory + 1
        self.S = [space.empty() for _ in range(slots)]
        self.Y = [space.empty() for _ in range(slots)]
        self.order = []  # history slots, oldest -> newest
        self.rho = {}
        self.sy = {}  # (i, j) -> s_i . y_j
        self.yy = {}  # (i, j) -> y_i . y_j (symmetric, both keys stored)
        self.sg = {}  # i -> s_i . g
        self.yg = {}  # i -> y_i . g
        self.d = space.empty()
        self.g = space.empty()
        self.g_new = space.empty()
        self.n = n
        self.switched_at = None

    # ------------------------------------------------------------ helpers
    def _free_slot(self):
        used = set(self.order)
        for s in range(self.memory + 1):
            if s not in used:
                return s
        raise RuntimeError("no free history slot")

    def _clear(self):
        self.order.clear()
        self.rho.clear()
        self.sy.clear()
        self.yy.clear()
        self.sg.clear()
        self.yg.clear()

    def _refresh_g_dots(self):
        if not self.order:
            return
        vecs = [self.S[i] for i in self.order] + [self.Y[i] for i in self.order]
        dots = self.sp.gram(vecs, [self.g])[:, 0]
        h = len(self.order)
        for t, i in enumerate(self.order):
            self.sg[i] = dots[t]
            self.yg[i] = dots[h + t]

    def _direction(self, gg):
        """d = -H g via the dot-product form of the two-loop recursion;
        returns d . g."""
        if not self.order:
            self.sp.lincomb([-1.0], [self.g], self.d)
            return -gg
        hist = self.order
        a = {}
        for idx in range(len(hist) - 1, -1, -1):  # newest -> oldest
            i = hist[idx]
            acc = self.sg[i]
            for j in hist[idx + 1:]:
                acc -= a[j] * self.sy[(i, j)]
            a[i] = self.rho[i] * acc
        newest = hist[-1]
        gamma = self.sy[(newest, newest)] / self.yy[(newest, newest)]
        b = {}
        for idx, i in enumerate(hist):  # oldest -> newest
            yq0 = self.yg[i] - sum(a[j] * self.yy[(i, j)] for j in hist)
            acc = gamma * yq0
            for j in hist[:idx]:
                acc += (a[j] - b[j]) * self.sy[(j, i)]
            b[i] = self.rho[i] * acc
        coefs = [-gamma] + [gamma * a[j] for j in hist] + [-(a[i] - b[i]) for i in hist]
        vecs = [self.g] + [self.Y[j] for j in hist] + [self.S[i] for i in hist]
        self.sp.lincomb(coefs, vecs, self.d)
        return (-gamma * gg + gamma * sum(a[j] * self.yg[j] for j in hist)
                - sum((a[i] - b[i]) * self.sg[i] for i in hist))

    # ------------------------------------------------------------ driver
    def run(self, x):
        """Minimise from the device vector x (updated in place).  Returns an
        LbfgsResult whose x is the same device vector."""
        self._line_held = False
        try:
            return self._run(x)
        finally:
            if self._line_held:
                self.sp.line_release()

    def _run(self, x):
        sp = self.sp
        evals = 0
        f, _, gg = sp.eval(x, None, 0.0, self.g, self.cur)
        evals += 1
        gnorm = math.sqrt(gg)
        target = self.grad_tol * max(1.0, gnorm)
        switch_level = self.switch_tol * max(1.0, gnorm)
        trace = []

        def log(it):
            self.timer.pause()
            extra = self.hook(it, x) if self.hook is not None else None
            extra = dict(extra or {})
            trace.append(IterationRecord(it, float(f), gnorm, self.timer.elapsed(), extra))
            self.timer.resume()

        def to_fp64():
            nonlocal f, gg, gnorm, evals
            self.cur = "fp64"
            self.switched_at = len(trace) - 1
            f, _, gg = sp.eval(x, None, 0.0, self.g, self.cur)
            evals += 1
            gnorm = math.sqrt(gg)
            self._refresh_g_dots()

        def final():  # may this precision declare convergence?
            return self.precision != "mixed" or self.cur == "fp64"

        log(0)
        if gnorm <= target and final():
            return LbfgsResult(x, float(f), gnorm, "converged", trace, evals)
        if self.precision == "mixed" and gnorm <= max(target, switch_level):
            to_fp64()
            if gnorm <= target:
                return LbfgsResult(x, float(f), gnorm, "converged", trace, evals)
        reason = "max_iter"
        it = 1
        while it <= self.max_iter:
            slope = self._direction(gg)
            if slope >= 0.0:  # lbfgs.py:165-171
                self._clear()
                sp.lincomb([-1.0], [self.g], self.d)
                slope = -(gnorm ** 2)
            a0 = 1.0 if self.order else min(1.0, 1.0 / max(gnorm, 1e-12))
            state = {"n": 0, "gg": 0.0}

            capped = self.precision == "mixed" and self.cur == "fp32"
            use_line = (self.cur == "fp64" and LINE_PROBES_AFTER is not None
                        and hasattr(sp, "line_setup"))
            line = {"tried": False, "on": False, "last": False}

            def probe(alpha):
                if capped and state["n"] >= FP32_PROBE_CAP:
                    raise _ProbeBudget
                if use_line and not line["tried"] and state["n"] >= LINE_PROBES_AFTER:
                    line["tried"] = True
                    line["on"] = bool(sp.line_setup(x, self.d))
                if line["on"]:
                    fv, gd = sp.line_probe(alpha)
                    line["last"] = True
                else:
                    fv, gd, gg_t = sp.eval(x, self.d, alpha, self.g_new, self.cur)
                    state["gg"] = gg_t
                    line["last"] = False
                state["n"] += 1
                if not math.isfinite(fv):
                    fv = math.inf  # lbfgs.py:58-59
                return fv, gd

            try:
                hit = strong_wolfe(probe, f, slope, a0, self.c1, self.c2)
            except _ProbeBudget:
                hit = None
            except BaseException:
                if line["on"]:
                    sp.line_release()
                raise
            if line["on"]:
                # the next long search reuses the stored-ray workspace; it is
                # freed when the run ends
                self._line_held = True
            evals += state["n"]
            if hit is not None and line["last"]:
                # accepted on a stored-ray probe: the full evaluation there gives
                # the gradient (and the objective the iteration carries on with)
                fv, _, state["gg"] = sp.eval(x, self.d, hit[0], self.g_new, self.cur)
                evals += 1
                hit = (hit[0], fv)
            if hit is None:
                if self.precision == "mixed" and self.cur == "fp32":
                    to_fp64()  # the fp32 noise floor, not the reference's floor: retry
                    if gnorm <= target:
                        reason = "converged"
                        break
                    continue
                reason = "line_search_failed"
                break
            alpha, f_new = hit
            gg_new = state["gg"]
            # s = alpha d, y = g_new - g into a free slot; then x += s
            slot = self._free_slot()
            s_v, y_v = self.S[slot], self.Y[slot]
            sp.lincomb([alpha], [self.d], s_v)
            sp.lincomb([1.0, -1.0], [self.g_new, self.g], y_v)
            sp.lincomb([1.0, 1.0], [x, s_v], x)
            hist = list(self.order)
            vecs = [self.S[i] for i in hist] + [self.Y[i] for i in hist] + [s_v, y_v]
            dots = sp.gram(vecs, [s_v, y_v, self.g_new])
            h = len(hist)
            sy = dots[2 * h, 1]
            ss = dots[2 * h, 0]
            yyn = dots[2 * h + 1, 1]
            keep = sy > 1e-12 * math.sqrt(max(ss, 0.0)) * math.sqrt(max(yyn, 0.0))
            # next-direction dots against g_new
            for t, i in enumerate(hist):
                self.sg[i] = dots[t, 2]
                self.yg[i] = dots[h + t, 2]
            if keep:
                for t, i in enumerate(hist):
                    self.sy[(i, slot)] = dots[t, 1]          # s_i . y_new
                    self.sy[(slot, i)] = dots[h + t, 0]      # y_i . s_new
                    self.yy[(i, slot)] = self.yy[(slot, i)] = dots[h + t, 1]
                self.sy[(slot, slot)] = sy
                self.yy[(slot, slot)] = yyn
                self.sg[slot] = dots[2 * h, 2]
                self.yg[slot] = dots[2 * h + 1, 2]
                self.rho[slot] = 1.0 / sy
                self.order.append(slot)
                if len(self.order) > self.memory:
                    old = self.order.pop(0)
                    for key in [k for k in self.sy if old in k]:
                        del self.sy[key]
                    for key in [k for k in self.yy if old in k]:
                        del self.yy[key]
                    self.rho.pop(old, None)
                    self.sg.pop(old, None)
                    self.yg.pop(old, None)
            self.g, self.g_new = self.g_new, self.g
            f, gg = f_new, gg_new
            gnorm = math.sqrt(gg)
            log(it)
            if gnorm <= target and final():
                reason = "converged"
                break
            if not final() and gnorm <= max(target, switch_level):
                to_fp64()
                if gnorm <= target:
                    reason = "converged"
                    break
            it += 1
        return LbfgsResult(x, float(f), gnorm, reason, trace, evals)
