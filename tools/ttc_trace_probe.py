"""Where the time to certificate goes: every evaluation of the C2 and the
single-GPU C5 solve (precision, line-search probe or not, wall time), the
initialisation and the certificate.
python tools/ttc_trace_probe.py [c2|c5]..."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200 import ProblemSpec, SolverConfig, certificate, solve_split_spcp  # noqa
from paper_1702_02241_b200 import solver as solver_mod  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

LOG = []
_orig_eval = solver_mod.SplitSpace.eval


def traced_eval(self, z, d, alpha, g_out, precision):
    t0 = time.perf_counter()
    r = _orig_eval(self, z, d, alpha, g_out, precision)
    LOG.append((precision, d is not None, float(alpha), time.perf_counter() - t0, float(r[0])))
    return r


solver_mod.SplitSpace.eval = traced_eval


def _wrap(name):
    orig = getattr(solver_mod.SplitSpace, name)

    def w(self, *a):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = orig(self, *a)
        torch.cuda.synchronize()
        LOG.append((name, False, float(a[0]) if name == "line_probe" else 0.0,
                    time.perf_counter() - t0, float(r[0]) if name == "line_probe" else 0.0))
        return r
    setattr(solver_mod.SplitSpace, name, w)


for _n in ("line_setup", "line_probe", "line_release"):
    _wrap(_n)
_orig_init = solver_mod.init_factors


def traced_init(*a, **kw):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = _orig_init(*a, **kw)
    torch.cuda.synchronize()
    LOG.append(("init", False, 0.0, time.perf_counter() - t0, 0.0))
    return r


solver_mod.init_factors = traced_init

CASES = {"c2": (20000, 20000, 20, 40.0), "c5": (200000, 20000, 50, 100.0)}
for name in sys.argv[1:] or ["c2", "c5"]:
    m, n, k, lam = CASES[name]
    x = gen_low_rank_plus_sparse_device(m, n, k, 0.05, 1e-3, seed=0)
    spec = ProblemSpec(x=x, lambda_l=lam, lambda_s=0.1)
    spec.device("mixed")
    for rep_i in range(2):
        LOG.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = solve_split_spcp(spec, k, SolverConfig())
        t1 = time.perf_counter()
        cert = certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        summ = {}
        for p, probe, a, dt, f in LOG:
            key = p if p.startswith(("init", "line")) else f"{p}_{'probe' if probe else 'point'}"
            c, s = summ.get(key, (0, 0.0))
            summ[key] = (c + 1, s + dt)
        print(json.dumps({"case": name, "run": rep_i, "solve_s": t1 - t0, "cert_s": t2 - t1,
                          "termination": rep.termination, "iters": len(rep.iterations) - 1,
                          "evals": rep.extra["n_evals"], "switch": rep.extra.get("fp64_switch_iter"),
                          "objective": rep.objective,
                          "by_kind": {kk: [c, round(s, 4)] for kk, (c, s) in summ.items()}}),
              flush=True)
        if rep_i == 1:
            for i, (p, probe, a, dt, f) in enumerate(LOG):
                print(f"  {i:3d} {p:5s} {'probe' if probe else 'point'} alpha={a:.3e} "
                      f"{dt * 1e3:8.2f} ms f={f:.12e}")
    del spec, x
    torch.cuda.empty_cache()
