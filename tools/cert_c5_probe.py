"""Where the certificate's time goes at C5 (200000 x 20000, k = 50; or c2) on one GPU:
every DeviceProblem product it calls, by kind, plus the total.
python tools/cert_c5_probe.py [c5|c2]"""
import collections
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200 import ProblemSpec, SolverConfig, certificate, solve_split_spcp  # noqa
from paper_1702_02241_b200 import device as devmod  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

STAT = collections.defaultdict(lambda: [0, 0.0])


def wrap(name, keyf):
    orig = getattr(devmod.DeviceProblem, name)

    def w(self, *a, **kw):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = orig(self, *a, **kw)
        torch.cuda.synchronize()
        key = keyf(a, kw)
        STAT[key][0] += 1
        STAT[key][1] += time.perf_counter() - t0
        return r
    setattr(devmod.DeviceProblem, name, w)


def apply_key(a, kw):
    wr = kw.get("w_right", a[2] if len(a) > 2 else None)
    wl = kw.get("w_left", a[3] if len(a) > 3 else None)
    b = (wr if wr is not None else wl).shape[1]
    sides = ("R" if wr is not None else "") + ("L" if wl is not None else "")
    return f"apply k={a[0]} {kw.get('precision', 'fp64')} b={b} {sides}"


wrap("apply", apply_key)
wrap("apply_stored", lambda a, kw: "apply_stored " + ("R" if kw.get("w_right") is not None
                                                       else "L"))
wrap("grad_store", lambda a, kw: "grad_store")
wrap("eval", lambda a, kw: "eval (fp64, t1-t3 route)")
wrap("gram", lambda a, kw: "gram")
wrap("matmul_small", lambda a, kw: "matmul_small")

CASES = {"c5": (200000, 20000, 50, 100.0), "c2": (20000, 20000, 20, 40.0)}
m, n, k, lam = CASES[sys.argv[1] if len(sys.argv) > 1 else "c5"]
x = gen_low_rank_plus_sparse_device(m, n, k, 0.05, 1e-3, seed=0)
spec = ProblemSpec(x=x, lambda_l=lam, lambda_s=0.1)
spec.device("mixed")
rep = solve_split_spcp(spec, k, SolverConfig())
wrap("grad_release", lambda a, kw: "grad_release")
for r in range(3):
    STAT.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cert = certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"certificate {tot * 1e3:.1f} ms  info {cert.info}")
    for key, (c, s) in sorted(STAT.items(), key=lambda kv: -kv[1][1]):
        print(f"   {key:40s} x{c:3d}  {s * 1e3:8.1f} ms")
