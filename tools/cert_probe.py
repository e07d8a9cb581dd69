"""C2 certificate breakdown: solve, then certificate with timing of its parts
(subspace iterations, apply passes).  python tools/cert_probe.py [tol]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200 import ProblemSpec, SolverConfig, certificate, solve_split_spcp  # noqa
import importlib  # noqa
cmod = importlib.import_module("paper_1702_02241_b200.certificate")  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

x = gen_low_rank_plus_sparse_device(20000, 20000, 20, 0.05, 1e-3, seed=0)
spec = ProblemSpec(x=x, lambda_l=40.0, lambda_s=0.1)
spec.device("mixed")
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = solve_split_spcp(spec, 20, SolverConfig())
t1 = time.perf_counter()
dp = spec.device("fp64")
z = torch.from_numpy(np.ascontiguousarray(rep.factors.flatten())).to(dp.device)
w = torch.randn(20000, 16, dtype=torch.float64, device=dp.device)
for _ in range(2):
    dp.apply(20, z, w_right=w)
torch.cuda.synchronize()
ta = time.perf_counter()
for _ in range(5):
    dp.apply(20, z, w_right=w)
torch.cuda.synchronize()
tb = time.perf_counter()
print(f"apply (b=16, fp64) {1e3 * (tb - ta) / 5:.2f} ms")
for tol in [float(a) for a in sys.argv[1:]] or [1e-9]:
    cmod._SUBSPACE_TOL = tol
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cert = certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"tol {tol:g}: solve {t1 - t0:.3f}s certificate {t3 - t2:.3f}s e_norm {cert.e_norm:.6e} "
          f"gap {cert.gap_bound:.6e} info {cert.info}")
