"""Time the certificate and a full mixed solve at C2 (device generator X),
several repetitions: python tools/cert_time_probe.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200 import ProblemSpec, SolverConfig, certificate, solve_split_spcp  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

if len(sys.argv) > 1:  # starting block of the certificate's subspace iteration
    import importlib

    importlib.import_module("paper_1702_02241_b200.certificate").SUBSPACE_BLOCK = int(sys.argv[1])
x = gen_low_rank_plus_sparse_device(20000, 20000, 20, 0.05, 1e-3, seed=0)
spec = ProblemSpec(x=x, lambda_l=40.0, lambda_s=0.1)
spec.device("mixed")
for rep_i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = solve_split_spcp(spec, 20, SolverConfig())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    cert = certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"solve {t1 - t0:.4f} s ({rep.extra['n_evals']} evals, {rep.termination}), "
          f"certificate {t2 - t1:.4f} s ({cert.info.get('iters')} passes)", flush=True)
