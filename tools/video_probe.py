"""Background subtraction at the full C3 shape (384x288 frames x 2000,
BASELINE configs[2]) on the device video generator: solve + certificate
wall time and how well supp(S) recovers the moving objects.

    python tools/video_probe.py [--k 3] [--lambda-l 100] [--lambda-s 0.05]  -> one JSON line
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=3)
    ap.add_argument("--lambda-l", type=float, default=100.0)
    ap.add_argument("--lambda-s", type=float, default=0.05)
    args = ap.parse_args()
    import torch

    import paper_1702_02241_b200 as api

    x, l_ref, fg = api.gen_video_device(seed=0)
    spec = api.ProblemSpec(x=x, lambda_l=args.lambda_l, lambda_s=args.lambda_s)
    spec.device("mixed")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = api.solve_split_spcp(spec, args.k, api.SolverConfig())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    cert = api.certificate(rep.factors, spec, f_bound_hint=rep.best_objective)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s = torch.from_numpy(rep.s).to(x.device)
    l = torch.from_numpy(rep.l).to(x.device)
    moved = (x.double() - l_ref.double()).abs() > 0.1
    s_on = s != 0
    out = {
        "shape": list(x.shape), "k": args.k, "lambda_l": args.lambda_l,
        "lambda_s": args.lambda_s, "solve_s": t1 - t0, "certificate_s": t2 - t1,
        "termination": rep.termination, "iterations": len(rep.iterations) - 1,
        "n_evals": rep.extra["n_evals"], "e_norm": cert.e_norm, "r": cert.r,
        "certified": cert.gap_bound <= 1e-2 * max(1.0, abs(rep.objective)),
        "fg_fraction": fg.float().mean().item(),
        "recall_moved_pixels": s_on[moved].float().mean().item(),
        "false_positive_rate": (s_on & ~fg).float().mean().item(),
        "l_rel_err": ((l - l_ref.double()).norm() / l_ref.double().norm()).item(),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
