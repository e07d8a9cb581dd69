"""Per-rank compute of the C5 strong-scaling workload (200000 x 20000, k = 50)
at N = 1, 2, 4, 8 column shards, measured on ONE B200: the fp32 and fp64
evaluation time of one rank's shard (200000 x 20000/N, the same columns the
sharded run generates).  What an N-GPU run adds on top is the per-evaluation
all-reduce of G_p V_p (200000 x 50 fp32 = 40 MB) and the host-side L-BFGS
logic; this probe does not model them.
python tools/c5_shard_probe.py"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200._lib import SPCP_F32, SPCP_F64  # noqa
from paper_1702_02241_b200.device import DeviceProblem  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

m, n, k = 200000, 20000, 50


def timed(dp, code, z, g, out, steps):
    for _ in range(2):
        dp.eval_async(k, code, z, None, 0.0, g, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dp.stream)
    for _ in range(steps):
        dp.eval_async(k, code, z, None, 0.0, g, out)
    e1.record(dp.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


res = []
for world in (1, 2, 4, 8):
    nl = n // world
    x = gen_low_rank_plus_sparse_device(m, nl, 50, 0.05, 1e-3, seed=0, col0=0, n_total=n)
    dp = DeviceProblem(x, 100.0, 0.1, store=("f32",), n_total=n, col0=0)
    del x
    torch.cuda.empty_cache()
    z = torch.randn((m + nl) * k, dtype=torch.float64, device="cuda")
    g = torch.empty_like(z)
    out = torch.empty(8, dtype=torch.float64, device="cuda")
    t32 = timed(dp, SPCP_F32, z, g, out, 20)
    t64 = timed(dp, SPCP_F64, z, g, out, 5)
    res.append({"n_gpus": world, "shard": f"{m}x{nl}", "fp32_ms": t32, "fp64_ms": t64})
    print(json.dumps(res[-1]), flush=True)
    dp.close()
    del dp, z, g
    torch.cuda.empty_cache()
base = res[0]
for r in res:
    r["fp32_speedup"] = base["fp32_ms"] / r["fp32_ms"]
    r["fp64_speedup"] = base["fp64_ms"] / r["fp64_ms"]
print(json.dumps(res))
