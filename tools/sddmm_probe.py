"""Sparse-observation path vs the dense tensor-core pass on the C4 shape
(50000 x 10000, k = 30) across observed fractions: per-evaluation step time
(stream-ordered, CUDA events) for both paths, fp32 and fp64.  Sets the
density threshold of the automatic choice (spcp_api.cu kSddmmDensity).
python tools/sddmm_probe.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200._lib import SPCP_F32, SPCP_F64  # noqa
from paper_1702_02241_b200.device import DeviceProblem  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

m, n, k, rank = 50000, 10000, 30, 30
x = gen_low_rank_plus_sparse_device(m, n, rank, 0.05, 1e-3, seed=0)
z = torch.randn((m + n) * k, dtype=torch.float64, device="cuda") * np.sqrt(rank / k)
g = torch.empty_like(z)
out = torch.empty(8, dtype=torch.float64, device="cuda")


def timed(dp, code, steps):
    for _ in range(3):
        dp.eval_async(k, code, z, None, 0.0, g, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dp.stream)
    for _ in range(steps):
        dp.eval_async(k, code, z, None, 0.0, g, out)
    e1.record(dp.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for obs in (0.01, 0.03, 0.05, 0.1, 0.15, 0.2, 0.3):
    mask = np.random.default_rng(1).random((m, n)) < obs
    row = [f"obs {obs:4.2f}"]
    for path in ("sparse", "dense"):
        dp = DeviceProblem(x, 20.0, 0.1, mask=mask, store=("f32", path))
        t32 = timed(dp, SPCP_F32, 20)
        t64 = timed(dp, SPCP_F64, 3)
        row.append(f"{path}: fp32 {t32:7.3f} ms fp64 {t64:8.3f} ms")
        del dp
        torch.cuda.empty_cache()
    print("  ".join(row), flush=True)
