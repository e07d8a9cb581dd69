"""Per-evaluation time of the fused fp32 path on every BASELINE config shape
(device-resident, stream-ordered evals, CUDA events), with B_alg-based GB/s.
python tools/configs_probe.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200._lib import SPCP_F32  # noqa
from paper_1702_02241_b200.device import DeviceProblem  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

CONFIGS = [  # name, m, n, k, rank, lambda_L, observed fraction
    ("C1 1000x1000 k=10", 1000, 1000, 10, 10, 10.0, None),
    ("C2 20000x20000 k=20", 20000, 20000, 20, 20, 40.0, None),
    ("C3 110592x2000 k=5", 110592, 2000, 5, 3, 30.0, None),
    ("C3 110592x2000 k=3", 110592, 2000, 3, 3, 30.0, None),
    ("C4 50000x10000 k=30 30% mask", 50000, 10000, 30, 30, 20.0, 0.3),
    ("C5/8 200000x2500 k=50 (per-GPU shard at 8 GPUs)", 200000, 2500, 50, 50, 100.0, None),
]
for name, m, n, k, rank, ll, obs in CONFIGS:
    x = gen_low_rank_plus_sparse_device(m, n, rank, 0.05, 1e-3, seed=0)
    mask = None if obs is None else (np.random.default_rng(1).random((m, n)) < obs)
    dp = DeviceProblem(x, ll, 0.1, mask=mask, store=("f32",))
    del x
    z = torch.randn((m + n) * k, dtype=torch.float64, device="cuda") * np.sqrt(rank / k)
    dz = torch.randn_like(z) * 1e-3
    g = torch.empty_like(z)
    out = torch.empty(8, dtype=torch.float64, device="cuda")
    for i in range(3):
        dp.eval_async(k, SPCP_F32, z, dz, 1e-3, g, out)
    torch.cuda.synchronize()
    dp.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 50
    e0.record(dp.stream)
    for i in range(steps):
        dp.eval_async(k, SPCP_F32, z, dz, 1e-3 * (i + 1), g, out)
    e1.record(dp.stream)
    torch.cuda.synchronize()
    k_ms, k_n, _ = dp.prof_read()
    dp.prof_enable(False)
    step = e0.elapsed_time(e1) / steps
    kern = k_ms / max(k_n, 1)
    b_alg = 4 * m * n + (((m * n + 7) // 8) if mask is not None else 0) + 8 * (m + n) * k
    print(f"{name:50s} step {step:7.3f} ms  kernel {kern:7.3f} ms  {b_alg / kern / 1e6:7.0f} GB/s"
          f"  ({1e3 / step:8.0f} evals/s)", flush=True)
    del dp
    torch.cuda.empty_cache()
