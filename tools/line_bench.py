"""Stored-ray probe costs at C2 and C5 (csrc/line.cuh): setup with and without
the workspace allocation, one probe, release, next to one fp64 evaluation.
python tools/line_bench.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200._lib import SPCP_F64  # noqa
from paper_1702_02241_b200.device import DeviceProblem  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for name, m, n, k in (("c2", 20000, 20000, 20), ("c5", 200000, 20000, 50)):
    x = gen_low_rank_plus_sparse_device(m, n, k, 0.05, 1e-3, seed=0)
    dp = DeviceProblem(x, 1.0, 0.1, store=("f32",))
    z = torch.randn((m + n) * k, dtype=torch.float64, device="cuda")
    d = 1e-3 * torch.randn_like(z)
    g = torch.empty_like(z)
    ev = [t(lambda: dp.eval(k, SPCP_F64, z, d, 0.5, g)) for _ in range(3)]
    s1 = t(lambda: dp.line_setup(k, z, d))
    s2 = t(lambda: dp.line_setup(k, z, d))
    pr = [t(lambda: dp.line_probe(0.5)) for _ in range(5)]
    rl = t(lambda: dp.line_release())
    print(f"{name}: fp64 eval {min(ev):.2f} ms | setup (alloc) {s1:.2f} ms, setup {s2:.2f} ms | "
          f"probe {min(pr):.2f} ms ({3 * m * n * 8 / min(pr) / 1e6:.0f} GB/s) | release {rl:.2f} ms",
          flush=True)
    dp.close()
    del x, dp, z, d, g
    torch.cuda.empty_cache()
