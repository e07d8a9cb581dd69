"""Time the fp64 evaluation (f64_stream_kernel, the L-BFGS polish) at C2 (k=20)
and on the C5 per-GPU shard (200000 x 2500, k=50):
python tools/fp64_probe.py [evals]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200._lib import SPCP_F64  # noqa
from paper_1702_02241_b200.device import DeviceProblem  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

n_ev = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for m, n, k, rank in ((20000, 20000, 20, 20), (200000, 2500, 50, 50)):
    x = gen_low_rank_plus_sparse_device(m, n, rank, 0.05, 1e-3, seed=0)
    dp = DeviceProblem(x, 40.0, 0.1, store=("f32",))
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    z = torch.randn((m + n) * k, generator=g, device="cuda", dtype=torch.float64) * np.sqrt(2.0)
    out = torch.empty_like(z)
    dp.eval(k, SPCP_F64, z, None, 0.0, out)
    torch.cuda.synchronize()
    dp.prof_enable(True)
    t0 = time.perf_counter()
    for _ in range(n_ev):
        dp.eval(k, SPCP_F64, z, None, 0.0, out)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n_ev
    kms, cnt, _ = dp.prof_read()
    print(f"fp64 eval {m}x{n} k={k}: {dt * 1e3:.3f} ms per eval, kernel "
          f"{kms / max(cnt, 1):.3f} ms ({6 * m * n * k / (kms / max(cnt, 1) * 1e-3) / 1e12:.2f} "
          f"TFLOP/s of 6mnk)", flush=True)
    dp.close()
    del x, dp
    torch.cuda.empty_cache()
