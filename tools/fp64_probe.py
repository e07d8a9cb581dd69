"""Time the fp64 evaluation (SIMT stream_kernel, the L-BFGS polish) at C2 and
leave it for an ncu capture: python tools/fp64_probe.py [evals]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200._lib import SPCP_F64  # noqa
from paper_1702_02241_b200.device import DeviceProblem  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

n_ev = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m = n = 20000
k = 20
x = gen_low_rank_plus_sparse_device(m, n, 20, 0.05, 1e-3, seed=0)
dp = DeviceProblem(x, 40.0, 0.1, store=("f32",))
g = torch.Generator(device="cuda")
g.manual_seed(5)
z = torch.randn((m + n) * k, generator=g, device="cuda", dtype=torch.float64) * np.sqrt(2.0)
out = torch.empty_like(z)
dp.eval(k, SPCP_F64, z, None, 0.0, out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n_ev):
    dp.eval(k, SPCP_F64, z, None, 0.0, out)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / n_ev
print(f"fp64 eval at C2: {dt * 1e3:.3f} ms ({6 * m * n * k / dt / 1e12:.2f} TFLOP/s of 6mnk)")
