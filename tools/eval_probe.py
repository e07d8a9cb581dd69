"""C2 per-evaluation time of each precision path (sync API): fp32 tensor-core, fp64 SIMT."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200._lib import SPCP_F32, SPCP_F64  # noqa
from paper_1702_02241_b200.device import DeviceProblem  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa

m = n = 20000
k = 20
x = gen_low_rank_plus_sparse_device(m, n, 20, 0.05, 1e-3, seed=0)
dp = DeviceProblem(x, 40.0, 0.1, store=("f32", "f64"))
z = torch.randn((m + n) * k, dtype=torch.float64, device="cuda") * np.sqrt(2.0)
g = torch.empty_like(z)
for name, dt in (("fp32", SPCP_F32), ("fp64", SPCP_F64)):
    for _ in range(3):
        dp.eval(k, dt, z, None, 0.0, g)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        dp.eval(k, dt, z, None, 0.0, g)
    torch.cuda.synchronize()
    print(f"{name}: {1e3 * (time.perf_counter() - t0) / 20:.3f} ms per synchronous eval")
