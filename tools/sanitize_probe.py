"""A few evaluations of every device path on a small problem, for
compute-sanitizer (memcheck / racecheck / synccheck): fused tcgen05 pass +
reduce (fp32), fp64 SIMT pass, sparse-observation passes, apply products.
compute-sanitizer --tool memcheck python tools/sanitize_probe.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200._lib import SPCP_F32, SPCP_F64  # noqa
from paper_1702_02241_b200.device import DeviceProblem  # noqa

rng = np.random.default_rng(0)
m, n, k = 700, 530, 20
x = (rng.standard_normal((m, 20)) @ rng.standard_normal((20, n))).astype(np.float32)
mask = rng.random((m, n)) < 0.08
z = torch.from_numpy(rng.standard_normal((m + n) * k)).cuda()
g = torch.empty_like(z)
for store, msk in ((("f32",), None), (("f32",), mask), (("f32", "sparse"), mask)):
    dp = DeviceProblem(x, 2.0, 0.1, mask=msk, store=store)
    for code in (SPCP_F32, SPCP_F64):
        out = dp.eval(k, code, z, None, 0.0, g)
        print(store, msk is not None, code, out[0], flush=True)
    w = torch.from_numpy(rng.standard_normal((n, 8))).cuda()
    left, _ = dp.apply(k, z, w_right=w)
    torch.cuda.synchronize()
    dp.close()
print("ok")
