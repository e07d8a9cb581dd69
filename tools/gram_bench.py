"""L-BFGS Gram pass (spcp_vec_gram) timing: 22 history vectors x 3 at the C2 and
C5 iterate lengths.  python tools/gram_bench.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200.device import DeviceProblem  # noqa

x = torch.zeros((256, 256), dtype=torch.float32, device="cuda")
dp = DeviceProblem(x, 1.0, 1.0, store=("f32",))
for name, length in (("c2", 40000 * 20), ("c5", 220000 * 50)):
    a = [torch.randn(length, dtype=torch.float64, device="cuda") for _ in range(22)]
    b = [torch.randn(length, dtype=torch.float64, device="cuda") for _ in range(3)]
    for _ in range(3):
        dp.vec_gram(a, b)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        g = dp.vec_gram(a, b)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    ref = torch.stack(a) @ torch.stack(b).T
    err = float((torch.from_numpy(g).cuda() - ref).abs().max() / ref.abs().max())
    gb = 25 * length * 8 / 1e9
    print(f"{name}: {dt * 1e3:.3f} ms per 22x3 Gram ({gb / dt:.0f} GB/s of vector reads), "
          f"max rel err {err:.1e}", flush=True)
    del a, b
dp.close()
