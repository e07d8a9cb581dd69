"""Time the pieces of the randomized-SVD initialisation (linalg.rand_svd_device)
at C2 (k = 20) and C5 (k = 50): host Gaussian sketch, the X passes, the thin
QRs, the host SVD of the width x n sketch.
python tools/init_probe.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_02241_b200 import ProblemSpec  # noqa
from paper_1702_02241_b200.linalg import device_thin_qr, svd_small  # noqa
from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device  # noqa


def tick(label, t0, acc):
    torch.cuda.synchronize()
    t = time.perf_counter()
    acc.append((label, (t - t0) * 1e3))
    return t


for name, m, n, k in (("c2", 20000, 20000, 20), ("c5", 200000, 20000, 50)):
    x = gen_low_rank_plus_sparse_device(m, n, k, 0.05, 1e-3, seed=0)
    spec = ProblemSpec(x=x, lambda_l=1.0, lambda_s=0.1)
    dp = spec.device("mixed")
    for rep in range(2):
        acc = []
        width = k + 10
        torch.cuda.synchronize()
        t = time.perf_counter()
        omega = np.random.default_rng(0).standard_normal((n, width))
        t = tick("omega host", t, acc)
        om = torch.from_numpy(omega).to(dp.device)
        t = tick("omega h2d", t, acc)
        y, _ = dp.apply(0, None, w_right=om)
        t = tick("apply X om (fp64)", t, acc)
        q, _ = device_thin_qr(dp, y)
        t = tick("thin qr", t, acc)
        _, z = dp.apply(0, None, w_left=q)
        t = tick("apply X^T q (fp64)", t, acc)
        q2, _ = device_thin_qr(dp, z)
        t = tick("thin qr", t, acc)
        y, _ = dp.apply(0, None, w_right=q2)
        t = tick("apply X q2 (fp64)", t, acc)
        q, _ = device_thin_qr(dp, y)
        t = tick("thin qr", t, acc)
        _, bt = dp.apply(0, None, w_left=q)
        t = tick("apply X^T q (fp64)", t, acc)
        bh = bt.cpu().numpy().T
        t = tick("bt d2h", t, acc)
        inner = svd_small(bh)
        t = tick("svd_small host", t, acc)
        u = dp.matmul_small(q, inner.u[:, :k])
        t = tick("matmul_small", t, acc)
        y32, _ = dp.apply(0, None, w_right=om, precision="fp32")
        t = tick("[apply X om fp32]", t, acc)
        print(name, rep, " | ".join(f"{a}: {b:.2f} ms" for a, b in acc), flush=True)
    spec.release_device()
    del x, spec, dp
    torch.cuda.empty_cache()
