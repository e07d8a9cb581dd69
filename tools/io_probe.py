"""Throughput of the SLRM file paths at the C2 shape (20000 x 20000 float64,
3.2 GB on disk): disk -> HBM ingest (`read_matrix(..., device=)`, fp32 and
fp64), HBM -> disk (`write_matrix` of a CUDA tensor) and the decomposition
writer (L and S materialised on the device, `write_decomposition`), next to
the reference's host path for the same file (numpy read + finite check, then
the upload the host path needs).  The file is written once and read back
warm (page cache), so these are host-memory/PCIe figures, not disk figures.

    python tools/io_probe.py [--m 20000 --n 20000 --dir /tmp]  -> one JSON line
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=20000)
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--dir", default="/tmp")
    args = ap.parse_args()
    import torch

    import paper_1702_02241_b200 as api
    from paper_1702_02241_b200.matrixio import read_matrix, write_decomposition, write_matrix
    from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse_device

    m, n = args.m, args.n
    nbytes = m * n * 8
    path = os.path.join(args.dir, "io_probe_x.bin")
    x = gen_low_rank_plus_sparse_device(m, n, 20, 0.05, 1e-3, seed=0, dtype="float64")
    res = {"shape": [m, n], "file_bytes": nbytes + 24}

    def timed(fn, reps=2):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return best, out

    dt, _ = timed(lambda: write_matrix(x, path), reps=1)
    res["write_device_GBps"] = nbytes / dt / 1e9
    dt, t32 = timed(lambda: read_matrix(path, device="cuda", dtype=torch.float32))
    res["read_device_f32_GBps"] = nbytes / dt / 1e9
    ok32 = bool(torch.equal(t32, x.float()))
    del t32
    dt, t64 = timed(lambda: read_matrix(path, device="cuda"))
    res["read_device_f64_GBps"] = nbytes / dt / 1e9
    ok64 = bool(torch.equal(t64, x))
    del t64

    def host_path():
        a = read_matrix(path)  # the reference's read: numpy + isfinite
        return torch.from_numpy(a).to("cuda", non_blocking=False)

    dt, th = timed(host_path, reps=1)
    res["read_host_then_upload_GBps"] = nbytes / dt / 1e9
    del th
    res["bitexact"] = ok32 and ok64

    spec = api.ProblemSpec(x=x, lambda_l=40.0, lambda_s=0.1)
    rep = api.solve_split_spcp(spec, 20, api.SolverConfig(max_iter=5))
    lp, sp = os.path.join(args.dir, "io_probe_l.bin"), os.path.join(args.dir, "io_probe_s.bin")
    dt, nnz = timed(lambda: write_decomposition(rep, lp, sp), reps=1)
    res["write_decomposition_GBps"] = 2 * nbytes / dt / 1e9
    res["write_decomposition_s"] = dt
    res["nnz_s"] = nnz
    for p in (path, lp, sp):
        os.unlink(p)
    res["nproc"] = os.cpu_count()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
