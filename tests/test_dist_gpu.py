"""Column-sharded solve + certificate on the GPU kernels:
world_size 2 over gloo with both ranks on cuda:0 (one GPU in this
environment; the NCCL transport is the same torch.distributed calls).
solve_split_spcp_sharded and certificate_sharded must reproduce the
single-GPU solve_split_spcp / certificate (solver.py:255-324,
certificate.py:77-141) on the same X: objective, L (k-space), the
certificate terms and verdict, identical on both ranks."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LAM_S = 0.2
CASES = {  # precision: (m, n, rank, k, lambda_L); mixed needs m n >= MIXED_MIN_ELEMS
    "fp64": (420, 330, 5, 5, 3.0),
    "mixed": (2600, 1700, 8, 8, 0.3 * np.sqrt(1700)),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(precision):
    from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse

    m, n, rank, _, _ = CASES[precision]
    x, _, _ = gen_low_rank_plus_sparse(m, n, rank, 0.05, 1e-3, seed=7)
    return x.astype(np.float32).astype(np.float64)


def _worker(rank, world, port, precision, out_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    from paper_1702_02241_b200 import SolverConfig
    from paper_1702_02241_b200.dist import certificate_sharded, shard_bounds, \
        solve_split_spcp_sharded

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = _problem(precision)
        _, n, _, k, lam_l = CASES[precision]
        c0, nl = shard_bounds(n, world, rank)
        rep = solve_split_spcp_sharded(np.ascontiguousarray(x[:, c0:c0 + nl]), lam_l, LAM_S, k,
                                       n, c0, SolverConfig(precision=precision))
        cert = certificate_sharded(rep)
        out_q.put((rank, rep.objective, rep.termination, rep.factors.u, rep.factors.v, c0,
                   cert.e_norm, cert.terms, cert.r, cert.gap_bound,
                   rep.extra["allreduce_calls"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_sharded_solve_and_certificate_match_single_gpu(precision):
    import torch.multiprocessing as mp

    from paper_1702_02241_b200 import ProblemSpec, SolverConfig, certificate, solve_split_spcp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, precision, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x = _problem(precision)
    _, _, _, k, lam_l = CASES[precision]
    spec = ProblemSpec(x=x, lambda_l=lam_l, lambda_s=LAM_S)
    ref = solve_split_spcp(spec, k, SolverConfig(precision=precision))
    rc = certificate(ref.factors, spec, f_bound_hint=ref.best_objective)
    u = res[0][3]
    v = np.concatenate([r[4] for r in res])
    lr = ref.factors.u @ ref.factors.v.T
    ls = u @ v.T
    tol = 1e-9 if precision == "fp64" else 1e-7
    for r in res:
        assert r[1] == pytest.approx(ref.objective, rel=tol)
        assert r[8] == rc.r
        assert (r[9] > 1e-2 * max(1.0, abs(r[1]))) == (rc.gap_bound > 1e-2 * max(1.0, abs(
            ref.objective)))
        assert r[10] > 0
    assert np.linalg.norm(ls - lr) <= 1e-4 * np.linalg.norm(lr)
    # both ranks hold the same replicated U and the same report
    np.testing.assert_array_equal(res[0][3], res[1][3])
    assert res[0][6] == res[1][6] and res[0][7] == res[1][7]
    # e_norm: equal where it measures distance, both at the noise floor otherwise
    # (there it depends on where each L-BFGS run stopped)
    assert abs(res[0][6] - rc.e_norm) <= 1e-3 * rc.e_norm + 1e-4 * lam_l
