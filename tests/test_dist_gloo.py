"""Column-sharded mode on the CPU with torch.distributed/gloo,
world_size 2.  Each rank owns a column shard; ShardedSpace's partial/all-reduce
/finish evaluation and its split U/V inner products must reproduce the
unsharded objective, gradient and L-BFGS trajectory.  The shard arithmetic is
the oracle's (tests/fakes.py); the GPU kernels behind the same calls are
checked in the -m gpu tests."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q, line=False):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist

    from fakes import NumpyLineShardProblem, NumpyShardProblem
    from oracle import spcp_oracle as orc
    from paper_1702_02241_b200.dist import ShardedSpace, shard_bounds
    import paper_1702_02241_b200.lbfgs as lb
    from paper_1702_02241_b200.lbfgs import DeviceLbfgs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, k, lam_l, lam_s = 60, 45, 4, 1.0, 0.3
        x, _, _ = orc.gen_low_rank_plus_sparse(m, n, 4, 0.1, 1e-3, seed=21)
        c0, nl = shard_bounds(n, world, rank)
        cls = NumpyLineShardProblem if line else NumpyShardProblem
        if line:  # every fp64 probe from the stored ray
            lb.LINE_PROBES_AFTER = 0
        dp = cls(np.ascontiguousarray(x[:, c0:c0 + nl]), lam_l, lam_s)
        sp = ShardedSpace(dp, k, m, nl, comm_device=torch.device("cpu"))
        u0, v0 = orc.init_factors(x, k, strategy="rsvd", seed=0)
        z = torch.from_numpy(np.concatenate([u0.ravel(), v0[c0:c0 + nl].ravel()]))
        g = sp.empty()
        f, gd, gg = sp.eval(z, None, 0.0, g, "fp64")
        eng = DeviceLbfgs(sp, grad_tol=1e-9, max_iter=400, precision="fp64")
        res = eng.run(z)
        if line:
            assert dp.setups > 0 and dp.releases == 1
        out_q.put((rank, f, gg, g.numpy().copy(), [r.objective for r in res.records],
                   res.termination, c0, nl))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("line", [False, True])
def test_sharded_eval_and_lbfgs_match_unsharded(oracle, line):
    """line=True: the fp64 searches answer their probes from each shard's
    stored ray (ShardedSpace.line_probe: replicated U regulariser once)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, line)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    m, n, k, lam_l, lam_s = 60, 45, 4, 1.0, 0.3
    x, _, _ = oracle.gen_low_rank_plus_sparse(m, n, 4, 0.1, 1e-3, seed=21)
    u0, v0 = oracle.init_factors(x, k, strategy="rsvd", seed=0)
    f_ref, gu_ref, gv_ref = oracle.split_objective(u0, v0, x, lam_l, lam_s)
    for rank, f, gg, g, objs, term, c0, nl in res:
        assert f == pytest.approx(f_ref, rel=1e-13)
        assert gg == pytest.approx(float(np.sum(gu_ref ** 2) + np.sum(gv_ref ** 2)), rel=1e-12)
        np.testing.assert_allclose(g[: m * k], gu_ref.ravel(), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(g[m * k:], gv_ref[c0:c0 + nl].ravel(), rtol=1e-12, atol=1e-12)
    # both ranks walk the identical trajectory (replicated U, summed dots)
    assert res[0][4] == res[1][4]
    ref = oracle.minimize_lbfgs(
        oracle.flat_objective(x, lam_l, lam_s, None, m, n, k),
        np.concatenate([u0.ravel(), v0.ravel()]), grad_tol=1e-9, max_iter=400)
    ours = res[0][4]
    cmp = min(15, len(ours), len(ref["records"]))
    np.testing.assert_allclose(ours[:cmp], [r[1] for r in ref["records"]][:cmp], rtol=1e-9)
    assert ours[-1] == pytest.approx(ref["objective"], rel=1e-9)
