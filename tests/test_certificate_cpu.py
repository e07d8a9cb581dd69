"""The certificate's device algorithm (certificate.certificate_core: factor SVD
by CholeskyQR2 / eigenbasis QR, fused D V1 / D^T U1 products, t4 by streaming
block subspace iteration with the power-method bound) run on CPU test doubles
(tests/fakes.py) against the oracle's dense certificate (certificate.py:77-141),
single shard and column-sharded over gloo world_size 2."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from fakes import NumpyCertProblem


def _cert_inputs(oracle, under_rank):
    m, n, lam_l, lam_s = 70, 52, 2.0, 0.3
    x, _, _ = oracle.gen_low_rank_plus_sparse(m, n, 6, 0.1, 1e-3, seed=41)
    k = 3 if under_rank else 8  # k = 8 > rank 6: rank-deficient factors
    res = oracle.solve_split_spcp(x, lam_l, lam_s, k, grad_tol=1e-10, max_iter=3000)
    return x, res["u"], res["v"], lam_l, lam_s, res["objective"]


@pytest.mark.parametrize("under_rank", [False, True])
def test_certificate_core_matches_oracle(oracle, under_rank):
    from paper_1702_02241_b200.certificate import CertOps, certificate_core

    x, u, v, lam_l, lam_s, obj = _cert_inputs(oracle, under_rank)
    m, n = x.shape
    k = u.shape[1]
    dp = NumpyCertProblem(x, lam_l, lam_s)
    z = torch.from_numpy(np.concatenate([u.ravel(), v.ravel()]))
    ours = certificate_core(dp, z, m, n, k, lam_l, 1e-10, dp.f_zero, obj, CertOps(n_total=n))
    ref = oracle.certificate(u, v, x, lam_l, lam_s, f_bound_hint=obj)
    assert ours.r == ref["r"]
    np.testing.assert_allclose(ours.terms[:3], ref["terms"][:3], rtol=1e-8, atol=1e-9)
    if under_rank:
        assert ours.info["n_sigma_over_1"] >= 1 and ours.info["converged"]
        assert ours.terms[3] == pytest.approx(ref["terms"][3], rel=1e-7)
    else:
        assert ours.terms[3] == 0.0 == ref["terms"][3]
        assert ours.info["converged"] and ours.info["sigma_p_max"] < 1.0
    assert ours.e_norm == pytest.approx(ref["e_norm"], rel=1e-7, abs=1e-6)  # noise level when converged
    assert oracle.certificate_warns(ref, obj) == (ours.gap_bound > 1e-2 * max(1.0, abs(obj)))


def test_rank_deficient_factor_qr(oracle):
    """Exactly rank-deficient V (a repeated column): the eigenbasis QR branch
    (no library QR) gives the reference's rank and terms."""
    from paper_1702_02241_b200.certificate import CertOps, certificate_core

    rng = np.random.default_rng(62)
    m, n, k = 12, 9, 4
    x = rng.standard_normal((m, n))
    u = rng.standard_normal((m, k))
    v = rng.standard_normal((n, k))
    v[:, 3] = v[:, 2]
    dp = NumpyCertProblem(x, 1.1, 0.4)
    z = torch.from_numpy(np.concatenate([u.ravel(), v.ravel()]))
    ours = certificate_core(dp, z, m, n, k, 1.1, 1e-10, dp.f_zero, None, CertOps(n_total=n))
    ref = oracle.certificate(u, v, x, 1.1, 0.4)
    assert ours.r == ref["r"] == 3
    np.testing.assert_allclose([ours.e_norm, *ours.terms], [ref["e_norm"], *ref["terms"]],
                               rtol=1e-8, atol=1e-10)


def test_power_bound_iterations():
    from paper_1702_02241_b200.certificate import _power_bound_iters

    from paper_1702_02241_b200.certificate import _TIERS

    # 0.824 sqrt(n) (1 - eps)^(q - 3/2) <= fail * eps / tiers at the returned q
    for n in (10, 1000, 20000, 200000):
        for ome, _ in _TIERS:
            q = _power_bound_iters(n, ome, 1e-6)
            eps = 1.0 - ome
            assert 0.824 * np.sqrt(n) * ome ** (q - 1.5) <= 1e-6 * eps / len(_TIERS)
            assert 0.824 * np.sqrt(n) * ome ** (q - 2.5) > 1e-6 * eps / len(_TIERS)
    assert [_power_bound_iters(20000, ome, 1e-6) for ome, _ in _TIERS] == [7, 9, 17, 32]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, under_rank, out_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    from fakes import NumpyCertProblem
    from oracle import spcp_oracle as orc
    from paper_1702_02241_b200.dist import certificate_sharded, shard_bounds
    from paper_1702_02241_b200.report import SolveReport

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, u, v, lam_l, lam_s, obj = _cert_inputs(orc, under_rank)
        m, n = x.shape
        k = u.shape[1]
        c0, nl = shard_bounds(n, world, rank)
        dp = NumpyCertProblem(np.ascontiguousarray(x[:, c0:c0 + nl]), lam_l, lam_s)
        z = torch.from_numpy(np.concatenate([u.ravel(), v[c0:c0 + nl].ravel()]))
        rep = SolveReport(solver="split", termination="converged", iterations=[], l=None,
                          s=None, objective=obj, factors=None,
                          extra={"n_total": n, "col0": c0})
        rep.device_state = (dp, k, z)
        cert = certificate_sharded(rep)
        out_q.put((rank, cert.e_norm, cert.terms, cert.r, cert.gap_bound, cert.f_bound))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("under_rank", [False, True])
def test_certificate_sharded_gloo(oracle, under_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, under_rank, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, u, v, lam_l, lam_s, obj = _cert_inputs(oracle, under_rank)
    ref = oracle.certificate(u, v, x, lam_l, lam_s, f_bound_hint=obj)
    for _, e_norm, terms, r, gap, fb in res:
        assert r == ref["r"]
        np.testing.assert_allclose(terms[:3], ref["terms"][:3], rtol=1e-8, atol=1e-9)
        assert terms[3] == pytest.approx(ref["terms"][3], rel=1e-7, abs=1e-12)
        assert e_norm == pytest.approx(ref["e_norm"], rel=1e-7, abs=1e-6)
        assert fb == pytest.approx(ref["f_bound"], rel=1e-12)
    assert res[0][1:] == res[1][1:]  # every rank holds the same report
