"""Stored-ray probes of the fp64 line searches (csrc/line.cuh, spcp_line_*):
F and grad F . dz at z + a dz from R0, D1, D2 agree with the full fp64
evaluation and with the oracle; solves that answer their long searches from
the stored ray reach the same objective and termination as direct probing."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import paper_1702_02241_b200 as pkg

    return pkg


@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("exact32", [False, True])
def test_line_probe_matches_eval_and_oracle(api, oracle, masked, exact32):
    import torch

    from paper_1702_02241_b200._lib import SPCP_F64

    rng = np.random.default_rng(40 + 2 * masked + exact32)
    m, n, k = 333, 517, 7
    x = rng.standard_normal((m, k)) @ rng.standard_normal((k, n)) + \
        0.3 * rng.standard_normal((m, n))
    if exact32:
        x = x.astype(np.float32).astype(np.float64)
    mask = (rng.random((m, n)) < 0.6) if masked else None
    ll, ls = 2.0, 0.4
    spec = api.ProblemSpec(x=x, lambda_l=ll, lambda_s=ls, mask=mask)
    dp = spec.device("fp64")
    z = rng.standard_normal((m + n) * k)
    d = 0.3 * rng.standard_normal((m + n) * k)
    zt = torch.from_numpy(z).cuda()
    dt = torch.from_numpy(d).cuda()
    g = torch.empty_like(zt)
    assert dp.line_setup(k, zt, dt)
    for a in (0.0, 1e-9, 1e-3, 0.37, 1.0, 2.5):
        lp = dp.line_probe(a)
        ev = dp.eval(k, SPCP_F64, zt, dt, a, g)
        assert lp[0] == pytest.approx(ev[0], rel=1e-12), a
        assert lp[1] == pytest.approx(ev[1], rel=1e-12), a
        assert lp[2] == pytest.approx(ev[2], rel=1e-12), a
        scale = float(np.linalg.norm(g.cpu().numpy()) * np.linalg.norm(d))
        assert abs(lp[3] - ev[3]) <= 1e-12 * scale, a
        w = z + a * d
        fo, go = oracle.flat_objective(x, ll, ls, mask, m, n, k)(w)
        assert lp[0] == pytest.approx(fo, rel=1e-11), a
        assert abs(lp[3] - float(go @ d)) <= 1e-11 * scale, a
    dp.line_release()
    with pytest.raises(ValueError):
        dp.line_probe(0.5)
    spec.release_device()


@pytest.mark.parametrize("after", [0, 3])
def test_solves_with_stored_ray_probes(api, golden, after, monkeypatch):
    """The golden solve cases with every fp64 search (after = 0) or the long
    ones (after = 3, the default) probed from the stored ray: same objective
    (1e-9) and termination as direct probing."""
    import paper_1702_02241_b200.lbfgs as lb

    d = golden("solve")
    for case in (1, 2, 4):
        m, n, k, masked, ll, ls, growth = d[f"s{case}_meta"]
        x = d[f"s{case}_x"]
        mask = d[f"s{case}_mask"] if masked else None
        cfg = api.SolverConfig(grad_tol=1e-9, max_iter=2000, rank_growth=bool(growth),
                               max_k=5 if growth else None, precision="fp64")
        res = {}
        for mode in (None, after):
            monkeypatch.setattr(lb, "LINE_PROBES_AFTER", mode)
            spec = api.ProblemSpec(x=x, lambda_l=ll, lambda_s=ls, mask=mask)
            res[mode] = api.solve_split_spcp(spec, int(k), cfg)
            spec.release_device()
        a, b = res[None], res[after]
        assert b.objective == pytest.approx(a.objective, rel=1e-9), case
        assert b.termination == a.termination, case
        assert b.objective == pytest.approx(float(d[f"s{case}_obj"]), rel=1e-8), case
