"""L-BFGS control flow on the CPU.

* minimize_lbfgs (host plug-in API) reproduces the reference's records and
  iterates exactly (golden fixtures from the real reference).
* DeviceLbfgs — the dot-product form of the two-loop recursion used on the
  GPU — driven through a numpy vector space follows the reference
  trajectory on the golden SPCP problems.
"""

import numpy as np
import pytest

from fakes import NumpySpace
from paper_1702_02241_b200 import FactorPair, SolverConfig, lbfgs_minimize, minimize_lbfgs
from paper_1702_02241_b200.lbfgs import DeviceLbfgs


def rosen(z):
    a, b = z
    f = (1 - a) ** 2 + 100.0 * (b - a * a) ** 2
    g = np.array([-2 * (1 - a) - 400.0 * a * (b - a * a), 200.0 * (b - a * a)])
    return f, g


def test_host_lbfgs_matches_reference_exactly(golden):
    d = golden("lbfgs")
    res = minimize_lbfgs(rosen, np.array([-1.2, 1.0]), grad_tol=1e-12, max_iter=200)
    assert res.termination == str(d["rosen_term"])
    assert res.n_evals == int(d["rosen_evals"])
    np.testing.assert_array_equal(res.x, d["rosen_x"])
    np.testing.assert_array_equal([r.objective for r in res.records], d["rosen_obj"])
    np.testing.assert_array_equal([r.grad_norm for r in res.records], d["rosen_gn"])
    c = d["quad_c"]
    res = minimize_lbfgs(lambda z: (0.5 * float((z - c) @ (z - c)), z - c), np.zeros(12),
                         grad_tol=1e-12, max_iter=12)
    assert res.termination == "converged"
    np.testing.assert_array_equal(res.x, d["quad_x"])


def test_host_lbfgs_reference_semantics():
    res = minimize_lbfgs(rosen, np.array([-1.2, 1.0]), grad_tol=1e-14, max_iter=3)
    assert res.termination == "max_iter" and len(res.records) == 4
    res = minimize_lbfgs(lambda z: (0.5 * float(z @ z), z.copy()), np.zeros(3), grad_tol=1e-8)
    assert res.termination == "converged" and len(res.records) == 1
    with pytest.raises(ValueError):
        minimize_lbfgs(rosen, np.zeros(2), c1=0.5, c2=0.1)
    res = minimize_lbfgs(lambda z: (0.5 * float(z @ z), z.copy()), np.ones(2),
                         iter_hook=lambda it, z: {"probe": it * 2}, max_iter=50)
    assert all(r.extra["probe"] == r.iteration * 2 for r in res.records)


def test_lbfgs_minimize_factor_wrapper():
    rep = lbfgs_minimize(rosen, FactorPair(np.array([[-1.2]]), np.array([[1.0]])),
                         SolverConfig(grad_tol=1e-12, max_iter=200))
    assert rep.objective <= 1e-10
    assert rep.factors.u[0, 0] == pytest.approx(1.0, abs=1e-5)


@pytest.mark.parametrize("case", [1, 2, 4])
def test_dot_product_two_loop_follows_reference(golden, oracle, case):
    """DeviceLbfgs (Gram-coefficient two-loop) vs the reference's two-loop on
    the same fp64 objective: identical accepted objectives to ~1e-10 over the
    well-conditioned part of the run, same final objective."""
    d = golden("solve")
    m, n, k, masked, ll, ls, growth = d[f"s{case}_meta"]
    m, n, k = int(m), int(n), int(k)
    x = d[f"s{case}_x"]
    u0, v0 = oracle.init_factors(x, k, strategy="rsvd", seed=0)
    sp = NumpySpace(x, ll, ls, m, n, k)
    eng = DeviceLbfgs(sp, memory=10, grad_tol=1e-9, max_iter=2000, precision="fp64")
    z = np.concatenate([u0.ravel(), v0.ravel()])
    res = eng.run(z)
    ref = d[f"s{case}_recobj"]
    ours = np.array([r.objective for r in res.records])
    cmp = min(len(ref), len(ours), 15)
    np.testing.assert_allclose(ours[:cmp], ref[:cmp], rtol=1e-9)
    assert res.objective == pytest.approx(float(d[f"s{case}_obj"]), rel=1e-9)
    assert res.termination in ("converged", "line_search_failed")


def test_mixed_precision_switch_logic(golden, oracle):
    """With a space whose 'fp32' is exact, mixed mode switches once and the
    trajectory continues; the switch costs one extra evaluation."""
    d = golden("solve")
    m, n, k = 120, 90, 8
    x = d["s4_x"]
    u0, v0 = oracle.init_factors(x, k, strategy="rsvd", seed=0)
    z = np.concatenate([u0.ravel(), v0.ravel()])
    sp = NumpySpace(x, 3.0, 0.2, m, n, k)
    eng = DeviceLbfgs(sp, grad_tol=1e-9, max_iter=2000, precision="mixed", switch_tol=1e-4)
    res = eng.run(z.copy())
    assert eng.switched_at is not None
    assert res.objective == pytest.approx(float(d["s4_obj"]), rel=1e-9)


@pytest.mark.parametrize("after", [0, 1, 3])
def test_stored_ray_probes_follow_the_direct_search(golden, oracle, after, monkeypatch):
    """fp64 searches answering probes from the stored ray (line_setup /
    line_probe) reach the direct run's objective and termination; every setup
    is released; a space whose ray does not fit keeps probing directly."""
    import paper_1702_02241_b200.lbfgs as lb

    from fakes import NumpyLineSpace

    d = golden("solve")
    m, n, k = 120, 90, 8
    x = d["s4_x"]
    u0, v0 = oracle.init_factors(x, k, strategy="rsvd", seed=0)
    z = np.concatenate([u0.ravel(), v0.ravel()])
    monkeypatch.setattr(lb, "LINE_PROBES_AFTER", None)
    direct = DeviceLbfgs(NumpySpace(x, 3.0, 0.2, m, n, k), grad_tol=1e-9, max_iter=2000,
                         precision="fp64").run(z.copy())
    monkeypatch.setattr(lb, "LINE_PROBES_AFTER", after)
    sp = NumpyLineSpace(x, 3.0, 0.2, m, n, k)
    res = DeviceLbfgs(sp, grad_tol=1e-9, max_iter=2000, precision="fp64").run(z.copy())
    assert res.objective == pytest.approx(direct.objective, rel=1e-10)
    assert res.termination == direct.termination
    assert sp.releases == (1 if sp.setups else 0)  # the workspace is freed when the run ends
    if after == 0:
        assert sp.line_probes > 0 and sp.setups == len(res.records) - 1 + (
            res.termination == "line_search_failed")
    nofit = NumpyLineSpace(x, 3.0, 0.2, m, n, k, fits=False)
    res2 = DeviceLbfgs(nofit, grad_tol=1e-9, max_iter=2000, precision="fp64").run(z.copy())
    assert nofit.line_probes == 0 and nofit.releases == 0
    assert res2.objective == pytest.approx(direct.objective, rel=1e-10)
