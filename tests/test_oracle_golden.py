"""Pin the CPU oracle against fixtures produced by the real reference.

These run on the CPU (no GPU marker).  The fixtures were written by
tests/golden/make_golden.py, which imports /root/reference/pkg/src/spcp.
"""

import numpy as np
import pytest


def test_phi_matches_reference(golden, oracle):
    d = golden("phi")
    for tag in ("full", "mask"):
        mask = d[f"{tag}_mask"] if f"{tag}_mask" in d else None
        val, g, s = oracle.phi_value_grad(d[f"{tag}_l"], d[f"{tag}_x"], 0.6, mask)
        assert val == float(d[f"{tag}_value"])
        np.testing.assert_array_equal(g, d[f"{tag}_grad"])
        np.testing.assert_array_equal(s, d[f"{tag}_s"])
    val, g, s = oracle.phi_value_grad(np.zeros((1, 1)), np.array([[2.0]]), 1.0)
    assert val == float(d["kat_value"]) == 1.5
    assert g[0, 0] == -1.0 and s[0, 0] == 1.0


def test_split_objective_matches_reference(golden, oracle):
    d = golden("split")
    for i in range(int(d["n_cases"])):
        m, n, k, masked, ll, ls = d[f"c{i}_meta"]
        mask = d[f"c{i}_mask"] if masked else None
        f, gu, gv = oracle.split_objective(d[f"c{i}_u"], d[f"c{i}_v"], d[f"c{i}_x"], ll, ls, mask)
        assert f == pytest.approx(float(d[f"c{i}_f"]), rel=1e-14)
        np.testing.assert_allclose(gu, d[f"c{i}_gu"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(gv, d[f"c{i}_gv"], rtol=1e-12, atol=1e-13)
    f, gu, gv = oracle.split_objective([[2.0]], [[3.0]], [[0.0]], 1.0, 10.0)
    assert (f, gu[0, 0], gv[0, 0]) == (24.5, 20.0, 15.0)
    assert f == float(d["kat_f"])


def test_lbfgs_matches_reference(golden, oracle):
    d = golden("lbfgs")

    def rosen(z):
        a, b = z
        f = (1 - a) ** 2 + 100.0 * (b - a * a) ** 2
        g = np.array([-2 * (1 - a) - 400.0 * a * (b - a * a), 200.0 * (b - a * a)])
        return f, g

    res = oracle.minimize_lbfgs(rosen, np.array([-1.2, 1.0]), grad_tol=1e-12, max_iter=200)
    assert res["termination"] == str(d["rosen_term"])
    assert res["n_evals"] == int(d["rosen_evals"])
    np.testing.assert_array_equal(res["x"], d["rosen_x"])
    np.testing.assert_array_equal([r[1] for r in res["records"]], d["rosen_obj"])
    c = d["quad_c"]
    res = oracle.minimize_lbfgs(lambda z: (0.5 * float((z - c) @ (z - c)), z - c), np.zeros(12),
                                grad_tol=1e-12, max_iter=12)
    assert res["termination"] == str(d["quad_term"])
    np.testing.assert_array_equal(res["x"], d["quad_x"])


def test_synth_and_rsvd_match_reference(golden, oracle):
    d = golden("synth")
    x, l_ref, s_ref = oracle.gen_low_rank_plus_sparse(30, 20, 3, 0.1, 1e-3, seed=5)
    np.testing.assert_array_equal(x, d["x"])
    np.testing.assert_array_equal(l_ref, d["l_ref"])
    np.testing.assert_array_equal(s_ref, d["s_ref"])
    np.testing.assert_array_equal(oracle.gen_mask(30, 20, 0.3, seed=6), d["mask"])
    u, s, v = oracle.rand_svd(x, 3, oversample=5, power_iters=1, seed=3)
    np.testing.assert_array_equal(u, d["rsvd_u"])
    np.testing.assert_array_equal(s, d["rsvd_s"])
    np.testing.assert_array_equal(v, d["rsvd_v"])


def test_solve_matches_reference(golden, oracle):
    d = golden("solve")
    for i in range(int(d["n_cases"])):
        m, n, k, masked, ll, ls, growth = d[f"s{i}_meta"]
        mask = d[f"s{i}_mask"] if masked else None
        res = oracle.solve_split_spcp(d[f"s{i}_x"], ll, ls, int(k), mask=mask, grad_tol=1e-9,
                                      max_iter=2000, rank_growth=bool(growth),
                                      max_k=5 if growth else None)
        assert res["termination"] == str(d[f"s{i}_term"])
        assert res["n_evals"] == int(d[f"s{i}_evals"])
        assert res["k_final"] == int(d[f"s{i}_kfinal"])
        np.testing.assert_array_equal([r[1] for r in res["records"]], d[f"s{i}_recobj"])
        np.testing.assert_array_equal(res["l"], d[f"s{i}_l"])
        np.testing.assert_array_equal(res["s"], d[f"s{i}_s"])
        cert = oracle.certificate(res["u"], res["v"], d[f"s{i}_x"], ll, ls, mask,
                                  f_bound_hint=min([r[1] for r in res["records"]]
                                                   + [res["objective"]]))
        ref = d[f"s{i}_cert"]
        assert cert["r"] == int(ref[7])
        assert cert["e_norm"] == pytest.approx(ref[0], rel=1e-9, abs=1e-12)
        assert cert["gap_bound"] == pytest.approx(ref[6], rel=1e-9, abs=1e-12)


def test_certificate_matches_reference(golden, oracle):
    d = golden("cert")
    for i in range(int(d["n_cases"])):
        cert = oracle.certificate(d[f"q{i}_u"], d[f"q{i}_v"], d[f"q{i}_x"], 1.1, 0.4)
        ref = d[f"q{i}_cert"]
        assert cert["r"] == int(ref[7])
        np.testing.assert_allclose([cert["e_norm"], *cert["terms"], cert["f_bound"],
                                    cert["gap_bound"], cert["l_norm"]],
                                   np.r_[ref[:7], ref[8]], rtol=1e-10, atol=1e-12)
    cert = oracle.certificate(np.zeros((6, 1)), np.zeros((5, 1)), d["zero_x"], 2.0, 0.3)
    assert cert["r"] == 0
    assert cert["e_norm"] == pytest.approx(float(d["zero_cert"][0]), rel=1e-12)


def test_c1_init_point_matches_reference(golden, oracle):
    """Config C1 rsvd init point and objective at it (C1 solve itself is checked
    on the GPU side against the same fixture)."""
    d = golden("c1")
    x, _, _ = oracle.gen_low_rank_plus_sparse(1000, 1000, 10, 0.05, 1e-3, seed=0)
    x = x.astype(np.float32).astype(np.float64)
    assert float(x.sum()) == float(d["x_sum"])
    u, v = oracle.init_factors(x, 10, strategy="rsvd", seed=0)
    np.testing.assert_allclose(u, d["init_u"], rtol=0, atol=1e-10)
    f, gu, gv = oracle.split_objective(u, v, x, 10.0, 0.1)
    assert f == pytest.approx(float(d["init_f"]), rel=1e-12)
