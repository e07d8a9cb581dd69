"""Host-side API contract on the CPU: validation, exceptions, dataclasses,
reports and the host linear-algebra helpers (no GPU calls)."""

import numpy as np
import pytest

import paper_1702_02241_b200 as api


def test_problem_spec_validation():
    with pytest.raises(ValueError):
        api.ProblemSpec(x=np.ones((2, 2)), lambda_l=0.0, lambda_s=1.0)
    with pytest.raises(ValueError):
        api.ProblemSpec(x=np.ones((2, 2)), lambda_l=1.0, lambda_s=-0.5)
    with pytest.raises(api.DimensionError):
        api.ProblemSpec(x=np.ones((2, 2)), lambda_l=1.0, lambda_s=1.0, mask=np.ones((3, 2), bool))
    with pytest.raises(ValueError):
        api.ProblemSpec(x=np.array([[np.nan, 1.0]]), lambda_l=1.0, lambda_s=1.0)
    with pytest.raises(api.DimensionError):
        api.ProblemSpec(x=np.ones(3), lambda_l=1.0, lambda_s=1.0)
    spec = api.ProblemSpec(x=[[1.0, 2.0]], lambda_l=1, lambda_s=2)
    assert spec.shape == (1, 2) and spec.lambda_l == 1.0 and spec.fp32_exact()
    spec = api.ProblemSpec(x=[[0.1]], lambda_l=1, lambda_s=2)
    assert not spec.fp32_exact()
    m = np.array([[True, False]])
    spec = api.ProblemSpec(x=[[1.0, 5.0]], lambda_l=1, lambda_s=2, mask=m)
    np.testing.assert_array_equal(spec.observed(), [[1.0, 0.0]])


def test_error_hierarchy():
    assert issubclass(api.DimensionError, ValueError)
    assert issubclass(api.DimensionError, api.SpcpError)
    assert issubclass(api.NumericalError, ArithmeticError)
    assert issubclass(api.PowerIterationError, api.NumericalError)
    assert issubclass(api.DeviceError, api.NumericalError)
    e = api.PowerIterationError("x", u=1, sigma=2.0, v=3)
    assert (e.u, e.sigma, e.v) == (1, 2.0, 3)


def test_factor_pair_and_config():
    fp = api.FactorPair(np.ones((4, 2)), np.ones((3, 2)))
    assert fp.k == 2 and fp.shape == (4, 3)
    z = fp.flatten()
    fp2 = api.FactorPair.from_flat(z, 4, 3, 2)
    np.testing.assert_array_equal(fp2.u, fp.u)
    with pytest.raises(api.DimensionError):
        api.FactorPair(np.ones((4, 2)), np.ones((3, 3)))
    with pytest.raises(ValueError):
        api.SolverConfig(wolfe_c1=0.5, wolfe_c2=0.1)
    with pytest.raises(ValueError):
        api.SolverConfig(memory=0)
    with pytest.raises(ValueError):
        api.SolverConfig(precision="bf16")
    cfg = api.SolverConfig()
    assert (cfg.memory, cfg.grad_tol, cfg.max_iter, cfg.wolfe_c1, cfg.wolfe_c2) == \
        (10, 1e-8, 500, 1e-4, 0.9)


def test_split_objective_shape_check_before_device():
    spec = api.ProblemSpec(x=np.ones((4, 4)), lambda_l=1.0, lambda_s=1.0)
    with pytest.raises(api.DimensionError):
        api.split_objective(api.FactorPair(np.ones((3, 2)), np.ones((4, 2))), spec)
    with pytest.raises(api.DimensionError):
        api.phi_value_grad(np.zeros((2, 3)), api.ProblemSpec(x=np.ones((3, 2)), lambda_l=1.0,
                                                             lambda_s=1.0))
    with pytest.raises(api.DimensionError):
        api.solve_split_spcp(spec, 5)
    with pytest.raises(api.DimensionError):
        api.init_factors(spec, 0)


def test_shrink_huber():
    assert api.shrink(2.0, 1.0) == 1.0 and api.shrink(-0.5, 1.0) == 0.0
    assert api.huber(0.5, 1.0) == 0.125 and api.huber(3.0, 1.0) == 2.5
    with pytest.raises(ValueError):
        api.huber(1.0, 0.0)


def test_host_linalg():
    q, r = api.thin_qr(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(q, [[0.6], [0.8]])
    assert r[0, 0] == 5.0
    t = api.svd_small(np.diag([3.0, 1.0]))
    np.testing.assert_allclose(t.sigma, [3.0, 1.0])
    a = np.outer([1.0, 2.0, 2.0], [3.0, 4.0])
    u, s, v = api.leading_triple(lambda x: a @ x, lambda y: a.T @ y, 3, 2, seed=1)
    assert s == pytest.approx(15.0)


def test_report_lazy_dense_and_trace():
    calls = []

    def mk():
        calls.append(1)
        return np.zeros((2, 2))

    rec = api.IterationRecord(0, 3.0, 1.0, 0.1, {"rank": 2})
    rep = api.SolveReport("split", "converged", [rec], mk, mk, 2.5)
    assert not calls
    assert rep.l.shape == (2, 2) and len(calls) == 1
    _ = rep.l
    assert len(calls) == 1  # cached
    assert rep.best_objective == 2.5 and rep.converged
    td = rep.trace_dict()
    assert td["iterations"][0]["rank"] == 2


def test_factor_svd_host():
    fp = api.FactorPair(np.array([[2.0], [0.0]]), np.array([[3.0], [0.0]]))
    t = api.factor_svd(fp)
    np.testing.assert_allclose(t.sigma, [6.0], atol=1e-14)
    assert api.factor_svd(api.FactorPair(np.zeros((5, 2)), np.zeros((4, 2)))).rank == 0


def test_collective_failure_maps_to_device_error(monkeypatch):
    """A failing collective (NCCL/gloo RuntimeError) surfaces as DeviceError,
    a NumericalError like every CUDA failure."""
    import numpy as np
    import torch.distributed as tdist

    from paper_1702_02241_b200 import dist as pdist
    from paper_1702_02241_b200.errors import DeviceError, NumericalError

    def boom(*a, **k):
        raise RuntimeError("NCCL error: unhandled system error")

    monkeypatch.setattr(tdist, "all_reduce", boom)
    with pytest.raises(DeviceError) as ei:
        pdist.allreduce_host(np.zeros(3), "cpu")
    assert isinstance(ei.value, NumericalError)
