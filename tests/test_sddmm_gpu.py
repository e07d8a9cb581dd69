"""Sparse-observation evaluation (sddmm.cuh): the CSR row
pass + CSC column pass over the observed entries only, against the oracle's
masked split objective (objective.py:108-110, solver.py:105-123) and against
the dense streaming pass on the same problem.  Tolerances: fp64 1e-10,
fp32 1e-5 (north star)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _case(m, n, k, obs, seed):
    from oracle import spcp_oracle as orc

    x, _, _ = orc.gen_low_rank_plus_sparse(m, n, min(k, 6), 0.05, 1e-3, seed=seed)
    x = x.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(seed + 100)
    mask = rng.random((m, n)) < obs
    mask[3, :] = False  # an empty row
    mask[:, 5] = False  # an empty column
    u = rng.standard_normal((m, k)) * 0.7
    v = rng.standard_normal((n, k)) * 0.7
    return x, mask, u, v


@pytest.mark.parametrize("m,n,k,obs", [(300, 200, 5, 0.05), (1000, 700, 20, 0.05),
                                       (1500, 1100, 40, 0.2), (700, 900, 64, 0.08)])
def test_sparse_eval_matches_oracle_and_dense(m, n, k, obs):
    import torch

    from oracle import spcp_oracle as orc
    from paper_1702_02241_b200._lib import SPCP_F32, SPCP_F64
    from paper_1702_02241_b200.device import DeviceProblem

    x, mask, u, v = _case(m, n, k, obs, seed=m + k)
    garbage = x.copy()
    garbage[~mask] = 1e6  # off-mask values must not matter (test_objective.py:166-178)
    ll, ls = 1.3, 0.2
    f_ref, gu_ref, gv_ref = orc.split_objective(u, v, x, ll, ls, mask)
    z = torch.from_numpy(np.r_[u.ravel(), v.ravel()]).cuda()
    sp = DeviceProblem(garbage, ll, ls, mask=mask, store=("f32", "f64", "sparse"))
    de = DeviceProblem(garbage, ll, ls, mask=mask, store=("f32", "f64", "dense"))
    assert sp.sparse_nnz == int(mask.sum()) and de.sparse_nnz is None
    g_ref = np.r_[gu_ref.ravel(), gv_ref.ravel()]
    for code, tol in ((SPCP_F64, 1e-10), (SPCP_F32, 1e-5)):
        outs = []
        for dp in (sp, de):
            g = torch.empty_like(z)
            out = dp.eval(k, code, z, None, 0.0, g)
            outs.append((out[0], g.cpu().numpy()))
            assert abs(out[0] - f_ref) <= tol * abs(f_ref), (code, out[0], f_ref)
            assert rel(outs[-1][1], g_ref) <= tol, (code, rel(outs[-1][1], g_ref))
        # the two paths agree with each other at the same tolerance
        assert rel(outs[0][1], outs[1][1]) <= tol
    # bitwise reproducible
    g1, g2 = torch.empty_like(z), torch.empty_like(z)
    o1 = sp.eval(k, SPCP_F32, z, None, 0.0, g1)
    o2 = sp.eval(k, SPCP_F32, z, None, 0.0, g2)
    assert o1[0] == o2[0] and torch.equal(g1, g2)


def test_sparse_solve_matches_oracle():
    """A 6%-observed completion problem takes the sparse path automatically;
    the solve (solver.py:255-324) matches the oracle's objective and L."""
    from oracle import spcp_oracle as orc
    from paper_1702_02241_b200 import ProblemSpec, SolverConfig, solve_split_spcp

    m, n, r = 600, 400, 4
    x, _, _ = orc.gen_low_rank_plus_sparse(m, n, r, 0.02, 1e-3, seed=12)
    mask = orc.gen_mask(m, n, 0.06, seed=13)
    spec = ProblemSpec(x=x, lambda_l=1.0, lambda_s=0.3, mask=mask)
    rep = solve_split_spcp(spec, r, SolverConfig(max_iter=2000))
    assert spec.device("fp64").sparse_nnz == int(mask.sum())
    ref = orc.solve_split_spcp(x, 1.0, 0.3, r, mask=mask, max_iter=2000)
    assert rep.objective == pytest.approx(ref["objective"], rel=1e-8)
    assert rel(rep.l, ref["l"]) <= 1e-4
