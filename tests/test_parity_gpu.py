"""GPU parity of the fused streaming kernel and the drop-in API against the
CPU oracle / golden fixtures of the real reference.

Tolerances (BASELINE.json north star): per-evaluation objective and gradient
1e-5 relative in fp32, 1e-10 in fp64; raw G.V / G^T.U checked separately
from the full gradient.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
FP64_TOL = 1e-10


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def api():
    import paper_1702_02241_b200 as pkg

    return pkg


def _spec(api, x, ll, ls, mask=None):
    return api.ProblemSpec(x=x, lambda_l=ll, lambda_s=ls, mask=mask)


def test_kats(api):
    spec = _spec(api, [[0.0]], 1.0, 10.0)
    for prec in ("fp64", "fp32"):
        f, gu, gv = api.split_objective(api.FactorPair([[2.0]], [[3.0]]), spec, precision=prec)
        assert (f, gu[0, 0], gv[0, 0]) == (24.5, 20.0, 15.0)
    spec = _spec(api, [[2.0]], 1.0, 1.0)
    val, g, s = api.phi_value_grad(np.zeros((1, 1)), spec)
    assert (val, g[0, 0], s[0, 0]) == (1.5, -1.0, 1.0)
    rng = np.random.default_rng(30)
    x = rng.standard_normal((10, 8)) * 2
    spec = _spec(api, x, 1.0, 0.7)
    f, gu, gv = api.split_objective(api.FactorPair(np.zeros((10, 3)), np.zeros((8, 3))), spec)
    assert f == pytest.approx(float(np.sum(api.huber(x, 0.7))), rel=1e-14)
    assert not gu.any() and not gv.any()
    val, g, s = api.phi_value_grad(x, spec)  # perfect fit
    assert val == 0.0 and not g.any() and not s.any()


def test_split_golden_fp64(api, golden):
    d = golden("split")
    for i in range(int(d["n_cases"])):
        m, n, k, masked, ll, ls = d[f"c{i}_meta"]
        mask = d[f"c{i}_mask"] if masked else None
        spec = _spec(api, d[f"c{i}_x"], ll, ls, mask)
        f, gu, gv = api.split_objective(api.FactorPair(d[f"c{i}_u"], d[f"c{i}_v"]), spec,
                                        precision="fp64")
        assert abs(f - float(d[f"c{i}_f"])) <= FP64_TOL * abs(float(d[f"c{i}_f"])), i
        assert rel(np.r_[gu.ravel(), gv.ravel()],
                   np.r_[d[f"c{i}_gu"].ravel(), d[f"c{i}_gv"].ravel()]) <= FP64_TOL, i


def test_split_golden_fp32(api, golden, oracle):
    """fp32 kernel vs the oracle on the same fp32-rounded X, U, V."""
    d = golden("split")
    for i in range(int(d["n_cases"])):
        m, n, k, masked, ll, ls = d[f"c{i}_meta"]
        mask = d[f"c{i}_mask"] if masked else None
        x, u, v = f32(d[f"c{i}_x"]), f32(d[f"c{i}_u"]), f32(d[f"c{i}_v"])
        spec = _spec(api, x, ll, ls, mask)
        f, gu, gv = api.split_objective(api.FactorPair(u, v), spec, precision="fp32")
        fr, gur, gvr = oracle.split_objective(u, v, x, ll, ls, mask)
        assert abs(f - fr) <= FP32_TOL * abs(fr), (i, f, fr)
        assert rel(np.r_[gu.ravel(), gv.ravel()], np.r_[gur.ravel(), gvr.ravel()]) <= FP32_TOL, i


SHAPES = [  # m, n, k, masked — multiple tiles / chunks / bands, ragged edges
    (1000, 1000, 10, False),
    (777, 1333, 20, True),
    (2049, 300, 3, False),
    (300, 2049, 32, True),
    (1500, 900, 50, False),
    (640, 520, 64, True),
    (400, 350, 70, False),  # beyond the fused widths: dense fallback
    (900, 700, 5, True),    # K-concatenated images, SEG = 8 (two K-steps)
    (700, 1100, 16, False),  # SEG = 16
    (5000, 260, 12, True),  # SEG = 12, tall-skinny (C3 shape class)
    (1100, 900, 21, False),  # SEG = 32 one-atom rows (k = 21..32), padded ranks
    (600, 1300, 27, True),
    (2000, 700, 30, False),  # C4's rank
]


@pytest.mark.parametrize("m,n,k,masked", SHAPES)
def test_eval_random_shapes(api, oracle, m, n, k, masked):
    rng = np.random.default_rng(m * 7 + n + k)
    x = f32(rng.standard_normal((m, n)) * 3.0)
    mask = rng.random((m, n)) < 0.6 if masked else None
    if mask is not None:
        x = np.where(mask, x, 1e6)  # garbage off the mask must be ignored
    u = f32(rng.standard_normal((m, k)) / np.sqrt(k))
    v = f32(rng.standard_normal((n, k)) / np.sqrt(k))
    ll, ls = 1.3, 0.5
    spec = _spec(api, x, ll, ls, mask)
    fr, gur, gvr = oracle.split_objective(u, v, x, ll, ls, mask)
    phi_r, gvr_raw, gtur_raw = oracle.split_raw_products(u, v, x, ls, mask)
    for prec, tol in (("fp64", FP64_TOL), ("fp32", FP32_TOL)):
        f, gu, gv = api.split_objective(api.FactorPair(u, v), spec, precision=prec)
        assert abs(f - fr) <= tol * abs(fr), (prec, f, fr)
        assert rel(np.r_[gu.ravel(), gv.ravel()], np.r_[gur.ravel(), gvr.ravel()]) <= tol, prec
        # raw reductions G V and G^T U
        assert rel(gu - ll * u, gvr_raw) <= tol, prec
        assert rel(gv - ll * v, gtur_raw) <= tol, prec


def test_phi_golden(api, golden):
    d = golden("phi")
    for tag in ("full", "mask"):
        mask = d[f"{tag}_mask"] if f"{tag}_mask" in d else None
        spec = _spec(api, d[f"{tag}_x"], 1.3, 0.6, mask)
        val, g, s = api.phi_value_grad(d[f"{tag}_l"], spec)
        assert val == pytest.approx(float(d[f"{tag}_value"]), rel=1e-13)
        np.testing.assert_array_equal(g, d[f"{tag}_grad"])
        np.testing.assert_allclose(s, d[f"{tag}_s"], rtol=0, atol=1e-15)


def test_eval_is_deterministic(api):
    rng = np.random.default_rng(5)
    x = f32(rng.standard_normal((1500, 1100)))
    spec = _spec(api, x, 2.0, 0.3)
    fp = api.FactorPair(rng.standard_normal((1500, 12)), rng.standard_normal((1100, 12)))
    for prec in ("fp32", "fp64"):
        a = api.split_objective(fp, spec, precision=prec)
        b = api.split_objective(fp, spec, precision=prec)
        assert a[0] == b[0]
        np.testing.assert_array_equal(a[1], b[1])
        np.testing.assert_array_equal(a[2], b[2])


def test_device_eval_trial_point(api, oracle):
    """spcp_eval at z + alpha dz (the line-search form) and its g.dz."""
    import torch

    from paper_1702_02241_b200._lib import SPCP_F32, SPCP_F64

    rng = np.random.default_rng(9)
    m, n, k = 900, 700, 16
    x = f32(rng.standard_normal((m, n)))
    spec = _spec(api, x, 1.7, 0.4)
    dp = spec.device("mixed")
    z = rng.standard_normal((m + n) * k)
    dz = rng.standard_normal((m + n) * k)
    alpha = 0.37
    w = z + alpha * dz
    fr, gr = oracle.flat_objective(x, 1.7, 0.4, None, m, n, k)(w)
    zt, dzt = torch.from_numpy(z).cuda(), torch.from_numpy(dz).cuda()
    g = torch.empty_like(zt)
    for code, tol in ((SPCP_F64, FP64_TOL), (SPCP_F32, FP32_TOL)):
        out = dp.eval(k, code, zt, dzt, alpha, g)
        assert abs(out[0] - fr) <= tol * abs(fr)
        assert rel(g.cpu().numpy(), gr) <= tol
        assert out[3] == pytest.approx(float(gr @ dz), rel=max(tol, 1e-12) * 10)
        assert out[4] == pytest.approx(float(gr @ gr), rel=max(tol, 1e-12) * 10)


def test_apply_products(api, oracle):
    """spcp_apply: G W and G^T W (k >= 1) and the raw observed-matrix
    products (k == 0) against numpy."""
    import torch

    rng = np.random.default_rng(11)
    m, n, k, b = 700, 500, 6, 13
    x = f32(rng.standard_normal((m, n)))
    mask = rng.random((m, n)) < 0.7
    spec = _spec(api, x, 1.1, 0.5, mask)
    dp = spec.device("fp64")
    u = rng.standard_normal((m, k))
    v = rng.standard_normal((n, k))
    z = torch.from_numpy(np.r_[u.ravel(), v.ravel()]).cuda()
    wr = rng.standard_normal((n, b))
    wl = rng.standard_normal((m, b))
    _, g, _ = oracle.phi_value_grad(u @ v.T, x, 0.5, mask)
    left, right = dp.apply(k, z, w_right=torch.from_numpy(wr).cuda(),
                           w_left=torch.from_numpy(wl).cuda())
    assert rel(left.cpu().numpy(), g @ wr) <= 1e-12
    assert rel(right.cpu().numpy(), g.T @ wl) <= 1e-12
    obs = np.where(mask, x, 0.0)
    left, right = dp.apply(0, None, w_right=torch.from_numpy(wr).cuda(),
                           w_left=torch.from_numpy(wl).cuda())
    assert rel(left.cpu().numpy(), obs @ wr) <= 1e-12
    assert rel(right.cpu().numpy(), obs.T @ wl) <= 1e-12


@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("b", [5, 30, 64, 71])
def test_apply0_tensor_core_products(api, masked, b):
    """k == 0 fp64 products of fp32-exact X (the rSVD sketches) on the FP64
    tensor cores: X W and X^T W, one side or both, widths up to 64 per pass
    (71: two passes), odd shapes, against numpy."""
    import torch

    rng = np.random.default_rng(100 + b + masked)
    m, n = 333, 517
    x = f32(rng.standard_normal((m, n)))
    mask = (rng.random((m, n)) < 0.6) if masked else None
    spec = _spec(api, x, 1.0, 0.5, mask)
    dp = spec.device("fp64")
    obs = x if mask is None else np.where(mask, x, 0.0)
    wr = rng.standard_normal((n, b))
    wl = rng.standard_normal((m, b))
    left, right = dp.apply(0, None, w_right=torch.from_numpy(wr).cuda(),
                           w_left=torch.from_numpy(wl).cuda())
    assert rel(left.cpu().numpy(), obs @ wr) <= 1e-13
    assert rel(right.cpu().numpy(), obs.T @ wl) <= 1e-13
    left, _ = dp.apply(0, None, w_right=torch.from_numpy(wr).cuda())
    assert rel(left.cpu().numpy(), obs @ wr) <= 1e-13
    _, right = dp.apply(0, None, w_left=torch.from_numpy(wl).cuda())
    assert rel(right.cpu().numpy(), obs.T @ wl) <= 1e-13
    spec.release_device()


def test_materialize_l_s(api, oracle):
    import torch

    rng = np.random.default_rng(12)
    m, n, k = 333, 257, 5
    x = f32(rng.standard_normal((m, n)) * 2)
    mask = rng.random((m, n)) < 0.8
    spec = _spec(api, x, 1.0, 0.45, mask)
    dp = spec.device("fp64")
    u = rng.standard_normal((m, k))
    v = rng.standard_normal((n, k))
    z = torch.from_numpy(np.r_[u.ravel(), v.ravel()]).cuda()
    l, s = dp.materialize(k, z)
    np.testing.assert_allclose(l, u @ v.T, rtol=0, atol=1e-12)
    _, _, s_ref = oracle.phi_value_grad(u @ v.T, x, 0.45, mask)
    np.testing.assert_allclose(s, s_ref, rtol=0, atol=1e-12)
    assert (s[~mask] == 0).all()


@pytest.mark.parametrize("k,b,masked", [(6, 13, True), (20, 40, False), (32, 8, True)])
def test_apply_f32_products(api, oracle, k, b, masked):
    """spcp_apply_f32 (the certificate's subspace-iteration products): fp32
    streaming over the fp32 copy of X, within the fp32 tolerance of numpy."""
    import torch

    from paper_1702_02241_b200.device import DeviceProblem

    rng = np.random.default_rng(100 + k)
    m, n = 900, 700
    x = f32(rng.standard_normal((m, n)) * 2.0)
    mask = rng.random((m, n)) < 0.6 if masked else None
    dp = DeviceProblem(x, 1.3, 0.5, mask=mask, store=("f32", "f64"))
    u = f32(rng.standard_normal((m, k)) / np.sqrt(k))
    v = f32(rng.standard_normal((n, k)) / np.sqrt(k))
    z = torch.from_numpy(np.r_[u.ravel(), v.ravel()]).cuda()
    wr = rng.standard_normal((n, b))
    wl = rng.standard_normal((m, b))
    _, g, _ = oracle.phi_value_grad(u @ v.T, x, 0.5, mask)
    left, right = dp.apply(k, z, w_right=torch.from_numpy(wr).cuda(),
                           w_left=torch.from_numpy(wl).cuda(), precision="fp32")
    assert rel(left.cpu().numpy(), g @ wr) <= FP32_TOL
    assert rel(right.cpu().numpy(), g.T @ wl) <= FP32_TOL


@pytest.mark.parametrize("k,masked", [(12, False), (20, True), (30, False)])
def test_sharded_partial_finish_on_one_gpu(api, k, masked):
    """The column-sharded C ABI (spcp_eval_partial -> all-reduce -> spcp_eval_finish,
    SURVEY §8(e)) with two column shards on one GPU and the all-reduce done by
    hand: f, g.dz and the gradient match the unsharded evaluation."""
    import torch

    from paper_1702_02241_b200._lib import SPCP_F32, SPCP_F64
    from paper_1702_02241_b200.device import DeviceProblem

    rng = np.random.default_rng(500 + k)
    m, n = 1100, 900
    x = f32(rng.standard_normal((m, n)) * 2.0)
    mask = rng.random((m, n)) < 0.7 if masked else None
    ll, ls = 1.7, 0.4
    u = rng.standard_normal((m, k)) / np.sqrt(k)
    v = rng.standard_normal((n, k)) / np.sqrt(k)
    du = rng.standard_normal((m, k)) * 1e-2
    dv = rng.standard_normal((n, k)) * 1e-2
    alpha = 0.3
    full = DeviceProblem(x, ll, ls, mask=mask, store=("f32", "f64"))
    z = torch.from_numpy(np.r_[u.ravel(), v.ravel()]).cuda()
    dz = torch.from_numpy(np.r_[du.ravel(), dv.ravel()]).cuda()
    cut = 413
    shards = [(0, cut), (cut, n)]
    for code, tol in ((SPCP_F64, FP64_TOL), (SPCP_F32, FP32_TOL)):
        g_full = torch.empty_like(z)
        out_full = full.eval(k, code, z, dz, alpha, g_full)
        gu_dtype = torch.float32 if code == SPCP_F32 else torch.float64
        parts = []
        for c0, c1 in shards:
            dp = DeviceProblem(np.ascontiguousarray(x[:, c0:c1]), ll, ls,
                               mask=None if mask is None else np.ascontiguousarray(mask[:, c0:c1]),
                               store=("f32", "f64"), n_total=n, col0=c0)
            zs = torch.cat([z[: m * k], z[m * k + c0 * k: m * k + c1 * k]])
            dzs = torch.cat([dz[: m * k], dz[m * k + c0 * k: m * k + c1 * k]])
            gu = torch.empty((m, k), dtype=gu_dtype, device="cuda")
            scal = torch.empty(4, dtype=torch.float64, device="cuda")
            gs = torch.empty_like(zs)
            dp.eval_partial(k, code, zs, dzs, alpha, gu, scal, gs)
            parts.append((dp, zs, dzs, gu, scal, gs, c0, c1))
        gu_sum = sum(pt[3].double() for pt in parts).to(gu_dtype)
        scal_sum = sum(pt[4] for pt in parts)
        for dp, zs, dzs, _, _, gs, c0, c1 in parts:
            out = dp.eval_finish(k, code, zs, dzs, alpha, gu_sum, scal_sum, gs)
            assert abs(out[0] - out_full[0]) <= tol * abs(out_full[0])
            assert out[3] == pytest.approx(out_full[3], rel=10 * tol, abs=1e-12)
            assert rel(gs[: m * k].cpu().numpy(), g_full[: m * k].cpu().numpy()) <= tol
            assert rel(gs[m * k:].cpu().numpy(),
                       g_full[m * k + c0 * k: m * k + c1 * k].cpu().numpy()) <= tol
