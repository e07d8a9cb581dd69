"""SLRM files streamed to / from HBM and the CLI end to end on the GPU
(SURVEY §8(f) row 2), against the host reader and the REAL reference's CLI
runs in `tests/golden/io.npz` (`make_golden.py gen_io`).

* `spcp_slrm_read_device`: fp32 / fp64 / u8-mask conversions and column
  windows equal the host read exactly, across several 64 MiB pinned chunks
  with a ragged last chunk; non-finite payloads raise NonFiniteDataError.
* `spcp_slrm_write_device`: the file equals the host writer's bytes
  (float32 widened exactly, strided sources).
* `decompose` on the reference's own input files: same exit code, stdout
  line, termination, L and S within 1e-4 relative Frobenius (north star),
  nnz(S), trace schema, final-certificate verdict; `certify` of the
  reference's L gives its rank and verdict.
"""

import io
import json
from contextlib import redirect_stderr, redirect_stdout

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


@pytest.fixture(scope="module")
def big(tmp_path_factory):
    """2500 x 3500 float64 (70 MB): two pinned chunks, the second ragged."""
    from paper_1702_02241_b200.matrixio import write_matrix

    a = np.random.default_rng(7).standard_normal((2500, 3500))
    a[::97, ::13] = 0.0
    path = tmp_path_factory.mktemp("io") / "big.bin"
    write_matrix(a, path)
    return a, path


def test_device_read_matches_host(torch, big):
    from paper_1702_02241_b200.matrixio import read_matrix

    a, path = big
    t64 = read_matrix(path, device="cuda")
    assert t64.dtype == torch.float64 and t64.is_cuda
    assert t64.cpu().numpy().tobytes() == a.tobytes()
    t32 = read_matrix(path, device="cuda", dtype=torch.float32)
    np.testing.assert_array_equal(t32.cpu().numpy(), a.astype(np.float32))


def test_device_read_column_window(torch, big):
    from paper_1702_02241_b200.matrixio import read_matrix

    a, path = big
    for col0, cols in ((0, 1750), (1750, 1750), (333, 1001), (3499, 1)):
        t = read_matrix(path, device="cuda", col0=col0, cols=cols)
        assert t.cpu().numpy().tobytes() == np.ascontiguousarray(a[:, col0:col0 + cols]).tobytes()


def test_device_mask_read(torch, big):
    from paper_1702_02241_b200.matrixio import read_mask

    a, path = big
    np.testing.assert_array_equal(read_mask(path, device="cuda"), a != 0.0)
    np.testing.assert_array_equal(read_mask(path, device="cuda", col0=100, cols=50),
                                  a[:, 100:150] != 0.0)


def test_device_read_rejects_non_finite_and_short(torch, tmp_path):
    import struct

    from paper_1702_02241_b200 import NonFiniteDataError, TruncatedPayloadError
    from paper_1702_02241_b200.matrixio import read_matrix

    p = tmp_path / "nan.bin"
    p.write_bytes(struct.pack("<4sIQQ", b"SLRM", 1, 2, 2) + struct.pack("<4d", 1, 2, np.inf, 4))
    with pytest.raises(NonFiniteDataError):
        read_matrix(p, device="cuda")
    q = tmp_path / "short.bin"
    q.write_bytes(struct.pack("<4sIQQ", b"SLRM", 1, 2, 2) + struct.pack("<3d", 1, 2, 3))
    with pytest.raises(TruncatedPayloadError):
        read_matrix(q, device="cuda")
    with pytest.raises(Exception):
        read_matrix(p, device="cuda", col0=1, cols=5)


def test_device_write_matches_host_bytes(torch, big, tmp_path):
    from paper_1702_02241_b200.matrixio import write_matrix

    a, _ = big
    host, dev = tmp_path / "h.bin", tmp_path / "d.bin"
    write_matrix(a, host)
    write_matrix(torch.from_numpy(a).cuda(), dev)
    assert dev.read_bytes() == host.read_bytes()
    # float32 source widened exactly; strided (column-sliced) source
    a32 = a.astype(np.float32)
    write_matrix(torch.from_numpy(a32).cuda(), dev)
    write_matrix(a32.astype(np.float64), host)
    assert dev.read_bytes() == host.read_bytes()
    t = torch.from_numpy(a).cuda()[:, 7:1007]
    write_matrix(t, dev)
    write_matrix(np.ascontiguousarray(a[:, 7:1007]), host)
    assert dev.read_bytes() == host.read_bytes()
    assert sorted(p.name for p in tmp_path.iterdir()) == ["d.bin", "h.bin"]


def _run(argv):
    from paper_1702_02241_b200 import cli

    out, err = io.StringIO(), io.StringIO()
    with redirect_stdout(out), redirect_stderr(err):
        code = cli.main(argv)
    return code, out.getvalue(), err.getvalue()


@pytest.mark.parametrize("tag", ["full", "mask", "grow", "csv"])
def test_cli_decompose_matches_reference_run(golden, tmp_path, tag):
    """full / mask: certificate final / every:3; grow: --rank-growth from k=1
    (test_cli.py:164-183); csv: CSV input and outputs (host parse, upload)."""
    from paper_1702_02241_b200.matrixio import read_matrix

    d = golden("io")
    ext = "csv" if tag == "csv" else "bin"
    (tmp_path / f"{tag}_x.{ext}").write_bytes(d[f"{tag}_x"].tobytes())
    if f"{tag}_m" in d:
        (tmp_path / f"{tag}_m.bin").write_bytes(d[f"{tag}_m"].tobytes())
    args = json.loads(str(d[f"{tag}_args"]))
    args = [str(tmp_path / a) if a.endswith((".bin", ".csv", ".json")) else a for a in args]
    code, out, err = _run(["decompose", "--input", str(tmp_path / f"{tag}_x.{ext}")] + args)
    assert code == int(d[f"{tag}_exit"]), err
    ref_out = str(d[f"{tag}_stdout"])
    assert out.split(",")[0] == ref_out.split(",")[0]  # "split: converged"
    obj = float(out.rsplit(" ", 1)[1])
    assert obj == pytest.approx(float(ref_out.rsplit(" ", 1)[1]), rel=1e-7)
    assert "warning" not in err
    l_dev = read_matrix(tmp_path / f"{tag}_l.{ext}")
    s_dev = read_matrix(tmp_path / f"{tag}_s.{ext}")
    assert rel(l_dev, d[f"{tag}_l"]) < 1e-4
    assert rel(s_dev, d[f"{tag}_s"]) < 1e-4
    ref_tr = json.loads(str(d[f"{tag}_trace"]))
    tr = json.loads((tmp_path / f"{tag}_trace.json").read_text())
    assert set(ref_tr) <= set(tr)
    assert tr["config"] == ref_tr["config"]
    assert tr["termination"] == ref_tr["termination"]
    assert tr["final"]["nnz_s"] == int(np.count_nonzero(s_dev))
    assert abs(tr["final"]["nnz_s"] - ref_tr["final"]["nnz_s"]) <= 2
    assert tr["final"]["cert"]["rank"] == ref_tr["final"]["cert"]["rank"]
    assert set(tr["iterations"][0]) >= set(ref_tr["iterations"][0]) - {"cert"}
    assert tr["k_final"] == ref_tr["k_final"]
    assert tr["columns_grown"] == ref_tr["columns_grown"]
    ranks = [r["rank"] for r in tr["iterations"]]
    assert ranks == sorted(ranks)
    if "every" in ref_tr["config"]["certificate"]:
        every = ref_tr["config"]["cert_every"]
        assert all(("cert" in r) == (r["iter"] % every == 0) for r in tr["iterations"])


@pytest.mark.parametrize("tag", ["full", "mask", "grow"])
def test_cli_certify_matches_reference(golden, tmp_path, tag):
    d = golden("io")
    from paper_1702_02241_b200.matrixio import write_matrix

    (tmp_path / "x.bin").write_bytes(d[f"{tag}_x"].tobytes())
    write_matrix(d[f"{tag}_l"], tmp_path / "l.bin")
    lam = json.loads(str(d[f"{tag}_trace"]))["config"]["lambda_l"]
    argv = ["certify", "--input", str(tmp_path / "x.bin"), "--lambda-l", str(lam),
            "--lambda-s", "0.1", "--l", str(tmp_path / "l.bin"), "--output",
            str(tmp_path / "c.json")]
    if f"{tag}_m" in d:
        (tmp_path / "m.bin").write_bytes(d[f"{tag}_m"].tobytes())
        argv += ["--mask", str(tmp_path / "m.bin")]
    code, out, _ = _run(argv)
    assert code == 0 and out.startswith("e_norm ")
    ref = json.loads(str(d[f"{tag}_cert"]))
    got = json.loads((tmp_path / "c.json").read_text())
    assert set(got) == set(ref) and got["command"] == "certify"
    assert got["rank"] == ref["rank"]
    assert got["f_bound"] == pytest.approx(ref["f_bound"], rel=1e-9)
    assert got["e_norm"] < 1e-5 and ref["e_norm"] < 1e-5  # same verdict: certified


def test_write_decomposition_streams_what_report_holds(tmp_path):
    import paper_1702_02241_b200 as api
    from paper_1702_02241_b200.matrixio import read_matrix, write_decomposition
    from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse

    x, _, _ = gen_low_rank_plus_sparse(300, 200, 3, 0.05, 1e-3, seed=2)
    spec = api.ProblemSpec(x=x, lambda_l=2.0, lambda_s=0.1)
    rep = api.solve_split_spcp(spec, 4)
    nnz = write_decomposition(rep, tmp_path / "l.bin", tmp_path / "s.bin")
    assert read_matrix(tmp_path / "l.bin").tobytes() == rep.l.tobytes()
    assert read_matrix(tmp_path / "s.bin").tobytes() == rep.s.tobytes()
    assert nnz == int(np.count_nonzero(rep.s))
    assert write_decomposition(rep) == nnz


def test_column_shards_read_from_file_match_unsharded(torch, tmp_path):
    """Each rank of the column-sharded mode reads only its own
    X / mask columns from the SLRM files (`col0` / `cols` windows, streamed to
    HBM) and the partial -> all-reduce (by hand, one GPU) -> finish evaluation
    matches the unsharded problem read whole."""
    from paper_1702_02241_b200._lib import SPCP_F32
    from paper_1702_02241_b200.device import DeviceProblem
    from paper_1702_02241_b200.matrixio import read_mask, read_matrix, write_matrix

    rng = np.random.default_rng(77)
    m, n, k = 900, 1000, 12
    x = rng.standard_normal((m, n)).astype(np.float32).astype(np.float64) * 2.0
    mask = rng.random((m, n)) < 0.6
    write_matrix(x, tmp_path / "x.bin")
    write_matrix(mask.astype(float), tmp_path / "m.bin")
    ll, ls = 1.3, 0.3
    full = DeviceProblem(read_matrix(tmp_path / "x.bin", device="cuda", dtype=torch.float32),
                         ll, ls, mask=read_mask(tmp_path / "m.bin", device="cuda"))
    z = torch.from_numpy(rng.standard_normal((m + n) * k) / np.sqrt(k)).cuda()
    dz = torch.from_numpy(rng.standard_normal((m + n) * k) * 1e-2).cuda()
    g_full = torch.empty_like(z)
    out_full = full.eval(k, SPCP_F32, z, dz, 0.25, g_full)
    parts = []
    for c0, c1 in ((0, 384), (384, 700), (700, n)):
        xs = read_matrix(tmp_path / "x.bin", device="cuda", dtype=torch.float32, col0=c0,
                         cols=c1 - c0)
        ms = read_mask(tmp_path / "m.bin", device="cuda", col0=c0, cols=c1 - c0)
        dp = DeviceProblem(xs, ll, ls, mask=ms, n_total=n, col0=c0)
        zs = torch.cat([z[: m * k], z[m * k + c0 * k: m * k + c1 * k]])
        dzs = torch.cat([dz[: m * k], dz[m * k + c0 * k: m * k + c1 * k]])
        gu = torch.empty((m, k), dtype=torch.float32, device="cuda")
        scal = torch.empty(4, dtype=torch.float64, device="cuda")
        gs = torch.empty_like(zs)
        dp.eval_partial(k, SPCP_F32, zs, dzs, 0.25, gu, scal, gs)
        parts.append((dp, zs, dzs, gu, scal, gs, c0, c1))
    gu_sum = sum(pt[3].double() for pt in parts).float()
    scal_sum = sum(pt[4] for pt in parts)
    for dp, zs, dzs, _, _, gs, c0, c1 in parts:
        out = dp.eval_finish(k, SPCP_F32, zs, dzs, 0.25, gu_sum, scal_sum, gs)
        assert out[0] == pytest.approx(out_full[0], rel=1e-5)
        assert rel(gs[: m * k].cpu().numpy(), g_full[: m * k].cpu().numpy()) <= 1e-5
        assert rel(gs[m * k:].cpu().numpy(),
                   g_full[m * k + c0 * k: m * k + c1 * k].cpu().numpy()) <= 1e-5


def test_csv_device_read_and_decomposition_csv_outputs(torch, tmp_path):
    """CSV files take the host parser and are uploaded (read_matrix(device=));
    CSV decomposition outputs go through the device-materialised arrays."""
    import paper_1702_02241_b200 as api
    from paper_1702_02241_b200.matrixio import read_matrix, write_decomposition, write_matrix
    from paper_1702_02241_b200.synth import gen_low_rank_plus_sparse

    x, _, _ = gen_low_rank_plus_sparse(50, 40, 2, 0.05, 1e-3, seed=4)
    write_matrix(x, tmp_path / "x.csv")
    t = read_matrix(tmp_path / "x.csv", device="cuda")
    assert t.is_cuda and t.cpu().numpy().tobytes() == read_matrix(tmp_path / "x.csv").tobytes()
    np.testing.assert_array_equal(
        read_matrix(tmp_path / "x.csv", device="cuda", col0=5, cols=7).cpu().numpy(), x[:, 5:12])
    spec = api.ProblemSpec(x=t, lambda_l=1.0, lambda_s=0.1)
    rep = api.solve_split_spcp(spec, 3)
    nnz = write_decomposition(rep, tmp_path / "l.csv", tmp_path / "s.bin")
    np.testing.assert_array_equal(read_matrix(tmp_path / "l.csv"), rep.l)
    assert read_matrix(tmp_path / "s.bin").tobytes() == rep.s.tobytes()
    assert nnz == int(np.count_nonzero(rep.s))


def test_video_background_subtraction(torch):
    """The background-subtraction use (BASELINE C3 shape, small): the device
    video generator's static + illumination background is recovered as L and
    the moving objects as the support of S; the result matches the numpy
    oracle run on the same frames."""
    import paper_1702_02241_b200 as api
    from oracle import spcp_oracle as orc

    x, l_ref, fg = api.gen_video_device(48, 36, 200, fg_size=(8, 6), n_objects=2, seed=0,
                                        dtype="float64")
    assert torch.linalg.matrix_rank(l_ref).item() == 3
    spec = api.ProblemSpec(x=x, lambda_l=1.0, lambda_s=0.05)
    rep = api.solve_split_spcp(spec, 3, api.SolverConfig(grad_tol=1e-6))
    xh, lh, fgh = x.cpu().numpy(), l_ref.cpu().numpy(), fg.cpu().numpy()
    moved = np.abs(xh - lh) > 0.1  # object pixels that differ from the background
    s_on = rep.s != 0
    assert s_on[moved].mean() > 0.99
    assert (s_on & ~fgh).mean() < 1e-3
    assert rel(rep.l, lh) < 0.02
    ref = orc.solve_split_spcp(xh, 1.0, 0.05, 3, grad_tol=1e-6, max_iter=500)
    assert rel(rep.l, ref["l"]) < 1e-4 and rel(rep.s, ref["s"]) < 1e-4


def test_reference_solver_drives_the_c_abi_plugin():
    """The drop-in boundary seen from the reference side:
    the UNMODIFIED reference L-BFGS (`spcp.solver.lbfgs_minimize` from
    baseline/_ref, installed by build()) drives `spcp_split_objective_host`
    (fp64 mode) as its plug-in `fun(z) -> (f, grad)`, and reaches the same
    iterates, termination and objective as with its own numpy objective."""
    import importlib
    import os
    import sys

    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "spcp")):
        pytest.skip("reference package not installed in baseline/_ref (run build())")
    sys.path.insert(0, ref_dir)
    try:
        spcp = importlib.import_module("spcp")
        ref_solver = importlib.import_module("spcp.solver")
    finally:
        sys.path.remove(ref_dir)
    from paper_1702_02241_b200._lib import SPCP_F64
    from paper_1702_02241_b200.device import DeviceProblem

    x, _, _ = spcp.gen_low_rank_plus_sparse(300, 200, 4, 0.05, 1e-3, seed=11)
    spec = spcp.ProblemSpec(x=x, lambda_l=2.0, lambda_s=0.1)
    m, n, k = 300, 200, 5
    start = spcp.init_factors(spec, k, strategy="rsvd", seed=0)
    cfg = spcp.SolverConfig(grad_tol=1e-6, max_iter=300)
    dp = DeviceProblem(x, 2.0, 0.1, store=("f64",))

    def gpu_fun(z):
        u = z[: m * k].reshape(m, k)
        v = z[m * k:].reshape(n, k)
        f, gu, gv = dp.split_objective_host(u, v, SPCP_F64)
        return f, np.concatenate([gu.ravel(), gv.ravel()])

    own = ref_solver.lbfgs_minimize(ref_solver._flat_split_objective(spec, m, n, k), start, cfg)
    ours = ref_solver.lbfgs_minimize(gpu_fun, start, cfg)
    assert own.termination == "converged" and ours.termination == "converged"
    assert ours.objective == pytest.approx(own.objective, rel=1e-10)
    # same trajectory (the stopping iteration may differ by one at the threshold)
    assert abs(len(ours.iterations) - len(own.iterations)) <= 1
    for a, b in zip(ours.iterations, own.iterations):
        assert a.objective == pytest.approx(b.objective, rel=1e-9)
    assert rel(ours.factors.compose(), own.factors.compose()) < 1e-5
