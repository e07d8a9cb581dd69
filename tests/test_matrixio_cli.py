"""Matrix files and the command line (spcp matrixio.py, cli.py; SURVEY §8(f)
row 2) — the host-side half, on the CPU.

Pinned to `tests/golden/io.npz`, written by the REAL reference
(`make_golden.py gen_io`): the bytes its writer produces for awkward and
random matrices, and the files its `synth` command writes.  The cases follow
the reference's own tests (`tests/test_matrixio.py`, `tests/test_cli.py`):
bit-exact binary round trips, each malformed-input error with its `code`,
CSV rules, atomic writes, and exit codes 1 for usage / I/O errors.  The
native header check (`spcp_slrm_header`) runs here too — it makes no CUDA
call.
"""

import io
import json
import os
import struct
from contextlib import redirect_stderr, redirect_stdout

import numpy as np
import pytest

from paper_1702_02241_b200 import (
    MalformedHeaderError,
    MatrixIOError,
    NonFiniteDataError,
    TruncatedPayloadError,
)
from paper_1702_02241_b200 import cli
from paper_1702_02241_b200.matrixio import (
    read_mask,
    read_matrix,
    slrm_shape,
    write_json_atomic,
    write_matrix,
)


def _run(argv):
    out, err = io.StringIO(), io.StringIO()
    with redirect_stdout(out), redirect_stderr(err):
        try:
            code = cli.main(argv)
        except SystemExit as exc:
            code = exc.code
    return code, out.getvalue(), err.getvalue()


# ------------------------------------------------------------ writer bytes
@pytest.mark.parametrize("tag", ["awk", "rnd"])
@pytest.mark.parametrize("ext", ["bin", "csv"])
def test_writer_bytes_match_reference(tmp_path, golden, tag, ext):
    d = golden("io")
    path = tmp_path / f"m.{ext}"
    write_matrix(d[f"{tag}_mat"], path)
    assert path.read_bytes() == d[f"{tag}_{ext}"].tobytes()


@pytest.mark.parametrize("tag", ["awk", "rnd"])
def test_binary_read_of_reference_bytes_is_bit_exact(tmp_path, golden, tag):
    d = golden("io")
    path = tmp_path / "m.bin"
    path.write_bytes(d[f"{tag}_bin"].tobytes())
    assert read_matrix(path).tobytes() == d[f"{tag}_mat"].tobytes()
    assert slrm_shape(path) == d[f"{tag}_mat"].shape


def test_csv_read_of_reference_bytes(tmp_path, golden):
    d = golden("io")
    path = tmp_path / "m.csv"
    path.write_bytes(d["rnd_csv"].tobytes())
    np.testing.assert_array_equal(read_matrix(path), d["rnd_mat"])


def test_empty_binary_matrix_round_trips(tmp_path):
    path = tmp_path / "e.bin"
    write_matrix(np.zeros((0, 4)), path)
    assert read_matrix(path).shape == (0, 4)


# ------------------------------------------------------------ binary errors
def test_bad_magic(tmp_path):
    path = tmp_path / "m.bin"
    path.write_bytes(b"XXXX" + b"\0" * 20)
    with pytest.raises(MalformedHeaderError) as err:
        read_matrix(path)
    assert err.value.code == "malformed_header"


def test_short_header(tmp_path):
    path = tmp_path / "m.bin"
    path.write_bytes(b"SLRM\x01")
    with pytest.raises(MalformedHeaderError):
        read_matrix(path)


def test_bad_version(tmp_path):
    path = tmp_path / "m.bin"
    path.write_bytes(struct.pack("<4sIQQ", b"SLRM", 9, 1, 1) + b"\0" * 8)
    with pytest.raises(MalformedHeaderError):
        read_matrix(path)


def test_truncated_payload(tmp_path):
    path = tmp_path / "m.bin"
    write_matrix(np.random.default_rng(111).standard_normal((4, 4)), path)
    path.write_bytes(path.read_bytes()[:-9])
    with pytest.raises(TruncatedPayloadError) as err:
        read_matrix(path)
    assert err.value.code == "truncated_payload"


def test_non_finite_rejected(tmp_path):
    path = tmp_path / "m.bin"
    path.write_bytes(struct.pack("<4sIQQ", b"SLRM", 1, 1, 2) + struct.pack("<2d", 1.0, np.nan))
    with pytest.raises(NonFiniteDataError) as err:
        read_matrix(path)
    assert err.value.code == "non_finite_data"


def test_missing_file_is_file_not_found(tmp_path):
    with pytest.raises(FileNotFoundError):
        read_matrix(tmp_path / "nope.bin")
    with pytest.raises(FileNotFoundError):
        read_matrix(tmp_path / "nope.csv")


# ------------------------------------------------------------ CSV rules
@pytest.mark.parametrize("text,exc", [
    ("1,2\n3\n", MatrixIOError),
    ("1,foo\n", MatrixIOError),
    ("", MatrixIOError),
    ("1,nan\n", NonFiniteDataError),
])
def test_csv_rejections(tmp_path, text, exc):
    path = tmp_path / "m.csv"
    path.write_text(text)
    with pytest.raises(exc):
        read_matrix(path)


def test_csv_skips_blank_lines_and_round_trips(tmp_path):
    path = tmp_path / "m.csv"
    path.write_text("1,2\n\n3,4\n")
    np.testing.assert_array_equal(read_matrix(path), [[1.0, 2.0], [3.0, 4.0]])
    a = np.random.default_rng(112).standard_normal((5, 4)) * 1e-7
    write_matrix(a, path)
    np.testing.assert_array_equal(read_matrix(path), a)


def test_format_selection(tmp_path):
    a = np.array([[1.5, 2.5]])
    write_matrix(a, tmp_path / "a.csv")
    write_matrix(a, tmp_path / "a.mat")
    assert (tmp_path / "a.csv").read_bytes().startswith(b"1.5")
    assert (tmp_path / "a.mat").read_bytes().startswith(b"SLRM")
    write_matrix(a, tmp_path / "b.csv", fmt="binary")
    assert (tmp_path / "b.csv").read_bytes().startswith(b"SLRM")
    np.testing.assert_array_equal(read_matrix(tmp_path / "b.csv", fmt="binary"), a)
    with pytest.raises(ValueError):
        write_matrix(a, tmp_path / "c.bin", fmt="hdf5")


def test_failed_write_leaves_no_temp_file(tmp_path):
    target = tmp_path / "keep.bin"
    write_matrix(np.ones((2, 2)), target)
    before = target.read_bytes()
    with pytest.raises(ValueError):
        write_matrix(np.array([[1.0, np.inf]]), target)
    assert target.read_bytes() == before
    assert sorted(p.name for p in tmp_path.iterdir()) == ["keep.bin"]


def test_write_json_atomic_format(tmp_path):
    obj = {"b": [1, 2.5], "a": {"z": None, "y": "s"}}
    path = tmp_path / "t.json"
    write_json_atomic(obj, path)
    assert path.read_text() == json.dumps(obj, indent=2, sort_keys=True) + "\n"


def test_mask_file_nonzero_is_observed(tmp_path):
    path = tmp_path / "m.bin"
    write_matrix(np.array([[0.0, 1.0, -2.0], [0.5, 0.0, -0.0]]), path)
    np.testing.assert_array_equal(read_mask(path), [[False, True, True], [True, False, False]])


# ------------------------------------------------------------ CLI (no GPU)
def test_cli_synth_writes_reference_files(tmp_path, golden):
    d = golden("io")
    x, m = tmp_path / "x.bin", tmp_path / "m.bin"
    code, out, _ = _run(["synth", "--m", "80", "--n", "60", "--rank", "3", "--sparse-frac",
                         "0.05", "--noise-rel", "1e-3", "--seed", "0", "--output-x", str(x),
                         "--observe-frac", "0.6", "--output-mask", str(m)])
    assert code == 0 and out.startswith("synth: wrote 80x60 problem")
    assert x.read_bytes() == d["full_x"].tobytes()
    assert m.read_bytes() == d["mask_m"].tobytes()


def test_cli_synth_mask_needs_observe_frac(tmp_path):
    code, _, err = _run(["synth", "--m", "4", "--n", "3", "--rank", "1", "--output-x",
                         str(tmp_path / "x.bin"), "--output-mask", str(tmp_path / "m.bin")])
    assert code == 1 and "--observe-frac" in err


@pytest.mark.parametrize("argv", [
    [],
    ["decompose"],
    ["decompose", "--input", "x.bin", "--lambda-l", "1"],
    ["decompose", "--input", "x.bin", "--lambda-l", "1", "--lambda-s", "1", "--solver", "admm"],
    ["frobnicate"],
])
def test_cli_usage_errors_exit_1(argv):
    code, _, err = _run(argv)
    assert code == 1 and "error" in err


def test_cli_io_errors_exit_1(tmp_path):
    code, _, err = _run(["decompose", "--input", str(tmp_path / "none.bin"), "--lambda-l", "1",
                         "--lambda-s", "1"])
    assert code == 1 and "error" in err
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOPE" + b"\0" * 20)
    code, _, err = _run(["decompose", "--input", str(bad), "--lambda-l", "1", "--lambda-s", "1"])
    assert code == 1 and "[malformed_header]" in err
    code, _, err = _run(["certify", "--input", str(bad), "--lambda-l", "1", "--lambda-s", "1",
                         "--l", str(bad)])
    assert code == 1 and "[malformed_header]" in err


def test_cli_bad_certificate_mode_exit_1(tmp_path):
    x = tmp_path / "x.bin"
    write_matrix(np.ones((3, 3)), x)
    for mode in ("sometimes", "every:0"):
        code, _, err = _run(["decompose", "--input", str(x), "--lambda-l", "1", "--lambda-s",
                             "1", "--certificate", mode])
        assert code == 1 and "error" in err


def test_cli_out_of_scope_solvers_exit_1(tmp_path):
    x = tmp_path / "x.bin"
    write_matrix(np.ones((3, 3)), x)
    code, _, err = _run(["decompose", "--input", str(x), "--lambda-l", "1", "--lambda-s", "1",
                         "--solver", "prox"])
    assert code == 1 and "prox" in err
    code, _, _ = _run(["bench", "--input", str(x), "--lambda-l", "1", "--lambda-s", "1"])
    assert code == 1


def test_cli_threads_env(monkeypatch):
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        monkeypatch.delenv(var, raising=False)
    monkeypatch.setenv("SPCP_NUM_THREADS", "3")
    cli._threads_from_env()
    assert os.environ["OMP_NUM_THREADS"] == "3" and os.environ["OPENBLAS_NUM_THREADS"] == "3"


def test_certificate_attribute_is_the_function_after_submodule_import():
    import importlib
    import inspect

    importlib.import_module("paper_1702_02241_b200.certificate")
    import paper_1702_02241_b200 as api

    assert inspect.isfunction(api.certificate)
    assert api.certificate.__name__ == "certificate"
