"""Matrix files: headerless CSV and the SLRM binary container
(spcp matrixio.py:1-136), with a device path that streams straight to HBM.

Host API, same names / arguments / errors as the reference:
`read_matrix(path, fmt=None)` -> float64 ndarray, `write_matrix(a, path,
fmt=None)`, `write_json_atomic(obj, path)`.  The format is inferred from the
extension (".csv" -> CSV, anything else -> binary, matrixio.py:32-37); binary
round trips are bit-exact; writes are atomic (temp file + rename); reads raise
`MalformedHeaderError`, `TruncatedPayloadError`, `NonFiniteDataError` or
`MatrixIOError` (each with its `code`), and `FileNotFoundError` for a missing
file.

B200 additions (keyword-only, the reference has no device):
* `read_matrix(path, device="cuda", dtype=torch.float32)` returns a CUDA
  tensor; binary files go disk -> pinned double buffer -> HBM through
  `spcp_slrm_read_device` (no m x n host array; the dtype conversion and the
  NaN/Inf check run on the device).  `col0` / `cols` read one column shard
  (SURVEY §8(e)).
* `write_matrix` of a CUDA tensor streams HBM -> file (`spcp_slrm_write_device`).
* `write_decomposition(report, l_path, s_path)` writes the solver's L and S
  by materialising them chunk by chunk on the device (`spcp_slrm_write_product`)
  and returns nnz(S) for the CLI trace (cli.py:264-270).
"""

import json
import os
import struct
import tempfile

import numpy as np

from .errors import (
    MalformedHeaderError,
    MatrixIOError,
    NonFiniteDataError,
    TruncatedPayloadError,
)
from .validation import as_matrix

__all__ = ["read_matrix", "write_matrix", "write_json_atomic", "read_mask", "slrm_shape",
           "write_decomposition", "FORMATS", "MAGIC", "VERSION"]

MAGIC = b"SLRM"
VERSION = 1
_HDR = struct.Struct("<4sIQQ")  # magic, version, rows, cols (matrixio.py:25-27)
FORMATS = ("csv", "binary")


def _fmt_of(path, fmt):
    """Explicit format or the extension rule of matrixio.py:32-37."""
    if fmt is None:
        return "csv" if str(path).endswith(".csv") else "binary"
    if fmt not in FORMATS:
        raise ValueError(f"unknown matrix format {fmt!r}; expected one of {FORMATS}")
    return fmt


def _replace_atomically(path, fill):
    """Write through a temp file in the target directory, then rename
    (matrixio.py:40-50); the temp file never survives a failure."""
    folder = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(dir=folder, prefix=".tmp-", suffix=".part")
    try:
        with os.fdopen(fd, "wb") as fh:
            fill(fh)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _is_cuda_tensor(a):
    return type(a).__module__.startswith("torch") and getattr(a, "is_cuda", False)


# ------------------------------------------------------------------ headers
def slrm_shape(path):
    """(rows, cols) of an SLRM file after validating header and payload length
    (matrixio.py:94-109) — the native check shared by the host and device
    readers."""
    import ctypes

    from ._lib import check, lib

    r, c = ctypes.c_int64(), ctypes.c_int64()
    check(lib.spcp_slrm_header(os.fsencode(str(path)), ctypes.byref(r), ctypes.byref(c)))
    return int(r.value), int(c.value)


def _host_binary(path):
    rows, cols = slrm_shape(path)
    with open(path, "rb") as fh:
        fh.seek(_HDR.size)
        data = np.fromfile(fh, dtype="<f8", count=rows * cols)
    if data.size != rows * cols:  # file shrank between the check and the read
        raise TruncatedPayloadError(f"{path}: payload has {data.size * 8} bytes, "
                                    f"expected {rows * cols * 8}")
    return np.ascontiguousarray(data.reshape(rows, cols), dtype=np.float64)


def _host_csv(path):
    table, width = [], None
    with open(path, "r", encoding="ascii") as fh:
        for no, raw in enumerate(fh, start=1):
            text = raw.strip()
            if not text:
                continue
            cells = text.split(",")
            if width is None:
                width = len(cells)
            if len(cells) != width:
                raise MatrixIOError(f"{path}: line {no} has {len(cells)} fields, expected {width}")
            try:
                table.append([float(c) for c in cells])
            except ValueError as exc:
                raise MatrixIOError(f"{path}: line {no}: {exc}") from exc
    if not table:
        raise MatrixIOError(f"{path}: empty CSV matrix")
    return np.array(table, dtype=np.float64)


# ------------------------------------------------------------------ reading
def read_matrix(path, fmt=None, *, device=None, dtype=None, col0=0, cols=None):
    """Read a matrix file, rejecting NaN/Inf (matrixio.py:116-126).

    Without `device`: a float64 ndarray, exactly the reference's result.
    With `device` (a CUDA device): a CUDA tensor of `dtype` (default float64),
    binary payloads streamed to HBM by the native reader; `col0`/`cols`
    select a column window (one rank's shard).
    """
    fmt = _fmt_of(path, fmt)
    if device is None:
        a = _host_csv(path) if fmt == "csv" else _host_binary(path)
        if not np.isfinite(a).all():
            raise NonFiniteDataError(f"{path}: matrix contains NaN or Inf entries")
        if col0 or cols is not None:
            a = np.ascontiguousarray(a[:, col0:None if cols is None else col0 + cols])
        return a
    import torch

    dtype = torch.float64 if dtype is None else dtype
    dev = torch.device(device)
    if fmt == "csv":  # text parse is host work; upload the parsed window
        a = read_matrix(path, "csv", col0=col0, cols=cols)
        return torch.from_numpy(a).to(device=dev, dtype=dtype)
    return _device_read(path, dev, dtype, col0, cols)


def _device_read(path, dev, dtype, col0=0, cols=None, mask=False):
    import ctypes

    import torch

    from ._lib import SPCP_F32, SPCP_F64, SPCP_U8, check, lib
    from .device import cuda_device

    cuda_device()  # DeviceError without a GPU: no host fallback
    rows, ncol = slrm_shape(path)
    cols = ncol - col0 if cols is None else int(cols)
    if mask:
        code, tdt = SPCP_U8, torch.uint8
    elif dtype == torch.float32:
        code, tdt = SPCP_F32, torch.float32
    elif dtype == torch.float64:
        code, tdt = SPCP_F64, torch.float64
    else:
        raise ValueError(f"device reads produce float32 or float64, got {dtype}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.empty((rows, max(cols, 0)), dtype=tdt, device=dev)
    stream = torch.cuda.current_stream(dev)
    check(lib.spcp_slrm_read_device(os.fsencode(str(path)), dev.index, 0, rows, int(col0),
                                    cols, ctypes.c_void_p(out.data_ptr()), code,
                                    max(cols, 1), ctypes.c_void_p(stream.cuda_stream)))
    return out


def read_mask(path, fmt=None, *, device=None, col0=0, cols=None):
    """Observation mask file -> bool ndarray, nonzero = observed
    (cli.py:165-167).  With `device` the payload is converted on the GPU and
    only the 1-byte mask crosses back to the host."""
    fmt = _fmt_of(path, fmt)
    if device is None or fmt == "csv":
        return read_matrix(path, fmt, col0=col0, cols=cols) != 0.0
    import torch

    m8 = _device_read(path, torch.device(device), None, col0, cols, mask=True)
    return m8.cpu().numpy().astype(bool)


# ------------------------------------------------------------------ writing
def write_matrix(a, path, fmt=None):
    """Write a matrix as CSV or SLRM binary (matrixio.py:53-71).  A CUDA
    tensor is streamed from HBM (binary) without a host copy of the whole
    matrix."""
    fmt = _fmt_of(path, fmt)
    if _is_cuda_tensor(a):
        if a.dim() != 2:
            from .errors import DimensionError

            raise DimensionError(f"matrix must be a 2-D matrix, got ndim={a.dim()}")
        if fmt == "binary":
            return _device_write(a, path)
        a = a.detach().cpu().numpy()
    a = as_matrix(a, "matrix")
    if fmt == "csv":

        def fill(fh):
            for row in a:
                fh.write(",".join(format(v, ".17g") for v in row).encode("ascii") + b"\n")
    else:

        def fill(fh):
            fh.write(_HDR.pack(MAGIC, VERSION, a.shape[0], a.shape[1]))
            fh.write(a.astype("<f8", copy=False).tobytes())

    _replace_atomically(path, fill)


def _device_write(t, path):
    import ctypes

    import torch

    from ._lib import SPCP_F32, SPCP_F64, check, lib

    if t.dtype not in (torch.float32, torch.float64):
        t = t.double()
    if not bool(torch.isfinite(t).all()):
        raise ValueError("matrix contains NaN or Inf entries")
    if t.stride(1) != 1:
        t = t.contiguous()
    code = SPCP_F32 if t.dtype == torch.float32 else SPCP_F64
    stream = torch.cuda.current_stream(t.device)
    check(lib.spcp_slrm_write_device(os.fsencode(os.path.abspath(str(path))), t.device.index,
                                     ctypes.c_void_p(t.data_ptr()), code, t.shape[0],
                                     t.shape[1], max(t.stride(0), t.shape[1], 1),
                                     ctypes.c_void_p(stream.cuda_stream)))


def write_decomposition(report, l_path=None, s_path=None, fmt=None):
    """Write a split solve's L and S (cli.py:256-259) and return nnz(S)
    (cli.py:268).  Binary outputs are materialised on the device in row chunks
    and streamed to disk; CSV goes through the (device-materialised) dense
    arrays."""
    handle = getattr(report, "device_state", None)
    fl = _fmt_of(l_path, fmt) if l_path else None
    fs = _fmt_of(s_path, fmt) if s_path else None
    if handle is None or "csv" in (fl, fs):
        if l_path:
            write_matrix(report.l, l_path, fmt=fmt)
        s = report.s
        if s_path:
            write_matrix(s, s_path, fmt=fmt)
        return int(np.count_nonzero(s))
    import ctypes

    from ._lib import check, lib
    from .device import dptr

    dp, k, z = handle
    nnz = ctypes.c_int64()
    enc = (lambda p: None if p is None else os.fsencode(os.path.abspath(str(p))))
    check(lib.spcp_slrm_write_product(dp.h, int(k), dptr(z), enc(l_path), enc(s_path),
                                      ctypes.byref(nnz)))
    return int(nnz.value)


def write_json_atomic(obj, path):
    """JSON (indent 2, sorted keys, trailing newline) via temp file + rename
    (matrixio.py:128-136)."""

    def fill(fh):
        fh.write(json.dumps(obj, indent=2, sort_keys=True).encode("utf-8") + b"\n")

    _replace_atomically(path, fill)
