"""ctypes binding of libspcp_b200.so (the C ABI declared in include/spcp_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` / `make`.
There is no fallback: if the library is missing or does not export the ABI,
importing the compute path raises immediately.
"""

import ctypes
import os

from .errors import (
    DeviceError,
    DimensionError,
    MalformedHeaderError,
    MatrixIOError,
    NonFiniteDataError,
    NumericalError,
    TruncatedPayloadError,
)

__all__ = ["lib", "check", "LIB_PATH", "SPCP_F32", "SPCP_F64", "SPCP_U8", "STORE_F32",
           "STORE_F64", "STORE_SPARSE", "STORE_DENSE", "EXPORTS"]

# SPCP_LIB_PATH: an alternative build of the same ABI (A/B timing tools only)
LIB_PATH = os.environ.get("SPCP_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libspcp_b200.so")

SPCP_OK, SPCP_ERR_VALUE, SPCP_ERR_DIMENSION, SPCP_ERR_NUMERICAL, SPCP_ERR_CUDA, \
    SPCP_ERR_UNSUPPORTED, SPCP_ERR_IO, SPCP_ERR_MALFORMED_HEADER, SPCP_ERR_TRUNCATED, \
    SPCP_ERR_NONFINITE, SPCP_ERR_NOT_FOUND = range(11)
SPCP_F32, SPCP_F64, SPCP_U8 = 0, 1, 2
STORE_F32, STORE_F64, STORE_SPARSE, STORE_DENSE = 1, 2, 4, 8

_i64, _i32, _u32 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint
_vp, _dp, _d = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_double
_pp = ctypes.POINTER(ctypes.c_void_p)

# name -> (argtypes); every function returns int status except the two noted
EXPORTS = {
    "spcp_abi_version": [],
    "spcp_last_error": [],
    "spcp_device_count": [ctypes.POINTER(_i32)],
    "spcp_problem_create": [_pp, _i32, _i64, _i64, _vp, _i64, _i32, _i32, _vp, _u32, _d, _d,
                            _i64, _i64, _vp],
    "spcp_problem_destroy": [_vp],
    "spcp_problem_set_stream": [_vp, _vp],
    "spcp_problem_info": [_vp, _dp],
    "spcp_eval": [_vp, _i64, _i32, _vp, _vp, _d, _vp, _dp],
    "spcp_eval_async": [_vp, _i64, _i32, _vp, _vp, _d, _vp, _vp],
    "spcp_eval_partial": [_vp, _i64, _i32, _vp, _vp, _d, _vp, _vp, _vp],
    "spcp_eval_finish": [_vp, _i64, _i32, _vp, _vp, _d, _vp, _vp, _vp, _dp],
    "spcp_split_objective_host": [_vp, _i64, _i32, _vp, _vp, _dp, _vp, _vp],
    "spcp_phi_dense_host": [_vp, _vp, _dp, _vp, _vp],
    "spcp_apply": [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp],
    "spcp_apply_f32": [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp],
    "spcp_materialize": [_vp, _i64, _vp, _i64, _i64, _vp, _vp, _i32],
    "spcp_materialize_grad": [_vp, _i64, _vp, _vp, _i64],
    "spcp_grad_store": [_vp, _i64, _vp, _i32],
    "spcp_apply_stored": [_vp, _i64, _vp, _vp, _vp, _vp],
    "spcp_grad_release": [_vp],
    "spcp_workspace_trim": [_vp],
    "spcp_line_setup": [_vp, _i64, _vp, _vp],
    "spcp_line_probe": [_vp, _d, _dp],
    "spcp_line_release": [_vp],
    "spcp_vec_multidot": [_vp, _i64, _i32, _pp, _pp, _dp],
    "spcp_vec_lincomb": [_vp, _i64, _i32, _dp, _pp, _vp],
    "spcp_vec_gram": [_vp, _i64, _i32, _pp, _i32, _pp, _dp],
    "spcp_vec_gram_dev": [_vp, _i64, _i32, _pp, _i32, _pp, _vp],
    "spcp_gram": [_vp, _i64, _i64, _vp, _i64, _vp, _dp],
    "spcp_matmul_small": [_vp, _i64, _i64, _vp, _i64, _dp, _vp],
    "spcp_prof_enable": [_vp, _i32],
    "spcp_prof_read": [_vp, _dp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "spcp_slrm_header": [ctypes.c_char_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "spcp_slrm_read_device": [ctypes.c_char_p, _i32, _i64, _i64, _i64, _i64, _vp, _i32, _i64,
                              _vp],
    "spcp_slrm_write_device": [ctypes.c_char_p, _i32, _vp, _i32, _i64, _i64, _i64, _vp],
    "spcp_slrm_write_product": [_vp, _i64, _vp, ctypes.c_char_p, ctypes.c_char_p,
                                ctypes.POINTER(_i64)],
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make` (there is no CPU fallback for the compute path)")
    so = ctypes.CDLL(LIB_PATH)
    for name, argtypes in EXPORTS.items():
        fn = getattr(so, name)  # AttributeError = ABI mismatch: fail loudly
        fn.argtypes = argtypes
        fn.restype = ctypes.c_char_p if name == "spcp_last_error" else ctypes.c_int
    if so.spcp_abi_version() != 1:
        raise ImportError("libspcp_b200.so ABI version mismatch")
    return so


lib = _load()


def check(rc):
    """Map a C status to the reference's exception types."""
    if rc == SPCP_OK:
        return
    msg = (lib.spcp_last_error() or b"").decode(errors="replace")
    if rc == SPCP_ERR_DIMENSION:
        raise DimensionError(msg)
    if rc in (SPCP_ERR_VALUE, SPCP_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == SPCP_ERR_CUDA:
        raise DeviceError(msg)
    if rc == SPCP_ERR_NOT_FOUND:
        raise FileNotFoundError(msg)
    io = {SPCP_ERR_IO: MatrixIOError, SPCP_ERR_MALFORMED_HEADER: MalformedHeaderError,
          SPCP_ERR_TRUNCATED: TruncatedPayloadError, SPCP_ERR_NONFINITE: NonFiniteDataError}
    if rc in io:
        raise io[rc](msg)
    raise NumericalError(msg)
