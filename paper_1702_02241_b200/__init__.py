"""B200-native Split-SPCP (arXiv:1702.02241): the marginalised Burer-Monteiro
RPCA objective + gradient as one fused sm_100a streaming kernel, a
device-resident L-BFGS, the convergence certificate and a column-sharded
multi-GPU mode, behind the reference package's Python API
(`spcp/__init__.py:50-99`, split-solver subset).

The compute path is libspcp_b200.so (CUDA, sm_100a); importing a compute
entry point without the built library raises — there is no CPU fallback.
"""

import sys as _sys
import types as _types

from .errors import (
    DeviceError,
    DimensionError,
    MalformedHeaderError,
    MatrixIOError,
    NonFiniteDataError,
    NumericalError,
    PowerIterationError,
    SpcpError,
    TruncatedPayloadError,
)
from .report import IterateState, IterationRecord, SolveReport, WorkTimer
from .validation import as_mask, as_matrix, check_rank_bound

__version__ = "0.1.0"

_LAZY = {
    "ProblemSpec": "objective", "huber": "objective", "shrink": "objective",
    "phi_value_grad": "objective", "set_default_precision": "objective",
    "get_default_precision": "objective",
    "LbfgsResult": "lbfgs", "minimize_lbfgs": "lbfgs",
    "SvdTriplet": "linalg", "thin_qr": "linalg", "svd_small": "linalg", "rand_svd": "linalg",
    "leading_triple": "linalg",
    "FactorPair": "solver", "SolverConfig": "solver", "split_objective": "solver",
    "init_factors": "solver", "factors_from_dense": "solver", "lbfgs_minimize": "solver",
    "solve_split_spcp": "solver",
    "CertificateReport": "certificate", "certificate": "certificate",
    "factor_svd": "certificate",
    "SplitSPCP": "estimators",
    "gen_low_rank_plus_sparse_device": "synth", "gen_video_device": "synth",
    "gen_low_rank_plus_sparse": "synth", "gen_mask": "synth",
    "solve_split_spcp_sharded": "dist",
}

__all__ = sorted(list(_LAZY) + [
    "DeviceError", "DimensionError", "MalformedHeaderError", "MatrixIOError",
    "NonFiniteDataError", "NumericalError", "PowerIterationError", "SpcpError",
    "TruncatedPayloadError", "IterateState", "IterationRecord", "SolveReport", "WorkTimer",
    "as_mask", "as_matrix", "check_rank_bound"])


class _Package(_types.ModuleType):
    """The `certificate` submodule shares its name with the `certificate`
    function (the reference package exports the function); importing the
    submodule must not replace the package attribute with the module."""

    def __setattr__(self, name, value):
        if name == "certificate" and isinstance(value, _types.ModuleType):
            value = value.certificate
        super().__setattr__(name, value)


_sys.modules[__name__].__class__ = _Package


def __getattr__(name):
    # compute modules load libspcp_b200.so on first use (ImportError if unbuilt)
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib

    val = getattr(importlib.import_module(f"{__name__}.{mod}"), name)
    globals()[name] = val
    return val
