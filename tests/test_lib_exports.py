"""The C-ABI library loads and exports every symbol include/spcp_b200.h declares
(CPU-only: no compute calls)."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "spcp_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(spcp_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("spcp_problem_create", "spcp_eval", "spcp_eval_partial", "spcp_eval_finish",
                 "spcp_split_objective_host", "spcp_phi_dense_host", "spcp_apply",
                 "spcp_materialize", "spcp_vec_gram", "spcp_vec_lincomb"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_1702_02241_b200 import _lib

    so = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(so, s)]
    assert not missing, missing
    # and the Python binding binds exactly the declared set
    assert set(_lib.EXPORTS) == set(declared_symbols())


def test_abi_version_and_error_channel():
    from paper_1702_02241_b200._lib import lib

    assert lib.spcp_abi_version() == 1
    assert isinstance(lib.spcp_last_error(), bytes)


def test_library_is_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess

    from paper_1702_02241_b200 import _lib

    tool = shutil.which("cuobjdump")
    if tool is None:
        return
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
