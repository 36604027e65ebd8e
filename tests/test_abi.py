"""CPU-side checks of the C-ABI boundary: the library exists, loads, and
exports every symbol include/ttb.h declares (no compute calls: no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ttb.h")


def declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(ttb_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("ttb_round", "ttb_inner", "ttb_orthonormalize", "ttb_add", "ttb_hadamard",
                 "ttb_tsqr_factor", "ttb_tsqr_apply", "ttb_truncated_svd", "ttb_ctx_create"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2011_06532_b200 import _lib
    if not os.path.exists(_lib.SO_PATH):
        from paper_2011_06532_b200 import build
        build.build()
    lib = ctypes.CDLL(_lib.SO_PATH)
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(_lib.SIGNATURES), "ctypes signature table out of sync with ttb.h"
    L = _lib.load()
    assert L.ttb_abi_version() == 1
    assert L.ttb_launch_counter() >= 0


def test_no_gpu_means_loud_failure():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2011_06532_b200 as T
    with pytest.raises(T.CapabilityError):
        T.default_comm()
