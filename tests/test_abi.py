"""The C-ABI library loads and exports exactly what include/tacsl_b200.h
declares; argument validation paths that need no GPU.  CPU only."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2408_06506_b200 import _lib, build
from paper_2408_06506_b200.errors import LutResolutionMismatch

HEADER = Path(__file__).resolve().parent.parent / "include" / "tacsl_b200.h"


def declared_symbols():
    return sorted(set(re.findall(r"TACSL_API\s+[\w\s\*]+?\b(tacsl_\w+)\s*\(", HEADER.read_text())))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for name in ("tacsl_depth_to_rgb", "tacsl_force_field", "tacsl_query_sdf", "tacsl_penalty_forces",
                 "tacsl_net_wrench", "tacsl_to_uint8", "tacsl_lut_create", "tacsl_sdf_create"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_abi_version(lib):
    assert lib.tacsl_abi_version() == _lib.ABI_VERSION


def test_lut_handle_and_validation(lib):
    c = np.zeros((3, 6))
    h = ctypes.c_void_p()
    assert lib.tacsl_lut_create(c.ctypes.data, 2, 80, 60, ctypes.byref(h)) == 0
    # resolution mismatch is detected before any device work
    rc = lib.tacsl_depth_to_rgb(h, None, 1, 61, 80, None, None, None)
    assert rc == 3
    with pytest.raises(LutResolutionMismatch):
        _lib.check(rc)
    assert lib.tacsl_depth_to_rgb(h, None, 1, 60, 80, None, None, None) == 1  # no output buffer
    lib.tacsl_lut_destroy(h)
    c5 = np.zeros((3, 21))
    rc = lib.tacsl_lut_create(c5.ctypes.data, 5, 80, 60, ctypes.byref(h))
    assert rc == 1 and "degree" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_penalty_validation(lib):
    rc = lib.tacsl_penalty_forces(None, None, None, None, 0, _lib.Penalty(-1.0, 0, 0, 0), None, None, None)
    assert rc == 1


def test_no_device_here_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert lib.tacsl_device_supported(0) == 0
    from paper_2408_06506_b200 import render
    with pytest.raises(RuntimeError):
        render.depth_to_rgb(np.zeros((60, 80), np.float32), render.synthetic_lut((80, 60)))
