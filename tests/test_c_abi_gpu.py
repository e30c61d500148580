"""The C ABI from C: examples/c_abi_example.c is compiled with gcc against
include/tacsl_b200.h and libtacsl_b200.so (no Python in the loop) and checks
closed-form answers (flat depth -> background colour, also at every level
of the K7 pyramid; a 1 mm press on a plane -> |f_n| = 1 N; the
resolution-mismatch and invalid-query status codes)."""
import shutil
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_c_abi_example(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "c_abi_example"
    lib_dir = ROOT / "paper_2408_06506_b200"
    cmd = ["gcc", "-O2", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
           str(ROOT / "examples" / "c_abi_example.c"), "-L", str(lib_dir), "-ltacsl_b200",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("ok"), out.stdout
    assert "0 of" in out.stdout
    assert "pyramid: 0 channel values differ" in out.stdout
