"""The C ABI from plain C (examples/c_api_demo.c): compiled against
include/eqc.h and libeqc.so without Python or torch (CPU test), and run on a
GPU (composite + RLE round trip checked inside the program)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1902_08755_b200")


def _build(tmp_path):
    from paper_1902_08755_b200 import build
    build.build()
    exe = str(tmp_path / "c_api_demo")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", LIBDIR, "-l:libeqc.so", f"-Wl,-rpath,{LIBDIR}",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-o", exe]
    subprocess.check_call(cmd)
    return exe


def test_c_api_demo_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_api_demo_runs(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "composite ok" in r.stdout and "decode ok" in r.stdout
