"""compute-sanitizer over every kernel family (SURVEY 4 layer 5, 5 "race
detection"): memcheck (out-of-bounds / misaligned accesses), racecheck
(shared-memory hazards: the encoder's phased byte stores, the decoders'
staging buffers), synccheck (barrier misuse: __syncwarp masks) and initcheck
(reads of uninitialised global memory) on config c1 and odd fuzz shapes
(scripts/sanitize_step.py, which also checks every result against the
oracle)."""
import os
import shutil
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer_clean(tool):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", "--print-limit", "20"]
    if tool == "initcheck":
        cmd += ["--track-unused-memory", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "scripts", "sanitize_step.py")]
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env)
    tail = (r.stdout[-3000:] + "\n" + r.stderr[-3000:])
    if "compute-sanitizer is closed" in tail:
        # the GPU pool's wrapper refuses the tool (runs under it left GPUs
        # needing a reset); the same workload with guard-zone and oracle checks
        # runs in test_guarded_sanitize_step below
        pytest.skip("compute-sanitizer refused by this GPU pool")
    assert r.returncode == 0, tail
    assert "SANITIZE_STEP OK" in r.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr, tail


def test_guarded_sanitize_step():
    # without the sanitizer: every output of scripts/sanitize_step.py sits
    # between guard zones whose pattern must survive (out-of-bounds writes),
    # every result equals the oracle, and no CUDA error is raised
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_step.py")], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "SANITIZE_STEP OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
