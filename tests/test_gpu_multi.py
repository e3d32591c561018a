"""GPU parity of the multi-GPU schedules (direct send, binary swap).

* Virtual ranks on one GPU (compose_*_local, the P:1289-1292 trick of
  running a sort-last compound on channels of one GPU): the identical
  schedule code with device copies standing in for NCCL.
* Real NCCL over NVLink when >= 2 GPUs are visible: tests/mp_compose.py under
  torch.distributed.run (one process per GPU).
Both must equal the oracle over ALL sources bit-exactly (R-C5) and
send n(n-1) band messages + (n-1) gathers for direct send.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import out_frame, to_dev, to_host  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def eqc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1902_08755_b200 import eqc as m
    return m


CASES = [
    # (algo, nranks, n_local, w, h, pitch, out_pitch, dest, rle, gen)
    ("ds", 1, 3, 64, 33, None, None, 0, 0, "scene"),
    ("ds", 2, 2, 300, 41, None, None, 0, 0, "scene"),
    ("ds", 3, 1, 130, 31, 136, None, 2, 0, "ties"),
    ("ds", 4, 2, 257, 1081 // 8, None, 260, 1, 0, "scene"),
    ("ds", 8, 1, 128, 9, None, None, 5, 0, "ties"),
    ("ds", 2, 2, 300, 41, None, None, 1, 1, "scene"),
    ("ds", 4, 2, 257, 77, None, 264, 3, 1, "scene"),
    ("ds", 3, 3, 129, 20, 132, None, 0, 1, "ties"),
    ("bs", 1, 2, 64, 16, None, None, 0, 0, "scene"),
    ("bs", 2, 2, 300, 41, None, None, 0, 0, "scene"),
    ("bs", 4, 1, 130, 37, 136, 140, 2, 0, "ties"),
    ("bs", 8, 1, 128, 19, None, None, 7, 0, "scene"),
    ("bs", 4, 2, 257, 77, None, None, 1, 1, "scene"),
    ("bs", 8, 1, 96, 5, None, None, 0, 1, "ties"),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}_n{c[1]}x{c[2]}_{c[3]}x{c[4]}_rle{c[8]}" for c in CASES])
def test_virtual_rank_schedule_equals_oracle(eqc, case):
    algo, nr, nl, w, h, pitch, opitch, dest, rle, gen = case
    N = nr * nl
    if gen == "scene":
        c, d = synth.depth_sources(synth.SEED_BASE + 3 + N, N, w, h)
    else:
        c, d = synth.random_frames(N + w, N, w, h, depth_alphabet=[0, 2, 0xFFFFFFFF])
    want, _ = oracle.depth_composite(c, d)
    dc = [to_dev(x, pitch) for x in c]
    dd = [to_dev(x, pitch) for x in d]
    out = out_frame(h, w, opitch)
    fn = eqc.compose_direct_send_local if algo == "ds" else eqc.compose_binary_swap_local
    stats = fn(nr, dc, dd, out, dest_rank=dest, flags=eqc.FLAG_RLE if rle else 0)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out), want)
    if algo == "ds" and h >= nr:
        assert stats[0] == nr * (nr - 1)  # band messages
        assert stats[1] == nr - 1         # gathers
    if algo == "bs" and h >= 2 * nr:
        assert stats[0] == nr * (nr.bit_length() - 1)
    assert stats[2] == stats[3]  # every byte sent is received


BLEND_CASES = [
    # (algo, nranks, n_local, w, h, pitch, out_pitch, dest, rle, gen) -- EQC_OP_BLEND
    ("ds", 1, 4, 64, 33, None, None, 0, 0, "bricks"),
    ("ds", 2, 8, 320, 180, None, None, 0, 0, "bricks"),
    ("ds", 4, 4, 257, 77, None, 264, 3, 0, "bricks"),
    ("ds", 3, 2, 130, 31, 136, None, 1, 0, "noise"),
    ("ds", 4, 2, 257, 77, None, None, 2, 1, "bricks"),
    ("ds", 2, 3, 129, 20, 132, None, 1, 1, "noise"),
    ("bs", 2, 8, 320, 180, None, None, 1, 0, "bricks"),
    ("bs", 4, 2, 130, 37, 136, 140, 2, 0, "noise"),
    ("bs", 8, 2, 128, 19, None, None, 7, 0, "bricks"),
    ("bs", 4, 4, 257, 77, None, None, 0, 1, "bricks"),
]


@pytest.mark.parametrize("case", BLEND_CASES,
                         ids=[f"{c[0]}_n{c[1]}x{c[2]}_{c[3]}x{c[4]}_rle{c[8]}" for c in BLEND_CASES])
def test_virtual_rank_blend_within_one_lsb(eqc, case):
    # global draw order = rank-block order (rank 0 holds the back-most layers);
    # the result must match O2 over ALL layers within 1/255 (R-C4, R-C6)
    algo, nr, nl, w, h, pitch, opitch, dest, rle, gen = case
    N = nr * nl
    layers = synth.volume_bricks(synth.SEED_BASE + 70 + N, N, w, h) if gen == "bricks" else \
        synth.premultiplied_noise(synth.SEED_BASE + 71 + N, N, w, h)
    want = oracle.blend_ordered(layers)
    dl = [to_dev(x, pitch) for x in layers]
    out = out_frame(h, w, opitch)
    fn = eqc.compose_direct_send_local if algo == "ds" else eqc.compose_binary_swap_local
    fn(nr, dl, None, out, dest_rank=dest, flags=eqc.FLAG_RLE if rle else 0, op=eqc.OP_BLEND)
    torch.cuda.synchronize()
    got = to_host(out)
    diff = np.abs(got.view(np.uint8).astype(int) - want.view(np.uint8).astype(int))
    assert diff.max() <= 1, f"max channel error {diff.max()} LSB"


S23_CASES = [
    # (nranks, n_local, w, h, pitch, out_pitch, dest, rle, op) -- 2-3 swap (R-C21)
    (1, 2, 64, 16, None, None, 0, 0, "depth"),
    (3, 2, 300, 41, None, None, 1, 0, "depth"),
    (5, 1, 130, 37, 136, 140, 4, 0, "depth"),
    (6, 1, 128, 19, None, None, 2, 1, "depth"),
    (7, 2, 257, 77, None, 264, 3, 0, "depth"),
    (12, 1, 96, 50, None, None, 11, 1, "depth"),
    (3, 3, 320, 90, None, None, 0, 0, "blend"),
    (5, 2, 130, 37, 136, None, 2, 1, "blend"),
    (6, 2, 128, 19, None, None, 5, 0, "blend"),
]


@pytest.mark.parametrize("case", S23_CASES,
                         ids=[f"n{c[0]}x{c[1]}_{c[2]}x{c[3]}_rle{c[7]}_{c[8]}" for c in S23_CASES])
def test_virtual_rank_swap23(eqc, case):
    nr, nl, w, h, pitch, opitch, dest, rle, op = case
    N = nr * nl
    out = out_frame(h, w, opitch)
    flags = eqc.FLAG_RLE if rle else 0
    if op == "depth":
        c, d = synth.random_frames(N + w + 1, N, w, h, depth_alphabet=[0, 2, 0xFFFFFFFF]) if nr % 2 else \
            synth.depth_sources(synth.SEED_BASE + 3 + N, N, w, h)
        dc = [to_dev(x, pitch) for x in c]
        dd = [to_dev(x, pitch) for x in d]
        stats = eqc.compose_swap23_local(nr, dc, dd, out, dest_rank=dest, flags=flags)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(to_host(out), oracle.depth_composite(c, d)[0])
        assert stats[2] == stats[3]
    else:
        layers = synth.volume_bricks(synth.SEED_BASE + 90 + N, N, w, h)
        dl = [to_dev(x, pitch) for x in layers]
        eqc.compose_swap23_local(nr, dl, None, out, dest_rank=dest, flags=flags, op=eqc.OP_BLEND)
        torch.cuda.synchronize()
        want = oracle.blend_ordered(layers)
        diff = np.abs(to_host(out).view(np.uint8).astype(int) - want.view(np.uint8).astype(int))
        assert diff.max() <= 1


def test_binary_swap_rejects_non_power_of_two(eqc):
    c, d = synth.random_frames(1, 3, 8, 8)
    with pytest.raises(eqc.EqcError) as e:
        eqc.compose_binary_swap_local(3, [to_dev(x) for x in c], [to_dev(x) for x in d], out_frame(8, 8))
    assert e.value.code == eqc.E_UNSUPPORTED


@pytest.mark.parametrize("nproc", [2, 3, 4])
def test_nccl_multi_gpu(eqc, nproc):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mp_compose.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ALL OK" in r.stdout
