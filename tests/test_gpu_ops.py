"""GPU parity of the §8(f) f4 per-pixel operators and the streaming chain:
compositor_average (subpixel accumulation + averaging, bit-exact vs the
oracle), EQC_OP_AVERAGE through every schedule, and compose_stream (the
sort-last chain) for all three operators, on virtual ranks of one GPU."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import out_frame, to_dev, to_host  # noqa: E402


@pytest.fixture(scope="module")
def eqc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1902_08755_b200 import eqc as m
    return m


@pytest.mark.parametrize("n,w,h,pitch,offset", [(1, 64, 8, None, 0), (2, 3, 5, None, 0), (7, 129, 33, 136, 0),
                                                 (16, 640, 90, None, 0), (64, 37, 9, 40, 1)])
def test_compositor_average_bit_exact(eqc, n, w, h, pitch, offset):
    c, _ = synth.random_frames(400 + n, n, w, h)
    dc = [to_dev(x, pitch, offset) for x in c]
    out = out_frame(h, w, pitch, offset)
    eqc.compositor_average(dc, out)
    np.testing.assert_array_equal(to_host(out), oracle.average(c))


def test_compositor_average_exhaustive_rounding(eqc):
    # every sum 0 .. 255 n for n = 2, 3, 5, 64: one pixel per (sum) pattern
    for n in (2, 3, 5, 64):
        sums = np.arange(0, 255 * n + 1)
        w = len(sums)
        frames = []
        rem = sums.copy()
        for i in range(n):
            v = np.minimum(rem, 255)
            rem -= v
            frames.append(np.tile((v | (v << 8) | (v << 16) | (v << 24)).astype(np.uint32), (2, 1)))
        out = out_frame(2, w)
        eqc.compositor_average([to_dev(f) for f in frames], out)
        np.testing.assert_array_equal(to_host(out), oracle.average(frames))


SCHED = ["ds", "bs", "s23", "stream"]


def _fn(eqc, algo):
    return {"ds": eqc.compose_direct_send_local, "bs": eqc.compose_binary_swap_local,
            "s23": eqc.compose_swap23_local, "stream": eqc.compose_stream_local}[algo]


@pytest.mark.parametrize("algo,nr,nl,w,h,dest,rle", [
    ("ds", 3, 2, 130, 31, 1, 0), ("ds", 4, 2, 257, 40, 3, 1), ("bs", 4, 2, 130, 37, 2, 0),
    ("bs", 2, 8, 64, 16, 0, 1), ("s23", 5, 1, 129, 20, 4, 0), ("s23", 6, 2, 96, 33, 0, 1),
    ("stream", 1, 3, 64, 8, 0, 0), ("stream", 4, 2, 130, 31, 0, 0), ("stream", 3, 3, 257, 17, 1, 1),
])
def test_average_through_schedules(eqc, algo, nr, nl, w, h, dest, rle):
    N = nr * nl
    c, _ = synth.random_frames(500 + N + w, N, w, h)
    out = out_frame(h, w)
    _fn(eqc, algo)(nr, [to_dev(x) for x in c], None, out, dest_rank=dest, flags=eqc.FLAG_RLE if rle else 0,
                   op=eqc.OP_AVERAGE)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out), oracle.average(c))


@pytest.mark.parametrize("nr,nl,w,h,pitch,opitch,dest,rle", [
    (2, 2, 300, 41, None, None, 0, 0), (3, 1, 130, 31, 136, None, 2, 0), (4, 2, 257, 77, None, 264, 1, 1),
    (5, 1, 64, 9, None, None, 4, 1), (8, 1, 128, 19, None, None, 7, 0),
])
def test_stream_chain_depth(eqc, nr, nl, w, h, pitch, opitch, dest, rle):
    N = nr * nl
    c, d = synth.random_frames(N + w, N, w, h, depth_alphabet=[0, 2, 0xFFFFFFFF]) if nr % 2 else \
        synth.depth_sources(synth.SEED_BASE + 3 + N, N, w, h)
    out = out_frame(h, w, opitch)
    stats = eqc.compose_stream_local(nr, [to_dev(x, pitch) for x in c], [to_dev(x, pitch) for x in d], out,
                                     dest_rank=dest, flags=eqc.FLAG_RLE if rle else 0)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out), oracle.depth_composite(c, d)[0])
    assert stats[0] == nr - 1  # one whole-frame message per hop


@pytest.mark.parametrize("nr,nl,rle", [(2, 4, 0), (4, 4, 1), (3, 2, 0)])
def test_stream_chain_blend(eqc, nr, nl, rle):
    N, w, h = nr * nl, 320, 90
    layers = synth.volume_bricks(synth.SEED_BASE + 95 + N, N, w, h)
    out = out_frame(h, w)
    eqc.compose_stream_local(nr, [to_dev(x) for x in layers], None, out, dest_rank=0,
                             flags=eqc.FLAG_RLE if rle else 0, op=eqc.OP_BLEND)
    torch.cuda.synchronize()
    want = oracle.blend_ordered(layers)
    assert np.abs(to_host(out).view(np.uint8).astype(int) - want.view(np.uint8).astype(int)).max() <= 1


def test_average_rejects_too_many_sources(eqc):
    c, _ = synth.random_frames(1, 64, 8, 4)
    with pytest.raises(eqc.EqcError):  # 5 x 64 = 320 sources exceed the exact 16-bit sums
        eqc.compose_direct_send_local(5, [to_dev(x) for x in c] * 5, None, out_frame(4, 8), op=eqc.OP_AVERAGE)


@pytest.mark.parametrize("algo,nr,h", [("s23", 6, 2), ("s23", 5, 1), ("stream", 4, 1), ("ds", 5, 3), ("bs", 8, 3)])
def test_schedules_with_fewer_rows_than_parts(eqc, algo, nr, h):
    # more ranks / parts than rows: empty bands and regions must be handled
    w = 70
    c, d = synth.random_frames(700 + nr + h, nr, w, h, depth_alphabet=[0, 1, 0xFFFFFFFF])
    out = out_frame(h, w)
    _fn(eqc, algo)(nr, [to_dev(x) for x in c], [to_dev(x) for x in d], out, dest_rank=nr - 1)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out), oracle.depth_composite(c, d)[0])
    out2 = out_frame(h, w)
    _fn(eqc, algo)(nr, [to_dev(x) for x in c], None, out2, dest_rank=0, flags=eqc.FLAG_RLE, op=eqc.OP_AVERAGE)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out2), oracle.average(c))
