"""GPU parity of the peer-memory (NVLink P2P) transport on ONE GPU.

compose_direct_send_p2p_local / compose_binary_swap_p2p_local /
compose_direct_send_rle_pull_local run the
multi-process peer-memory host code and kernels for virtual ranks of one
process (their "peer mappings" are plain device pointers, every virtual rank
on its own stream): the plain peer-memory direct send, the pipelined variant
(pieces, progress counters in peer memory), frame slots read in place, the
computed-ROI variant, and the compressed direct send whose fused decode reads
every rank's streams in place for band j (compositor_depth_rle over a row
band with y0 > 0).  Async compositing pipeline and early assembly:
P:2302-2310; schedule P:1569-1589.  Each must equal the oracle
(O1 over ALL sources, R-C5) bit-exactly.  Also: a flag wait whose peer never
arrives gives up after EQC_P2P_TIMEOUT_MS and the call reports EQC_E_NCCL.
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


def _scene(N, w, h, seed, ties=False):
    if ties:
        return synth.random_frames(seed, N, w, h, depth_alphabet=[0, 2, 0xFFFFFFFF])
    return synth.depth_sources(seed, N, w, h)


P2P_CASES = [
    # (mode, nranks, n_local, w, h, pitch, out_pitch, dest, flags, gen)
    ("plain", 2, 2, 300, 41, None, None, 0, 0, "scene"),
    ("plain", 3, 1, 130, 31, 136, None, 2, 0, "ties"),
    ("plain", 4, 2, 257, 135, None, 260, 1, 0, "scene"),
    ("plain", 8, 1, 128, 9, None, None, 5, 0, "ties"),
    ("plain", 4, 3, 640, 360, None, None, 3, 0, "scene"),
    ("roi", 2, 2, 300, 41, None, None, 1, "roi", "scene"),
    ("roi", 4, 2, 513, 200, 516, None, 0, "roi", "scene"),
    ("pipelined", 2, 2, 300, 41, None, None, 0, 0, "scene"),
    ("pipelined", 4, 2, 257, 135, None, 264, 2, 0, "scene"),
    ("pipelined", 3, 3, 129, 20, 132, None, 1, 0, "ties"),
    ("slots", 2, 1, 300, 41, None, None, 1, 0, "scene"),
    ("slots", 4, 1, 640, 360, None, None, 0, 0, "scene"),
    ("slots", 3, 1, 130, 31, 136, 140, 2, 0, "ties"),
]


@pytest.mark.parametrize("case", P2P_CASES, ids=[f"{c[0]}_n{c[1]}x{c[2]}_{c[3]}x{c[4]}_d{c[7]}" for c in P2P_CASES])
def test_p2p_direct_send_virtual_ranks_equal_oracle(eqc, case):
    mode, nr, nl, w, h, pitch, opitch, dest, fl, gen = case
    N = nr * nl
    c, d = _scene(N, w, h, synth.SEED_BASE + 90 + N + w, ties=gen == "ties")
    want, _ = oracle.depth_composite(c, d)
    dc = [to_dev(x, pitch) for x in c]
    dd = [to_dev(x, pitch) for x in d]
    out = out_frame(h, w, opitch)
    m = {"plain": eqc.P2P_PLAIN, "roi": eqc.P2P_PLAIN, "pipelined": eqc.P2P_PIPELINED, "slots": eqc.P2P_SLOTS}[mode]
    flags = eqc.FLAG_ROI if fl == "roi" else 0
    stats = eqc.compose_direct_send_p2p_local(nr, dc, dd, out, dest_rank=dest, flags=flags, mode=m)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out), want)
    if h >= nr:
        assert stats[0] == nr * (nr - 1)  # band pulls
        assert stats[1] == nr - 1         # bands pushed to the destination


def test_p2p_pipelined_large_bands(eqc):
    # the size at which compose_direct_send itself picks the pipelined path
    # (>= 2 sources, >= 6 Mpx per band): 2 virtual ranks x 2 sources of
    # 3840x3400, checked on sampled rows + depth-min at every pixel
    nr, nl, w, h = 2, 2, 3840, 3400
    c, d = synth.depth_sources(synth.SEED_BASE + 93, nr * nl, w, h)
    dc = [to_dev(x) for x in c]
    dd = [to_dev(x) for x in d]
    out = out_frame(h, w)
    eqc.compose_direct_send_p2p_local(nr, dc, dd, out, dest_rank=1, mode=eqc.P2P_PIPELINED)
    torch.cuda.synchronize()
    got = to_host(out)
    rows = np.unique(np.r_[0, h // 2 - 1, h // 2, h - 1, np.linspace(0, h - 1, 12).astype(int)])
    want, _ = oracle.depth_composite([x[rows] for x in c], [x[rows] for x in d])
    np.testing.assert_array_equal(got[rows], want)


RLE_PULL_CASES = [
    # (nranks, n_local, w, h, dest)
    (2, 2, 300, 41, 0),
    (3, 1, 333, 20, 2),
    (4, 2, 640, 130, 1),
    (2, 4, 1920, 1080, 1),
]


def _encode_rank_streams(eqc, imgs_c, imgs_d, w, h):
    """One contiguous buffer per rank: its colour streams (swizzled), then
    depth, image_rle_max_size bytes apart -- as eqc_comm_stream_buffers."""
    cap = eqc.image_rle_max_size(w, h)
    nl = len(imgs_c)
    buf = torch.zeros(2 * nl * cap, dtype=torch.uint8, device="cuda")
    streams = [buf[i * cap:(i + 1) * cap] for i in range(2 * nl)]
    sizes = torch.zeros(2 * nl, dtype=torch.int64, device="cuda")
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(2 * nl, w, h), dtype=torch.uint8, device="cuda")
    kinds = [eqc.KIND_RGBA8] * nl + [eqc.KIND_DEPTH32] * nl
    flags = [eqc.FLAG_SWIZZLE] * nl + [0] * nl
    eqc.image_compress_rle_batch(list(imgs_c) + list(imgs_d), kinds, flags, streams, sizes, ws)
    return buf, cap


@pytest.mark.parametrize("case", RLE_PULL_CASES, ids=[f"n{c[0]}x{c[1]}_{c[2]}x{c[3]}_d{c[4]}" for c in RLE_PULL_CASES])
def test_rle_pull_virtual_ranks_equal_oracle(eqc, case):
    nr, nl, w, h, dest = case
    N = nr * nl
    c, d = synth.depth_sources(synth.SEED_BASE + 95 + N, N, w, h)
    want, _ = oracle.depth_composite(c, d)
    dc = [to_dev(x) for x in c]
    dd = [to_dev(x) for x in d]
    bufs = []
    cap = None
    for q in range(nr):
        b, cap = _encode_rank_streams(eqc, dc[q * nl:(q + 1) * nl], dd[q * nl:(q + 1) * nl], w, h)
        bufs.append(b)
    out = out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    stats = eqc.compose_direct_send_rle_pull_local(nr, nl, bufs, cap, w, h, out, status, dest_rank=dest)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    np.testing.assert_array_equal(to_host(out), want)
    assert stats[1] == nr - 1


SCATTER_CASES = [
    # (nranks, n_local, w, h, dest): uneven bands (h % n != 0), ragged chunks (w % 128 != 0)
    (2, 2, 300, 41, 0),
    (3, 1, 333, 20, 2),
    (4, 2, 640, 130, 1),
    (2, 4, 1920, 1080, 1),
]


@pytest.mark.parametrize("case", SCATTER_CASES, ids=[f"n{c[0]}x{c[1]}_{c[2]}x{c[3]}_d{c[4]}" for c in SCATTER_CASES])
def test_scatter_virtual_ranks_equal_oracle(eqc, case):
    """compositor_depth_rle_scatter (each rank's fused decode stores band j
    into rank j's frame slot) + compose_direct_send_scattered (band composite
    of the copies, colour to the destination) on virtual ranks: bit-exact
    against O1 over all ranks' sources in rank-major order."""
    nr, nl, w, h, dest = case
    N = nr * nl
    c, d = synth.depth_sources(synth.SEED_BASE + 97 + N, N, w, h)
    want, _ = oracle.depth_composite(c, d)
    dc = [to_dev(x) for x in c]
    dd = [to_dev(x) for x in d]
    cs, ds = [], []
    for q in range(nr):
        b, cap = _encode_rank_streams(eqc, dc[q * nl:(q + 1) * nl], dd[q * nl:(q + 1) * nl], w, h)
        cs += [b[i * cap:(i + 1) * cap] for i in range(nl)]
        ds += [b[(nl + i) * cap:(nl + i + 1) * cap] for i in range(nl)]
    out = out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    stats = eqc.compose_direct_send_scatter_local(nr, cs, ds, w, h, out, status, dest_rank=dest)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    np.testing.assert_array_equal(to_host(out), want)
    assert stats[0] == nr * (nr - 1)  # every rank received a band copy from every peer


def test_p2p_flag_wait_timeout_reports_nccl_error():
    # a virtual rank that never arrives (EQC_P2P_DROP_RANK): every other
    # rank's flag wait must give up after EQC_P2P_TIMEOUT_MS (no GPU hang)
    # and the call report EQC_E_NCCL.  In a subprocess: the dropped rank's
    # missing barrier leaves the peers' later reads undefined.
    code = r"""
import sys, time, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import synth
from gpu_util import to_dev, out_frame
from paper_1902_08755_b200 import eqc
c, d = synth.depth_sources(7, 2, 256, 32)
out = out_frame(32, 256)
t = time.time()
try:
    eqc.compose_direct_send_p2p_local(2, [to_dev(x) for x in c], [to_dev(x) for x in d], out)
    print("NOERROR")
except eqc.EqcError as e:
    print("CODE", e.code, round(time.time() - t, 2))
""" % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, EQC_P2P_TIMEOUT_MS="300", EQC_P2P_DROP_RANK="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith(("CODE", "NOERROR"))][-1]
    assert line.startswith("CODE -6"), line  # EQC_E_NCCL
    assert float(line.split()[2]) < 60.0


BS_CASES = [
    # (nranks, n_local, w, h, pitch, out_pitch, dest, op, gen)
    (2, 2, 300, 41, None, None, 0, "depth", "scene"),
    (4, 1, 130, 37, 136, 140, 2, "depth", "ties"),
    (8, 1, 128, 19, None, None, 7, "depth", "scene"),
    (4, 2, 640, 360, None, None, 1, "depth", "scene"),
    (2, 8, 320, 180, None, None, 1, "blend", "bricks"),
    (4, 2, 257, 77, None, 264, 3, "blend", "bricks"),
]


@pytest.mark.parametrize("case", BS_CASES, ids=[f"n{c[0]}x{c[1]}_{c[2]}x{c[3]}_{c[7]}_d{c[6]}" for c in BS_CASES])
def test_p2p_binary_swap_virtual_ranks(eqc, case):
    # depth: bit-exact vs O1 over all sources (R-C5 tie rule: bit-0 group);
    # blend: within 1/255 of O2 over all layers (R-C4, R-C6)
    nr, nl, w, h, pitch, opitch, dest, op, gen = case
    N = nr * nl
    out = out_frame(h, w, opitch)
    if op == "depth":
        c, d = _scene(N, w, h, synth.SEED_BASE + 97 + N + w, ties=gen == "ties")
        want, _ = oracle.depth_composite(c, d)
        stats = eqc.compose_binary_swap_p2p_local(nr, [to_dev(x, pitch) for x in c], [to_dev(x, pitch) for x in d],
                                                  out, dest_rank=dest)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(to_host(out), want)
        if h >= 2 * nr:
            assert stats[0] == nr * (nr.bit_length() - 1)  # one half sent per rank per round
            assert stats[1] == nr - 1
    else:
        layers = synth.volume_bricks(synth.SEED_BASE + 98 + N, N, w, h)
        want = oracle.blend_ordered(layers)
        eqc.compose_binary_swap_p2p_local(nr, [to_dev(x, pitch) for x in layers], None, out, dest_rank=dest,
                                          op=eqc.OP_BLEND)
        torch.cuda.synchronize()
        got = to_host(out)
        diff = np.abs(got.view(np.uint8).astype(int) - want.view(np.uint8).astype(int))
        assert diff.max() <= 1


S23_CASES = [
    # (nranks, n_local, w, h, dest, op, gen) -- 2-3 swap over peer memory (R-C21)
    (3, 2, 300, 41, 0, "depth", "scene"),
    (5, 1, 130, 37, 4, "depth", "ties"),
    (6, 1, 257, 77, 2, "depth", "scene"),
    (7, 2, 128, 45, 5, "depth", "ties"),
    (2, 3, 200, 30, 1, "depth", "scene"),
    (3, 4, 320, 180, 1, "blend", "bricks"),
    (5, 2, 130, 37, 0, "blend", "bricks"),
]


@pytest.mark.parametrize("case", S23_CASES, ids=[f"n{c[0]}x{c[1]}_{c[2]}x{c[3]}_{c[5]}_d{c[4]}" for c in S23_CASES])
def test_p2p_swap23_virtual_ranks(eqc, case):
    nr, nl, w, h, dest, op, gen = case
    N = nr * nl
    out = out_frame(h, w)
    if op == "depth":
        c, d = _scene(N, w, h, synth.SEED_BASE + 99 + N + w, ties=gen == "ties")
        want, _ = oracle.depth_composite(c, d)
        eqc.compose_swap23_p2p_local(nr, [to_dev(x) for x in c], [to_dev(x) for x in d], out, dest_rank=dest)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(to_host(out), want)
    else:
        layers = synth.volume_bricks(synth.SEED_BASE + 100 + N, N, w, h)
        want = oracle.blend_ordered(layers)
        eqc.compose_swap23_p2p_local(nr, [to_dev(x) for x in layers], None, out, dest_rank=dest, op=eqc.OP_BLEND)
        torch.cuda.synchronize()
        diff = np.abs(to_host(out).view(np.uint8).astype(int) - want.view(np.uint8).astype(int))
        assert diff.max() <= 1
