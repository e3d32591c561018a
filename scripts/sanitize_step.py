"""Small invocations of every libeqc kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): config c1 (2 x 64x64) and odd
fuzz shapes (ragged chunks, pitch > w, misaligned rows), each result checked
against the oracle so a silent corruption is also caught.  The peer-memory
virtual-rank executors are left out: their flag barriers need the ranks'
kernels to run concurrently, which the sanitizer does not guarantee.

    compute-sanitizer --tool memcheck python scripts/sanitize_step.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import to_dev, to_host  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402

SHAPES = [(64, 64, None, 0), (333, 7, 340, 1), (129, 5, None, 0), (130, 3, 136, 1)]
GUARD = 4096  # words of guard zone on each side of every output
_guards = []


def out_frame(h, w, pitch=None):
    """An output frame [h][w] (row pitch `pitch`) inside a buffer whose guard
    zones before, between rows and after hold a pattern that must survive."""
    P = pitch or w
    buf = torch.full((GUARD + h * P + GUARD,), 0x6B6B6B6B, dtype=torch.int64).to(torch.int32).cuda()
    view = buf[GUARD:GUARD + h * P].view(h, P)[:, :w]
    _guards.append((buf, h, w, P))
    return view


_bguards = []


def stream_buf(cap):
    """A stream buffer of `cap` bytes between guard zones."""
    buf = torch.full((GUARD + cap + GUARD,), 0x6B, dtype=torch.uint8, device="cuda")
    _bguards.append((buf, cap))
    return buf[GUARD:GUARD + cap]


def guards_intact():
    ok = True
    for buf, cap in _bguards:
        a = buf.cpu().numpy()
        ok &= bool((a[:GUARD] == 0x6B).all() and (a[GUARD + cap:] == 0x6B).all())
    for buf, h, w, P in _guards:
        a = buf.cpu().numpy().view(np.uint32)
        body = a[GUARD:GUARD + h * P].reshape(h, P)
        ok &= bool((a[:GUARD] == 0x6B6B6B6B).all() and (a[GUARD + h * P:] == 0x6B6B6B6B).all())
        ok &= bool((body[:, w:] == 0x6B6B6B6B).all())
    return ok


def main():
    ok = True
    for (w, h, pitch, off) in SHAPES:
        n = 2
        c, d = synth.depth_sources(synth.SEED_BASE + w + h, n, w, h)
        dc = [to_dev(x, pitch, off) for x in c]
        dd = [to_dev(x, pitch, off) for x in d]
        # depth composite
        want_c, want_d = oracle.depth_composite(c, d)
        oc, od = out_frame(h, w), out_frame(h, w)
        eqc.compositor_depth(dc, dd, oc, od)
        ok &= np.array_equal(to_host(oc), want_c) and np.array_equal(to_host(od), want_d)
        # blend
        layers = synth.volume_bricks(synth.SEED_BASE + 2 + w, 3, w, h)
        ob = out_frame(h, w)
        eqc.compositor_blend_ordered([to_dev(x, pitch, off) for x in layers], ob)
        wb = oracle.blend_ordered(layers)
        ok &= int(np.abs(to_host(ob).view(np.uint8).astype(int) - wb.view(np.uint8).astype(int)).max()) <= 1
        # encode (v1 batch with swizzle, RLE-64), decode, fused decode
        cap = eqc.image_rle_max_size(w, h)
        for r64 in (0, 1):
            imgs = dc + dd
            kinds = [eqc.KIND_RGBA8] * n + [eqc.KIND_DEPTH32] * n
            fl = ([eqc.FLAG_RLE64] * 2 * n) if r64 else ([eqc.FLAG_SWIZZLE] * n + [0] * n)
            streams = [stream_buf(cap) for _ in imgs]
            sizes = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
            ws = torch.zeros(eqc.image_rle_workspace_size_batch(2 * n, w, h), dtype=torch.uint8, device="cuda")
            eqc.image_compress_rle_batch(imgs, kinds, fl, streams, sizes, ws)
            torch.cuda.synchronize()
            outs = [out_frame(h, w, pitch) for _ in imgs]
            st = torch.zeros(1, dtype=torch.int32, device="cuda")
            eqc.image_decompress_rle_batch(streams, outs, st)
            torch.cuda.synchronize()
            ok &= int(st.item()) == 0
            ok &= all(np.array_equal(to_host(o), x) for o, x in zip(outs, list(c) + list(d)))
            if not r64:
                ok &= bytes(streams[0][:int(sizes[0])].cpu().numpy()) == oracle.rle_encode(c[0], kind=0, flags=1)
                fc, fd = out_frame(h, w), out_frame(h, w)
                eqc.compositor_depth_rle(streams[:n], streams[n:], fc, fd, st)
                torch.cuda.synchronize()
                ok &= int(st.item()) == 0 and np.array_equal(to_host(fc), want_c)
        # ROI scan
        roi = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
        eqc.image_roi(dd, roi, 0xFFFFFFFF)
        torch.cuda.synchronize()
        # virtual-rank schedules (device copies for NCCL), raw and RLE
        for fn in (eqc.compose_direct_send_local, eqc.compose_binary_swap_local):
            for fl in (0, eqc.FLAG_RLE):
                o = out_frame(h, w)
                fn(2, dc, dd, o, dest_rank=1, flags=fl)
                torch.cuda.synchronize()
                ok &= np.array_equal(to_host(o), want_c)
        o = out_frame(h, w)
        eqc.compose_tiles_local(2, dc, dd, o, tiles_x=2, tiles_y=1)
        torch.cuda.synchronize()
        ok &= np.array_equal(to_host(o), want_c)
    torch.cuda.synchronize()
    g = guards_intact()
    print("guard zones intact:", g, flush=True)
    ok &= g
    print("SANITIZE_STEP", "OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
