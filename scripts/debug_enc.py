"""Encoder debugging aid: encode seeded images on the GPU and report, per
case, whether the stream equals the oracle's, else the first differing chunk
(table entry, plane records) of each side.  Test infrastructure only."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import to_dev, bytes_of  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402


def split(b, nch):
    tab = np.frombuffer(b[32:32 + 8 * nch], dtype=np.uint32).reshape(nch, 2)
    return tab, b[32 + 8 * nch:]


def report(name, got, want, nch):
    if got == want:
        print(f"{name}: OK ({len(want)} B)")
        return True
    print(f"{name}: MISMATCH got {len(got)} B want {len(want)} B; header eq {got[:32] == want[:32]}")
    tg, pg = split(got, nch)
    tw, pw = split(want, nch)
    for c in range(nch):
        if not np.array_equal(tg[c], tw[c]) or pg[tg[c][0]:tg[c][0] + sum(tg[c][1].tobytes())] != pw[tw[c][0]:tw[c][0] + sum(tw[c][1].tobytes())]:
            print(f"  chunk {c}: table got off={tg[c][0]} ps={list(tg[c][1].tobytes())} want off={tw[c][0]} ps={list(tw[c][1].tobytes())}")
            o = tw[c][0]
            for p, s in enumerate(tw[c][1].tobytes()):
                print(f"   want plane {p}: {pw[o:o + s].hex()}")
                o += s
            o = tg[c][0]
            for p, s in enumerate(tg[c][1].tobytes()):
                print(f"   got  plane {p}: {pg[o:o + s].hex()}")
                o += s
            break
    return False


def run(name, img, kind, flags):
    h, w = img.shape
    want = oracle.rle_encode(img, kind=kind, flags=flags)
    src = to_dev(img)
    cap = eqc.image_rle_max_size(w, h)
    dst = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    d_size = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(1, w, h), dtype=torch.uint8, device="cuda")
    eqc.image_compress_rle(src, kind, flags, dst, d_size, ws)
    torch.cuda.synchronize()
    n = int(d_size.item())
    got = bytes_of(dst, max(n, 0))
    nch = ((w + 127) // 128) * h
    return report(name, got, want, nch)


def main():
    ok = True
    rng = np.random.default_rng(1)
    ok &= run("const 128x1", np.full((1, 128), 0x11223344, np.uint32), 1, 0)
    a = np.full((1, 128), 7, np.uint32); a[0, 5] = 9
    ok &= run("one diff 128x1", a, 1, 0)
    ok &= run("ramp 128x1", np.arange(128, dtype=np.uint32).reshape(1, 128), 1, 0)
    ok &= run("noise 128x1", rng.integers(0, 2**32, size=(1, 128), dtype=np.uint32), 1, 0)
    ok &= run("noise 256x2", rng.integers(0, 2**32, size=(2, 256), dtype=np.uint32), 1, 0)
    v = np.repeat(rng.integers(0, 4, size=128), 1)[:128].astype(np.uint32) * 0x01010101
    ok &= run("smallalpha 128x1", v.reshape(1, 128).copy(), 1, 0)
    c, d = synth.depth_sources(7, 1, 640, 360)
    ok &= run("depth 640x360", d[0], 1, 0)
    ok &= run("colour 640x360 swz", c[0], 0, 1)
    ok &= run("odd 333x7", rng.integers(0, 3, size=(7, 333), dtype=np.uint32), 1, 0)
    print("ALL OK" if ok else "FAIL")


if __name__ == "__main__":
    main()
