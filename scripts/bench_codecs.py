"""Codec comparison on one B200: the basic
64-bit RLE (RLE-64), per-component RLE, and per-component RLE with the swizzle
preconditioner, on the bench workload (8 sort-last sources 3840x2160: colour
and depth).  Reports compression rate (1 - compressed/raw, R-C10) per codec
and buffer kind, and encode / decode time of the 16-stream batch (CUDA graphs,
median of 20 replays of 5 calls).  Prints one JSON line.

    python scripts/bench_codecs.py
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402


def timed(fn, reps=5, steps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    return statistics.median(ts)


def main():
    W, H, N = 3840, 2160, 8
    dev = torch.device("cuda", 0)
    c, d = synth.depth_sources(synth.SEED_BASE + 10, N, W, H)
    imgs = [torch.from_numpy(x.view(np.int32)).to(dev) for x in list(c) + list(d)]
    kinds = [0] * N + [1] * N
    cap = eqc.image_rle_max_size(W, H)
    streams = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in imgs]
    sizes = torch.zeros(len(imgs), dtype=torch.int64, device=dev)
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(len(imgs), W, H), dtype=torch.uint8, device=dev)
    outs = [torch.empty((H, W), dtype=torch.int32, device=dev) for _ in imgs]
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    raw = W * H * 4
    res = {}
    for name, fl in [("rle64", [eqc.FLAG_RLE64] * (2 * N)), ("per_component", [0] * (2 * N)),
                     ("per_component_swizzle", [eqc.FLAG_SWIZZLE] * N + [0] * N)]:
        enc = lambda: eqc.image_compress_rle_batch(imgs, kinds, fl, streams, sizes, ws)  # noqa: E731
        t_enc = timed(enc)
        enc()
        torch.cuda.synchronize()
        sz = sizes.cpu().numpy()
        t_dec = timed(lambda: eqc.image_decompress_rle_batch(streams, outs, status))
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        assert all(torch.equal(a, b) for a, b in zip(imgs, outs))
        res[name] = {"rate_colour": round(1 - float(sz[:N].sum()) / (N * raw), 4),
                     "rate_depth": round(1 - float(sz[N:].sum()) / (N * raw), 4),
                     "encode_ms": round(t_enc, 4), "decode_ms": round(t_dec, 4),
                     "encode_gbs": round((2 * N * raw + float(sz.sum())) / t_enc / 1e6, 1),
                     "decode_gbs": round((2 * N * raw + float(sz.sum())) / t_dec / 1e6, 1)}
    print(json.dumps({"bench": "codecs", "workload": "8 x 3840x2160 colour + depth (16 streams)",
                      "rate": "1 - compressed/raw (R-C10)", "results": res}))


if __name__ == "__main__":
    main()
