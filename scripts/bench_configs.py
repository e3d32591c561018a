"""Every BASELINE config on one B200: c1 (2 x 64x64,
launch-bound: CUDA-graph replay), c2 (8 x 1920x1080: composite only, and the
RLE pipeline), c3 (16 x 3840x2160 ordered blend), c4 all local on one GPU
(8 x 7680x4320 composite).  Each op is captured in a CUDA graph (10 calls)
and replayed 20 times between CUDA events; achieved = algorithmic bytes /
time against the measured HBM copy peak.  Prints one JSON line.

    python scripts/bench_configs.py [--skip-c4]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402

HBM = 6542.7


def graph_time(fn, reps=10, steps=20):
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


def dev(frames):
    return [torch.from_numpy(x.view(np.int32)).cuda() for x in frames]


def composite_case(seed, n, w, h):
    c, d = synth.depth_sources(seed, n, w, h)
    dc, dd = dev(c), dev(d)
    oc = torch.empty((h, w), dtype=torch.int32, device="cuda")
    od = torch.empty_like(oc)
    t = graph_time(lambda: eqc.compositor_depth(dc, dd, oc, od))
    b = (8 * n + 8) * w * h
    return {"ms": round(t, 4), "source_mpx_per_s": round(n * w * h / t / 1e3, 1),
            "alg_bytes": b, "gbs": round(b / t / 1e6, 1), "frac": round(b / t / 1e6 / HBM, 3)}, (dc, dd)


def pipeline_case(dc, dd, n, w, h):
    imgs = dc + dd
    kinds, flags = [0] * n + [1] * n, [1] * n + [0] * n
    cap = eqc.image_rle_max_size(w, h)
    st = [torch.empty(cap, dtype=torch.uint8, device="cuda") for _ in imgs]
    sz = torch.zeros(len(imgs), dtype=torch.int64, device="cuda")
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(len(imgs), w, h), dtype=torch.uint8, device="cuda")
    oc = torch.empty((h, w), dtype=torch.int32, device="cuda")
    od = torch.empty_like(oc)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")

    def step():
        eqc.image_compress_rle_batch(imgs, kinds, flags, st, sz, ws)
        eqc.compositor_depth_rle(st[:n], st[n:], oc, od, status)
    t = graph_time(step)
    comp = float(sz.sum().item())
    b = 2 * n * 4 * w * h + 2 * comp + 8 * w * h
    return {"ms": round(t, 4), "source_mpx_per_s": round(n * w * h / t / 1e3, 1), "r": round(comp / (2 * n * 4 * w * h), 4),
            "alg_bytes": int(b), "gbs": round(b / t / 1e6, 1), "frac": round(b / t / 1e6 / HBM, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c4", action="store_true")
    a = ap.parse_args()
    res = {}
    res["c1_composite_2x64x64"], (dc, dd) = composite_case(synth.SEED_BASE + 0, 2, 64, 64)
    res["c1_rle_pipeline_2x64x64"] = pipeline_case(dc, dd, 2, 64, 64)
    res["c2_composite_8x1920x1080"], (dc, dd) = composite_case(synth.SEED_BASE + 1, 8, 1920, 1080)
    res["c2_rle_pipeline_8x1920x1080"] = pipeline_case(dc, dd, 8, 1920, 1080)
    del dc, dd
    layers = dev(synth.volume_bricks(synth.SEED_BASE + 2, 16, 3840, 2160))
    out = torch.empty((2160, 3840), dtype=torch.int32, device="cuda")
    t = graph_time(lambda: eqc.compositor_blend_ordered(layers, out))
    b = (4 * 16 + 4) * 3840 * 2160
    res["c3_blend_16x3840x2160"] = {"ms": round(t, 4), "source_mpx_per_s": round(16 * 3840 * 2160 / t / 1e3, 1),
                                    "alg_bytes": b, "gbs": round(b / t / 1e6, 1), "frac": round(b / t / 1e6 / HBM, 3)}
    del layers
    if not a.skip_c4:
        res["c4_composite_8x7680x4320_one_gpu"], _ = composite_case(synth.SEED_BASE + 3, 8, 7680, 4320)
    print(json.dumps({"bench": "configs", "hbm_peak_gbs": HBM, "timing": "CUDA graph of 10 calls, median of 20 replays",
                      "results": res}))


if __name__ == "__main__":
    main()
