"""Region of interest on one B200: full-frame compositing
against ROI compositing (image_roi on the device + compositor_*_roi), for
compact and scattered sort-last scenes (8 x 3840x2160 colour + depth) and the
c3 volume bricks (16 x 3840x2160 blend).  10 calls captured in a CUDA graph, replays
timed with CUDA events (median of 20); inputs > L2.  Prints one JSON line.

    python scripts/bench_roi.py
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

HBM = 6542.7
BG = 0xFFFFFFFF


def timed(fn, steps=20, warm=3, reps=10):
    """GPU time of one call: `reps` calls captured in a CUDA graph, replayed
    `steps` times between events (median / reps).  The graph removes the
    Python/ctypes launch overhead, which exceeds these kernels' run time."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
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
    W, H = 3840, 2160
    dev = torch.device("cuda", 0)
    res = {}
    for mode in ("compact", "scattered"):
        c, d = synth.depth_sources(synth.SEED_BASE + 10, 8, W, H, mode=mode)
        dc = [torch.from_numpy(x.view(np.int32)).to(dev) for x in c]
        dd = [torch.from_numpy(x.view(np.int32)).to(dev) for x in d]
        oc = torch.empty((H, W), dtype=torch.int32, device=dev)
        od = torch.empty((H, W), dtype=torch.int32, device=dev)
        r = torch.zeros((8, 4), dtype=torch.int32, device=dev)
        t_full = timed(lambda: eqc.compositor_depth(dc, dd, oc, od))
        ref = oc.clone()
        t_roi_only = timed(lambda: eqc.image_roi(dd, r, BG))
        t_comp = timed(lambda: eqc.compositor_depth_roi(dc, dd, r, oc, od))

        def both():
            eqc.image_roi(dd, r, BG)
            eqc.compositor_depth_roi(dc, dd, r, oc, od)
        t_both = timed(both)
        assert torch.equal(oc, ref), "ROI composite differs from the full composite"
        rois = r.cpu().numpy()
        cover = float(sum(int(x[2]) * int(x[3]) for x in rois)) / (W * H)
        P = W * H
        b_full = (8 * 8 + 8) * P
        b_roi_comp = 8 * cover * P + 8 * P  # ROI pixels read (colour + depth), full output written
        res[f"depth_{mode}"] = {
            "full_ms": round(t_full, 4), "image_roi_ms": round(t_roi_only, 4),
            "composite_roi_ms": round(t_comp, 4), "roi_plus_composite_ms": round(t_both, 4),
            "speedup_vs_full": round(t_full / t_both, 2), "roi_area_sum_frames": round(cover, 3),
            "full_gbs": round(b_full / t_full / 1e6, 1), "roi_composite_gbs": round(b_roi_comp / t_comp / 1e6, 1),
            "image_roi_gbs": round(4 * 8 * P / t_roi_only / 1e6, 1)}
        del dc, dd
    layers = synth.volume_bricks(synth.SEED_BASE + 2, 16, W, H)
    dl = [torch.from_numpy(x.view(np.int32)).to(dev) for x in layers]
    out = torch.empty((H, W), dtype=torch.int32, device=dev)
    r = torch.zeros((16, 4), dtype=torch.int32, device=dev)
    t_full = timed(lambda: eqc.compositor_blend_ordered(dl, out))
    ref = out.clone()
    t_roi_only = timed(lambda: eqc.image_roi(dl, r, 0))
    t_comp = timed(lambda: eqc.compositor_blend_ordered_roi(dl, r, out))

    def both_b():
        eqc.image_roi(dl, r, 0)
        eqc.compositor_blend_ordered_roi(dl, r, out)
    t_both = timed(both_b)
    assert torch.equal(out, ref), "ROI blend differs from the full blend"
    rois = r.cpu().numpy()
    cover = float(sum(int(x[2]) * int(x[3]) for x in rois)) / (W * H)
    P = W * H
    res["blend_c3_bricks"] = {
        "full_ms": round(t_full, 4), "image_roi_ms": round(t_roi_only, 4), "blend_roi_ms": round(t_comp, 4),
        "roi_plus_blend_ms": round(t_both, 4), "speedup_vs_full": round(t_full / t_both, 2),
        "roi_area_sum_frames": round(cover, 3), "full_gbs": round((4 * 16 + 4) * P / t_full / 1e6, 1),
        "roi_blend_gbs": round((4 * cover + 4) * P / t_comp / 1e6, 1)}
    print(json.dumps({"bench": "roi", "hbm_peak_gbs": HBM, "results": res}))


if __name__ == "__main__":
    main()
