"""Run the bench step a few times (for ncu captures): 8 x 3840x2160 sources,
RLE encode batch -> fused decode + depth composite; plus one plain
compositor_depth and one ordered blend of 16 bricks.

    python scripts/prof_step.py [--steps N] [--which all|step|composite|blend]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--which", default="all")
args = ap.parse_args()

W, H, N = 3840, 2160, 8
dev = torch.device("cuda", 0)
c, d = synth.depth_sources(20190213 + 10, N, W, H)
colors = [torch.from_numpy(x.view(np.int32)).to(dev) for x in c]
depths = [torch.from_numpy(x.view(np.int32)).to(dev) for x in d]
out_c = torch.empty((H, W), dtype=torch.int32, device=dev)
out_d = torch.empty((H, W), dtype=torch.int32, device=dev)
if args.which in ("all", "step"):
    imgs = colors + depths
    kinds = [0] * N + [1] * N
    flags = [1] * N + [0] * N
    cap = eqc.image_rle_max_size(W, H)
    streams = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in imgs]
    sizes = torch.zeros(len(imgs), dtype=torch.int64, device=dev)
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(len(imgs), W, H), dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    for _ in range(args.steps):
        eqc.image_compress_rle_batch(imgs, kinds, flags, streams, sizes, ws)
        eqc.compositor_depth_rle(streams[:N], streams[N:], out_c, out_d, status)
    outs = [torch.empty((H, W), dtype=torch.int32, device=dev) for _ in imgs]
    for _ in range(args.steps):
        eqc.image_decompress_rle_batch(streams, outs, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
if args.which in ("all", "composite"):
    for _ in range(args.steps):
        eqc.compositor_depth(colors, depths, out_c, out_d)
if args.which in ("all", "blend"):
    del colors, depths
    layers = synth.volume_bricks(20190213 + 2, 16, W, H)
    dl = [torch.from_numpy(x.view(np.int32)).to(dev) for x in layers]
    for _ in range(args.steps):
        eqc.compositor_blend_ordered(dl, out_c)
torch.cuda.synchronize()
print("prof_step ok")
