"""Single GPU: does the asynchronous pipeline pay on one GPU?
Sequential step (encode 16 streams -> fused decode + composite, one stream)
vs two streams with double-buffered RLE streams (encode of frame k+1 overlaps
the decode + composite of frame k).  Bench workload; events around K steps."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402


def main():
    W, H, N, K = 3840, 2160, 8, 100
    dev = torch.device("cuda", 0)
    c, d = synth.depth_sources(synth.SEED_BASE + 10, N, W, H)
    imgs = [torch.from_numpy(x.view(np.int32)).to(dev) for x in list(c) + list(d)]
    kinds, flags = [0] * N + [1] * N, [1] * N + [0] * N
    cap = eqc.image_rle_max_size(W, H)
    sets = [[torch.empty(cap, dtype=torch.uint8, device=dev) for _ in imgs] for _ in range(2)]
    sizes = [torch.zeros(len(imgs), dtype=torch.int64, device=dev) for _ in range(2)]
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(len(imgs), W, H), dtype=torch.uint8, device=dev)
    oc = torch.empty((H, W), dtype=torch.int32, device=dev)
    od = torch.empty((H, W), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    s0 = torch.cuda.current_stream()
    res = {}
    for prio in (0, -1):
        s1 = torch.cuda.Stream(device=dev, priority=prio)
        for mode in ("sequential", "pipelined"):
            enc_done = [torch.cuda.Event() for _ in range(2)]
            dec_done = [None, None]

            def step(k):
                b = k % 2 if mode == "pipelined" else 0
                if mode == "pipelined" and dec_done[b] is not None:
                    s0.wait_event(dec_done[b])
                eqc.image_compress_rle_batch(imgs, kinds, flags, sets[b], sizes[b], ws, stream=s0)
                if mode == "sequential":
                    eqc.compositor_depth_rle(sets[b][:N], sets[b][N:], oc, od, status, stream=s0)
                    return
                enc_done[b].record(s0)
                s1.wait_event(enc_done[b])
                eqc.compositor_depth_rle(sets[b][:N], sets[b][N:], oc, od, status, stream=s1)
                ev = torch.cuda.Event()
                ev.record(s1)
                dec_done[b] = ev

            for k in range(6):
                step(k)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(s0)
            for k in range(K):
                step(k)
            for e in dec_done:
                if e is not None:
                    s0.wait_event(e)
            t1.record(s0)
            torch.cuda.synchronize()
            assert int(status.item()) == 0
            res[f"{mode}_prio{prio}"] = round(t0.elapsed_time(t1) / K, 4)
    print(json.dumps({"ms_per_step": res}))


if __name__ == "__main__":
    import gc
    gc.disable()
    main()
