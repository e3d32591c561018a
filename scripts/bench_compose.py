"""Multi-GPU compositing schedules on config c4 of BASELINE.json: 8 sources of
7680x4320 RGBA8 + depth32 split over N GPUs (rank g holds 8/N sources),
direct send (NVLink peer-memory pull, or NCCL, or RLE over NCCL) and binary
swap, timed with CUDA events (max over ranks), against the NVLink roofline of
SURVEY 8(e): the destination receives (N-1)/N * 12 * P bytes (colour+depth
band exchange + colour gather).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        scripts/bench_compose.py [--w 7680 --h 4320 --sources 8 --steps 20]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402

NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--w", type=int, default=7680)
    ap.add_argument("--h", type=int, default=4320)
    ap.add_argument("--sources", type=int, default=8)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--scene", default="scattered", choices=["scattered", "compact", "bricks"])
    a = ap.parse_args()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    out = os.fdopen(json_fd, "w")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, n = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    comm = eqc.Comm.from_torch_distributed()
    W, H, N = a.w, a.h, a.sources
    assert N % n == 0
    nl = N // n
    blend = a.scene == "bricks"  # config c3: ordered blend of volume bricks (EQC_OP_BLEND)
    if blend:
        c, d = synth.volume_bricks(synth.SEED_BASE + 2, N, W, H), None
    else:
        c, d = synth.depth_sources(synth.SEED_BASE + 3, N, W, H, mode=a.scene)  # config index 3 (c4)
    mine = range(rank * nl, (rank + 1) * nl)
    dc = [torch.from_numpy(c[i].view(np.int32)).to(dev) for i in mine]
    dd = None if blend else [torch.from_numpy(d[i].view(np.int32)).to(dev) for i in mine]
    del c, d  # parity of these schedules at this size: tests/mp_compose.py (c4 case)
    final = torch.empty((H, W), dtype=torch.int32, device=dev) if rank == 0 else None
    P = W * H
    s = torch.cuda.current_stream()
    results = {}
    variants = [("direct_send_p2p", eqc.compose_direct_send, 0),
                ("direct_send_p2p_roi", eqc.compose_direct_send, eqc.FLAG_ROI),
                ("direct_send_nccl", eqc.compose_direct_send, eqc.FLAG_NCCL),
                ("direct_send_rle", eqc.compose_direct_send, eqc.FLAG_RLE)]
    if n & (n - 1) == 0:
        variants += [("binary_swap_p2p", eqc.compose_binary_swap, 0),
                     ("binary_swap_nccl", eqc.compose_binary_swap, eqc.FLAG_NCCL),
                     ("binary_swap_rle", eqc.compose_binary_swap, eqc.FLAG_RLE)]
    variants += [("swap23_p2p", eqc.compose_swap23, 0), ("swap23_nccl", eqc.compose_swap23, eqc.FLAG_NCCL),
                 ("swap23_rle", eqc.compose_swap23, eqc.FLAG_RLE), ("stream_nccl", eqc.compose_stream, 0)]
    op = eqc.OP_BLEND if blend else eqc.OP_DEPTH
    if not blend:  # application-provided ROIs: here the sources' exact boxes, from image_roi
        app_roi = torch.zeros((len(dd), 4), dtype=torch.int32, device=dev)
        eqc.image_roi(dd, app_roi, 0xFFFFFFFF)
        torch.cuda.synchronize()

        def ds_app_roi(comm_, dc_, dd_, final_, dest_rank=0, flags=0, op=0, stream=None):
            return eqc.compose_direct_send_roi(comm_, dc_, dd_, app_roi, final_, dest_rank=dest_rank, flags=flags,
                                               stream=stream)
        variants.insert(2, ("direct_send_p2p_app_roi", ds_app_roi, 0))
        fb = comm.frame_buffers(W, H, 0) if nl == 1 else None
        if fb is not None:  # one partial per GPU already in a peer-mapped frame slot: no pre-composite copy
            fb[0].copy_(dc[0])
            fb[1].copy_(dd[0])
            torch.cuda.synchronize()

            def ds_slots(comm_, dc_, dd_, final_, dest_rank=0, flags=0, op=0, stream=None):
                return eqc.compose_direct_send(comm_, [fb[0]], [fb[1]], fb[2] if rank == dest_rank else None,
                                               dest_rank=dest_rank, flags=flags, stream=stream)
            variants.insert(1, ("direct_send_p2p_slots", ds_slots, 0))
    if blend:
        variants = [v for v in variants if "roi" not in v[0]]
    for name, fn, flags in variants:
        for _ in range(a.warmup):
            fn(comm, dc, dd, final, dest_rank=0, flags=flags, op=op, stream=s)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.steps):
            fn(comm, dc, dd, final, dest_rank=0, flags=flags, op=op, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        st = comm.stats()
        results[name] = {"ms": round(float(t.item()), 4), "stats_rank0": st if rank == 0 else None}
    if rank == 0:
        inbound = (n - 1) / n * 12 * P  # blend: 8 B unorm16 partial + 4 B colour gather, the same
        t_nvl_us = inbound / (NVLINK_GBS * 1e9) * 1e6
        for r in results.values():
            r["source_mpx_per_s"] = round(N * P / (r["ms"] * 1e-3) / 1e6, 1)
            r["frac_of_nvlink_roof"] = round(t_nvl_us / (r["ms"] * 1e3), 3) if n > 1 else None
        tag = "c3 blend" if blend else "c4"
        line = {"config": f"{tag}: {N} sources {W}x{H} ({a.scene}), {n} GPU(s), {nl} source(s) per GPU", "n_gpus": n,
                "nvlink_roof_us": round(t_nvl_us, 1), "nvlink_gbs_per_dir": NVLINK_GBS,
                "dest_inbound_bytes": int(inbound), "results": results}
        out.write(json.dumps(line) + "\n")
        out.flush()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
