"""Streaming sort-last chain on N GPUs: measured chain time
against the thesis's latency formula t_draw + (n - 1) (t_readback + t_assemble)
(P:2237-2238), with each term measured on this machine:
  t_local    local pre-composite of a rank's sources (stands for t_draw's
             compositing share: the sources are already rendered),
  t_transfer whole partial frame (colour + depth, 8 B/px) rank k -> k+1 (NCCL),
  t_merge    2-input composite of the whole frame (compositor_depth),
  t_final    colour of the completed frame to dest (if dest != n - 1).
Config c4-style: 8 sources of W x H split over the ranks.  CUDA events, max
over ranks.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/bench_stream.py
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


def timed(fn, steps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    t = torch.tensor([statistics.median(ts)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--w", type=int, default=3840)
    ap.add_argument("--h", type=int, default=2160)
    ap.add_argument("--sources", type=int, default=8)
    ap.add_argument("--steps", type=int, default=20)
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
    nl = N // n
    c, d = synth.depth_sources(synth.SEED_BASE + 3, N, W, H)
    mine = range(rank * nl, (rank + 1) * nl)
    dc = [torch.from_numpy(c[i].view(np.int32)).to(dev) for i in mine]
    dd = [torch.from_numpy(d[i].view(np.int32)).to(dev) for i in mine]
    del c, d
    final = torch.empty((H, W), dtype=torch.int32, device=dev)
    pc, pd = torch.empty_like(final), torch.empty_like(final)
    res = {}
    res["chain_ms"] = timed(lambda: eqc.compose_stream(comm, dc, dd, final if rank == 0 else None, dest_rank=0), a.steps)
    res["t_local_ms"] = timed(lambda: eqc.compositor_depth(dc, dd, pc, pd), a.steps)
    res["t_merge_ms"] = timed(lambda: eqc.compositor_depth([pc, pc], [pd, pd], final, pd), a.steps)
    buf = torch.empty((2, H, W), dtype=torch.int32, device=dev)

    def xfer():
        if n < 2:
            return
        if rank == 0:
            dist.send(buf, 1)
        elif rank == 1:
            dist.recv(buf, 0)
    res["t_transfer_ms"] = timed(xfer, a.steps)

    def gath():
        if n < 2:
            return
        if rank == n - 1:
            dist.send(buf[0], 0)
        elif rank == 0:
            dist.recv(buf[0], n - 1)
    res["t_final_ms"] = timed(gath, a.steps)
    pred = res["t_local_ms"] + (n - 1) * (res["t_transfer_ms"] + res["t_merge_ms"]) + (res["t_final_ms"] if n > 1 else 0)
    res["predicted_ms"] = round(pred, 4)
    res["measured_over_predicted"] = round(res["chain_ms"] / pred, 3)
    if rank == 0:
        out.write(json.dumps({"bench": "stream_chain", "config": f"{N} sources {W}x{H}, {n} GPU(s)", "n_gpus": n,
                              "formula": "t_local + (n-1)(t_transfer + t_merge) + t_final (P:2237-2238)",
                              "results": {k: round(v, 4) if isinstance(v, float) else v for k, v in res.items()}}) + "\n")
        out.flush()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
