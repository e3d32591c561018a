"""Multi-GPU bench step with the compressed direct send (torchrun): every rank
encodes its 8 x 4K sources (16 streams) into a peer-mapped stream slot, and
compose_direct_send_rle_pull decodes + composites band j of ALL sources on
rank j, pulling the peers' records over NVLink.  Pipelined: the compose of
frame k (own stream) overlaps the encode of frame k+1.  Prints ms/step."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402


def main():
    import gc
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, n = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    comm = eqc.Comm.from_torch_distributed()
    W, H, NS, K = 3840, 2160, 8, 100
    c, d = synth.depth_sources(synth.SEED_BASE + 10 + rank, NS, W, H)
    imgs = [torch.from_numpy(x.view(np.int32)).to(dev) for x in list(c) + list(d)]
    kinds, flags = [0] * NS + [1] * NS, [1] * NS + [0] * NS
    cap = eqc.image_rle_max_size(W, H)
    sb = [comm.stream_buffers(2 * NS, cap, i) for i in range(2)]
    fb = comm.frame_buffers(W, H, 0)
    final = fb[2] if rank == 0 else None
    sizes = torch.zeros(2 * NS, dtype=torch.int64, device=dev)
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(2 * NS, W, H), dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    s0 = torch.cuda.current_stream()
    res = {}
    for mode in ("pipelined", "sequential"):
        s1 = torch.cuda.Stream(device=dev, priority=-1) if mode == "pipelined" else s0
        composed = [None, None]

        def step(k):
            b = k % 2
            if composed[b] is not None:
                s0.wait_event(composed[b])
            eqc.image_compress_rle_batch(imgs, kinds, flags, sb[b], sizes, ws, stream=s0)
            if s1 is not s0:
                ev = torch.cuda.Event()
                ev.record(s0)
                s1.wait_event(ev)
            eqc.compose_direct_send_rle_pull(comm, NS, W, H, b, final, status, dest_rank=0, stream=s1)
            ev2 = torch.cuda.Event()
            ev2.record(s1)
            composed[b] = ev2

        for k in range(6):
            step(k)
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        gc.collect()
        gc.disable()
        dist.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s0)
        for k in range(K):
            step(k)
        for e in composed:
            s0.wait_event(e)
        t1.record(s0)
        torch.cuda.synchronize()
        gc.enable()
        ms = t0.elapsed_time(t1) / K
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[mode] = {"ms_per_step": round(float(t.item()), 4),
                     "source_mpx_per_s": round(n * NS * W * H / (float(t.item()) * 1e-3) / 1e6, 1)}
        dist.barrier()
    if rank == 0:
        print(json.dumps({"bench": "rle_pull", "n_gpus": n, "results": res}), flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
