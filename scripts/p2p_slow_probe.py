"""Do kernels run slower once the peer-memory comm is set up?  (torchrun N=2)
Times image_compress_rle_batch and compositor_depth_rle per call on each rank
before and after eqc.Comm + frame slots, decoding into a plain tensor and into
a frame slot."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402

W, H, N = 3840, 2160, 8


def per_call(fn, reps=10):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps, 4)


def main():
    rank = int(os.environ.get("RANK", 0))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl")
    c, d = synth.depth_sources(synth.SEED_BASE + 10 + rank, N, W, H)
    imgs = [torch.from_numpy(x.view(np.int32)).to(dev) for x in list(c) + list(d)]
    kinds, flags = [0] * N + [1] * N, [1] * N + [0] * N
    cap = eqc.image_rle_max_size(W, H)
    streams = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in imgs]
    sizes = torch.zeros(len(imgs), dtype=torch.int64, device=dev)
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(len(imgs), W, H), dtype=torch.uint8, device=dev)
    oc = torch.empty((H, W), dtype=torch.int32, device=dev)
    od = torch.empty((H, W), dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    enc = lambda: eqc.image_compress_rle_batch(imgs, kinds, flags, streams, sizes, ws)
    dec = lambda o: (lambda: eqc.compositor_depth_rle(streams[:N], streams[N:], o[0], o[1], st))
    res = {"before": (per_call(enc), per_call(dec((oc, od))))}
    dist.barrier()
    comm = eqc.Comm.from_torch_distributed()
    fb = comm.frame_buffers(W, H, 0)
    torch.cuda.synchronize()
    dist.barrier()
    res["after_comm_plain"] = (per_call(enc), per_call(dec((oc, od))))
    res["after_comm_slot"] = (per_call(enc), per_call(dec((fb[0], fb[1]))))
    oc2 = torch.empty((H, W), dtype=torch.int32, device=dev)
    od2 = torch.empty((H, W), dtype=torch.int32, device=dev)
    res["after_comm_new_alloc"] = (per_call(enc), per_call(dec((oc2, od2))))
    dist.barrier()
    print(f"rank {rank}: {res}", flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
