"""One process per GPU: compose_direct_send / compose_binary_swap over NCCL
(NVLink) against the oracle over all ranks' sources.  Launched by
tests/test_gpu_multi.py with torch.distributed.run."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    comm = eqc.Comm.from_torch_distributed()
    dev = torch.device("cuda", local)
    failures = []
    # (algo, n_local, w, h, dest, flags[, scene]): flags 0 = NVLink peer-memory direct
    # send, FLAG_NCCL = NCCL grouped send/recv, FLAG_RLE = RLE streams over NCCL,
    # FLAG_ROI = peer-memory direct send restricted to each partial's ROI
    R, X, O = eqc.FLAG_RLE, eqc.FLAG_NCCL, eqc.FLAG_ROI
    cases = [("ds", 2, 640, 361, 0, 0), ("ds", 1, 300, 41, world - 1, eqc.FLAG_OVERLAP), ("ds", 2, 1920, 1080, 1 % world, 0),
             ("ds", 2, 640, 361, 0, X), ("ds", 1, 300, 41, world - 1, R), ("ds", 2, 1920, 1080, 0, R),
             ("ds", 2, 640, 361, 0, O, "compact"), ("ds", 1, 301, 43, world - 1, O, "compact"),
             ("ds", 3, 1920, 1080, 1 % world, O, "compact"), ("ds", 2, 640, 361, 0, O, "scattered"),
             ("ds", 1, 64, 16, 0, O, "empty")]
    if world & (world - 1) == 0:
        cases += [("bs", 2, 640, 361, 0, 0), ("bs", 1, 300, 41, world - 1, R), ("bs", 2, 1920, 1080, 0, R)]
    # 2-3 swap (any rank count, R-C21)
    cases += [("s23", 2, 640, 361, 0, 0), ("s23", 1, 300, 41, world - 1, R), ("s23", 2, 1920, 1080, 1 % world, 0)]
    # streaming chain
    cases += [("st", 2, 640, 361, 0, 0), ("st", 1, 300, 41, world - 1, R)]
    # config c4 (8 sources of 7680x4320 over the ranks), checked on sampled rows
    if 8 % world == 0:
        cases += [("ds", 8 // world, 7680, 4320, 0, 0), ("ds", 8 // world, 7680, 4320, 0, R),
                  ("ds", 8 // world, 7680, 4320, 0, eqc.FLAG_OVERLAP)]
        if world & (world - 1) == 0:
            cases += [("bs", 8 // world, 7680, 4320, 0, 0)]
    for algo, nl, w, h, dest, rle, *scene in cases:
        N = world * nl
        mode = scene[0] if scene else "scattered"
        if mode == "empty":  # every source all background: ROIs are empty
            c = [np.zeros((h, w), np.uint32) for _ in range(N)]
            d = [np.full((h, w), 0xFFFFFFFF, np.uint32) for _ in range(N)]
        else:
            c, d = synth.depth_sources(synth.SEED_BASE + 3 + N + w, N, w, h, mode=mode)
        mine = range(rank * nl, (rank + 1) * nl)
        dc = [torch.from_numpy(c[i].view(np.int32)).to(dev) for i in mine]
        dd = [torch.from_numpy(d[i].view(np.int32)).to(dev) for i in mine]
        out = torch.zeros((h, w), dtype=torch.int32, device=dev)
        fn = {"ds": eqc.compose_direct_send, "bs": eqc.compose_binary_swap, "s23": eqc.compose_swap23,
              "st": eqc.compose_stream}[algo]
        for _ in range(2):  # the second call reuses the communicator's scratch
            fn(comm, dc, dd, out if rank == dest else None, dest_rank=dest, flags=rle)
        torch.cuda.synchronize()
        st = comm.stats()
        if rank == dest:
            got = out.cpu().numpy().view(np.uint32)
            if h > 2000:  # full-size c4: the oracle on sampled rows
                rows = np.random.default_rng(h).choice(h, 6, replace=False)
                for yy in rows:
                    want, _ = oracle.depth_composite([x[yy:yy + 1] for x in c], [x[yy:yy + 1] for x in d])
                    if not (got[yy:yy + 1] == want).all():
                        failures.append(f"{algo} nl={nl} {w}x{h} flags={rle}: row {yy} mismatch")
            else:
                want, _ = oracle.depth_composite(c, d)
                if not (got == want).all():
                    failures.append(f"{algo} nl={nl} {w}x{h} flags={rle}: mismatch {(got != want).sum()} px")
        if algo == "ds" and st[0] != world - 1:
            failures.append(f"{algo}: rank {rank} sent {st[0]} band messages, want {world - 1}")
        dist.barrier()
    # application-provided source ROIs, P2P and NCCL transports
    # (the 7680x4320, 2-per-rank case takes the pipelined peer-memory branch:
    # >= 2 sources and >= 6 Mpx per band)
    for nl, w, h, dest, fl in [(2, 640, 361, 0, 0), (1, 300, 41, world - 1, X), (2, 1920, 1080, 1 % world, 0),
                               (2, 7680, 4320, 0, 0)]:
        N = world * nl
        c, d = synth.depth_sources(synth.SEED_BASE + 90 + N + w, N, w, h, mode="compact")
        mine = range(rank * nl, (rank + 1) * nl)
        dc = [torch.from_numpy(c[i].view(np.int32)).to(dev) for i in mine]
        dd = [torch.from_numpy(d[i].view(np.int32)).to(dev) for i in mine]
        r = torch.tensor([list(oracle.roi(d[i], 0xFFFFFFFF)) for i in mine], dtype=torch.int32, device=dev)
        out = torch.zeros((h, w), dtype=torch.int32, device=dev)
        for _ in range(2):
            eqc.compose_direct_send_roi(comm, dc, dd, r, out if rank == dest else None, dest_rank=dest, flags=fl)
        torch.cuda.synchronize()
        if rank == dest and not (out.cpu().numpy().view(np.uint32) == oracle.depth_composite(c, d)[0]).all():
            failures.append(f"app-roi nl={nl} {w}x{h} flags={fl}: mismatch")
        dist.barrier()
    # EQC_OP_BLEND: layers in rank-block draw order, result
    # within 1/255 of O2 over all layers (unorm16 partials across GPUs, R-C6)
    bcases = [("ds", 4, 640, 361, 0, 0), ("ds", 2, 300, 41, world - 1, X), ("ds", 3, 320, 181, 1 % world, R)]
    if world & (world - 1) == 0:
        bcases += [("bs", 4, 640, 361, 0, 0), ("bs", 2, 300, 41, world - 1, R)]
    bcases += [("s23", 3, 640, 361, 0, 0), ("s23", 2, 300, 41, world - 1, R), ("st", 2, 320, 181, 0, 0)]
    if 16 % world == 0:  # config c3: 16 bricks of 3840x2160, sampled rows
        bcases += [("ds", 16 // world, 3840, 2160, 0, 0)]
    for algo, nl, w, h, dest, fl in bcases:
        N = world * nl
        layers = synth.volume_bricks(synth.SEED_BASE + 2 if h == 2160 else synth.SEED_BASE + 80 + N, N, w, h)
        mine = range(rank * nl, (rank + 1) * nl)
        dl = [torch.from_numpy(layers[i].view(np.int32)).to(dev) for i in mine]
        out = torch.zeros((h, w), dtype=torch.int32, device=dev)
        fn = {"ds": eqc.compose_direct_send, "bs": eqc.compose_binary_swap, "s23": eqc.compose_swap23,
              "st": eqc.compose_stream}[algo]
        for _ in range(2):
            fn(comm, dl, None, out if rank == dest else None, dest_rank=dest, flags=fl, op=eqc.OP_BLEND)
        torch.cuda.synchronize()
        if rank == dest:
            got = out.cpu().numpy().view(np.uint32)
            rows = np.random.default_rng(h).choice(h, 8, replace=False) if h > 2000 else np.arange(h)
            want = oracle.blend_ordered([x[rows] for x in layers])
            diff = np.abs(got[rows].view(np.uint8).astype(int) - want.view(np.uint8).astype(int)).max()
            if diff > 1:
                failures.append(f"blend {algo} nl={nl} {w}x{h} flags={fl}: max error {diff} LSB")
        dist.barrier()
    # EQC_OP_AVERAGE (subpixel accumulation + averaging): bit-exact
    for algo, nl, w, h, dest, fl in [("ds", 2, 640, 361, 0, 0), ("ds", 3, 300, 41, world - 1, R),
                                     ("s23", 2, 320, 181, 0, 0), ("st", 2, 320, 181, 1 % world, R)]:
        N = world * nl
        c, _ = synth.random_frames(600 + N + w, N, w, h)
        mine = range(rank * nl, (rank + 1) * nl)
        dl = [torch.from_numpy(c[i].view(np.int32)).to(dev) for i in mine]
        out = torch.zeros((h, w), dtype=torch.int32, device=dev)
        fn = {"ds": eqc.compose_direct_send, "s23": eqc.compose_swap23, "st": eqc.compose_stream}[algo]
        for _ in range(2):
            fn(comm, dl, None, out if rank == dest else None, dest_rank=dest, flags=fl, op=eqc.OP_AVERAGE)
        torch.cuda.synchronize()
        if rank == dest and not (out.cpu().numpy().view(np.uint32) == oracle.average(c)).all():
            failures.append(f"average {algo} nl={nl} {w}x{h} flags={fl}: mismatch")
        dist.barrier()
    # comm-owned peer-mapped frame slots (eqc_comm_frame_buffers): partials
    # written into slot k % 2 are pulled in place; the destination's frame is
    # either the comm's gather buffer (no band copy) or a caller tensor
    for w, h, dest in [(640, 361, 0), (1920, 1080, world - 1), (300, 41, 1 % world)]:
        fb = [comm.frame_buffers(w, h, i) for i in range(2)]
        if any(x is None for x in fb):
            failures.append(f"frame slots {w}x{h}: E_UNSUPPORTED on a peer-capable box")
            break
        user_out = torch.zeros((h, w), dtype=torch.int32, device=dev)
        for k in range(4):
            c, d = synth.depth_sources(synth.SEED_BASE + 700 + 10 * k + w, world, w, h)
            sc, sd, fin = fb[k % 2]
            sc.copy_(torch.from_numpy(c[rank].view(np.int32)))
            sd.copy_(torch.from_numpy(d[rank].view(np.int32)))
            out = fin if k < 2 else user_out
            eqc.compose_direct_send(comm, [sc], [sd], out if rank == dest else None, dest_rank=dest,
                                    flags=eqc.FLAG_OVERLAP if k % 2 else 0)
            torch.cuda.synchronize()
            st = comm.stats()
            if rank == dest and not (out.cpu().numpy().view(np.uint32) == oracle.depth_composite(c, d)[0]).all():
                failures.append(f"frame slot {k % 2} {w}x{h} out={'gather' if k < 2 else 'user'}: mismatch")
            if st[0] != world - 1:
                failures.append(f"frame slots: rank {rank} sent {st[0]} band messages, want {world - 1}")
            dist.barrier()
    # direct send of the compressed sources: each rank encodes its sources into
    # a peer-mapped stream slot; the fused decoder of band j pulls every rank's
    # records over NVLink (compose_direct_send_rle_pull)
    for k, (nl, w, h, dest) in enumerate([(2, 640, 361, 0), (3, 1920, 1080, world - 1), (1, 300, 41, 1 % world),
                                          (2, 640, 361, 0)]):
        N = world * nl
        c, d = synth.depth_sources(synth.SEED_BASE + 800 + N + w + k, N, w, h)
        mine = range(rank * nl, (rank + 1) * nl)
        imgs = [torch.from_numpy(c[i].view(np.int32)).to(dev) for i in mine] + \
               [torch.from_numpy(d[i].view(np.int32)).to(dev) for i in mine]
        cap = eqc.image_rle_max_size(w, h)
        sb = comm.stream_buffers(2 * nl, cap, k % 2)
        if sb is None:
            failures.append("stream slots: E_UNSUPPORTED on a peer-capable box")
            break
        sizes = torch.zeros(2 * nl, dtype=torch.int64, device=dev)
        ws = torch.zeros(eqc.image_rle_workspace_size_batch(2 * nl, w, h), dtype=torch.uint8, device=dev)
        eqc.image_compress_rle_batch(imgs, [0] * nl + [1] * nl, [1] * nl + [0] * nl, sb, sizes, ws)
        fb = comm.frame_buffers(w, h, 0)
        out = fb[2] if k == 3 else torch.zeros((h, w), dtype=torch.int32, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        eqc.compose_direct_send_rle_pull(comm, nl, w, h, k % 2, out if rank == dest else None, status, dest_rank=dest)
        torch.cuda.synchronize()
        if int(status.item()) != 0:
            failures.append(f"rle-pull {w}x{h} nl={nl}: status {int(status.item())}")
        if rank == dest and not (out.cpu().numpy().view(np.uint32) == oracle.depth_composite(c, d)[0]).all():
            failures.append(f"rle-pull {w}x{h} nl={nl} out={'gather' if k == 3 else 'user'}: mismatch")
        dist.barrier()
    # the exchange riding the decoder: each rank's fused decode stores band j
    # of its sources into rank j's frame slot (compositor_depth_rle_scatter),
    # then every rank composites the copies of its band from its own slot
    # (compose_direct_send_scattered); unequal bands (h % n != 0) included
    for k, (nl, w, h, dest) in enumerate([(2, 640, 361, 0), (3, 1920, 1080, world - 1), (1, 300, 41, 1 % world),
                                          (2, 640, 361, 0)]):
        N = world * nl
        c, d = synth.depth_sources(synth.SEED_BASE + 900 + N + w + k, N, w, h)
        mine = range(rank * nl, (rank + 1) * nl)
        imgs = [torch.from_numpy(c[i].view(np.int32)).to(dev) for i in mine] + \
               [torch.from_numpy(d[i].view(np.int32)).to(dev) for i in mine]
        cap = eqc.image_rle_max_size(w, h)
        streams = [torch.zeros(cap, dtype=torch.uint8, device=dev) for _ in imgs]
        sizes = torch.zeros(2 * nl, dtype=torch.int64, device=dev)
        ws = torch.zeros(eqc.image_rle_workspace_size_batch(2 * nl, w, h), dtype=torch.uint8, device=dev)
        eqc.image_compress_rle_batch(imgs, [0] * nl + [1] * nl, [1] * nl + [0] * nl, streams, sizes, ws)
        fb = comm.frame_buffers(w, h, k % 2)
        out = fb[2] if k == 3 else torch.zeros((h, w), dtype=torch.int32, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        eqc.compositor_depth_rle_scatter(comm, streams[:nl], streams[nl:], w, h, k % 2, status)
        eqc.compose_direct_send_scattered(comm, w, h, k % 2, out if rank == dest else None, dest_rank=dest,
                                          flags=eqc.FLAG_OVERLAP if k % 2 else 0)
        torch.cuda.synchronize()
        if int(status.item()) != 0:
            failures.append(f"scatter {w}x{h} nl={nl}: status {int(status.item())}")
        if rank == dest and not (out.cpu().numpy().view(np.uint32) == oracle.depth_composite(c, d)[0]).all():
            failures.append(f"scatter {w}x{h} nl={nl} out={'gather' if k == 3 else 'user'}: mismatch")
        if comm.stats()[0] != world - 1:
            failures.append(f"scatter: rank {rank} received {comm.stats()[0]} bands, want {world - 1}")
        dist.barrier()
    comm.destroy()
    t = torch.tensor([len(failures)], device=dev)
    dist.all_reduce(t)
    for f in failures:
        print(f"rank {rank}: {f}", flush=True)
    if rank == 0 and int(t.item()) == 0:
        print("ALL OK", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
