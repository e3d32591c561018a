"""Display-wall benchmark: 64 full-wall sources of
15360 x 5760 (a 6 x 4 wall of 2560 x 1440 tiles, ~70 % background, F = 0.3),
drawn on the GPU (synth.depth_sources_torch, seed 20190213 + 4).

Single process (one GPU):
  * composite   compositor_depth over all 64 sources (46.0 GB moved; the
                SURVEY 8(d) roof 7.03 ms at the copy-measured HBM peak);
  * tiles_vN    compose_tiles_local, N virtual ranks, RLE transport: each
                rank pre-composites 64/N sources, encodes its 24 partial
                tiles, the owner of tile t (rank floor(t N / 24)) runs the
                fused decode + composite of its tiles; no gather.
Under torchrun (N GPUs): compose_tiles over NCCL, rank g holding sources
[g 64/N, (g+1) 64/N), max over ranks.

    python scripts/bench_wall.py [--steps 5]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/bench_wall.py
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1902_08755_b200 import eqc  # noqa: E402

W, H, TX, TY, N = 15360, 5760, 6, 4, 64


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, steps, stream):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--virtual", default="1,2,4")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    s = torch.cuda.current_stream()
    P = W * H
    peak = peak_gbs()
    out = {"config": "c5: 64 sources x 15360x5760 (6x4 wall of 2560x1440 tiles), F = 0.3, RLE transport",
           "hbm_peak_gbs": peak, "results": {}}
    if world == 1:
        c, d = synth.depth_sources_torch(synth.SEED_BASE + 4, N, W, H, F=0.3)
        wall = torch.empty((H, W), dtype=torch.int32, device="cuda")
        comp_bytes = (8 * N + 4) * P
        ms = timed(lambda: eqc.compositor_depth(c, d, wall), a.steps, s)
        out["results"]["composite"] = {"ms": round(ms, 3), "alg_bytes": comp_bytes,
                                       "roof_ms": round(comp_bytes / (peak * 1e9) * 1e3, 3),
                                       "frac_of_hbm_peak": round(comp_bytes / (ms * 1e-3) / 1e9 / peak, 3),
                                       "source_mpx_per_s": round(N * P / (ms * 1e-3) / 1e6, 1)}
        for nv in [int(x) for x in a.virtual.split(",")]:
            ms = timed(lambda: eqc.compose_tiles_local(nv, c, d, wall, tiles_x=TX, tiles_y=TY, flags=eqc.FLAG_RLE),
                       a.steps, s)
            out["results"][f"tiles_v{nv}"] = {"ms": round(ms, 3), "source_mpx_per_s": round(N * P / (ms * 1e-3) / 1e6, 1),
                                              "note": "virtual ranks serialised on one GPU (no overlap of ranks)"}
    else:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = eqc.Comm.from_torch_distributed()
        nl = N // world
        c, d = synth.depth_sources_torch(synth.SEED_BASE + 4, N, W, H, F=0.3,
                                         indices=range(rank * nl, (rank + 1) * nl))
        wall = torch.empty((H, W), dtype=torch.int32, device="cuda")
        for name, fl in (("tiles_rle", eqc.FLAG_RLE), ("tiles_raw", 0)):
            def f():
                eqc.compose_tiles(comm, c, d, wall, tiles_x=TX, tiles_y=TY, flags=fl)
            for _ in range(2):
                f()
            torch.cuda.synchronize()
            dist.barrier()
            ms = timed(f, a.steps, s)
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out["results"][name] = {"ms": round(float(t.item()), 3),
                                    "source_mpx_per_s": round(N * P / (float(t.item()) * 1e-3) / 1e6, 1)}
        out["n_gpus"] = world
        comm.destroy()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
