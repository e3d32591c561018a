"""A/B timing of tuning variants of libeqc on the bench workload (8 x 4K
colour + depth -> image_compress_rle_batch of 16 streams, then the fused
decode).  Builds each variant (csrc compiled with extra -D defines) next to
the default library, times it in a fresh process, and checks every variant's
streams are byte-identical to the default library's (whose parity against
the oracle is tests/test_gpu_parity.py).

    python scripts/ab_encode.py "EQC_ENC_WARPS=1" "EQC_ENC_WARPS=4" ...
    python scripts/ab_encode.py paper_1902_08755_b200/variants/libeqc_w1.so ...   (prebuilt)
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    import numpy as np
    import torch
    sys.path.insert(0, ROOT)
    import synth
    from paper_1902_08755_b200 import eqc
    W, H, N = 3840, 2160, 8
    dev = torch.device("cuda", 0)
    c, d = synth.depth_sources(synth.SEED_BASE + 10, N, W, H)  # the bench workload
    imgs = [torch.from_numpy(x.view(np.int32)).to(dev) for x in list(c) + list(d)]
    kinds, flags = [0] * N + [1] * N, [1] * N + [0] * N
    cap = eqc.image_rle_max_size(W, H)
    streams = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in imgs]
    sizes = torch.zeros(len(imgs), dtype=torch.int64, device=dev)
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(len(imgs), W, H), dtype=torch.uint8, device=dev)
    out_c = torch.empty((H, W), dtype=torch.int32, device=dev)
    out_d = torch.empty((H, W), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    res = {}
    for name, fn in [("encode", lambda: eqc.image_compress_rle_batch(imgs, kinds, flags, streams, sizes, ws)),
                     ("fused", lambda: eqc.compositor_depth_rle(streams[:N], streams[N:], out_c, out_d, status))]:
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for _ in range(15):  # 5 back-to-back calls per sample: host overhead hidden
            e[0].record()
            for _ in range(5):
                fn()
            e[1].record()
            e[1].synchronize()
            ts.append(e[0].elapsed_time(e[1]) / 5)
        ts.sort()
        res[name + "_ms"] = round(ts[len(ts) // 2], 4)
    h = hashlib.sha1()
    for s, n in zip(streams, sizes.tolist()):
        h.update(s[:n].cpu().numpy().tobytes())
    h.update(out_c.cpu().numpy().tobytes())
    res["digest"] = h.hexdigest()
    res["status"] = int(status.item())
    print("RESULT " + json.dumps(res), flush=True)


def main():
    if sys.argv[1:2] == ["--child"]:
        return child()
    sys.path.insert(0, ROOT)
    from paper_1902_08755_b200 import build
    variants = [("default", build.LIB)]
    for i, spec in enumerate(sys.argv[1:]):
        if spec.endswith(".so"):  # prebuilt variant
            variants.append((spec, os.path.abspath(spec)))
            continue
        out = os.path.join(build.HERE, "variants", f"libeqc_v{i}.so")
        os.makedirs(os.path.dirname(out), exist_ok=True)
        build.build(out=out, defines=[x for x in spec.split(",") if x])
        variants.append((spec, out))
    build.build()
    base = None
    # the first child warms the GPU (clocks, module loading) and is not reported
    for spec, lib in [("warmup", build.LIB)] + variants:
        env = dict(os.environ, EQC_LIB=lib)
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        if not line:
            print(json.dumps({"variant": spec, "error": r.stderr[-800:]}))
            continue
        res = json.loads(line[0][7:])
        if spec == "warmup":
            continue
        base = base or res["digest"]
        res["identical_to_default"] = res["digest"] == base
        res["variant"] = spec
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
