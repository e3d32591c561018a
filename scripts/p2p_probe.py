"""NVLink peer-read probe (2 GPUs, one process): bandwidth of a kernel that
reads a peer GPU's memory (compositor_depth with remote source pointers, the
pull of the peer-memory direct send) against a copy-engine peer copy."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08755_b200 import eqc
from cuda.bindings import runtime as cudart

def t(fn, steps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)

H, W = 2160, 7680  # half of an 8K frame: one direct-send band on 2 GPUs
torch.cuda.set_device(1)
rc_ = torch.randint(0, 2**31, (H, W), dtype=torch.int32, device="cuda:1")
rd_ = torch.randint(0, 2**31, (H, W), dtype=torch.int32, device="cuda:1")
torch.cuda.set_device(0)
print(cudart.cudaDeviceEnablePeerAccess(1, 0))
lc = torch.randint(0, 2**31, (H, W), dtype=torch.int32, device="cuda:0")
ld = torch.randint(0, 2**31, (H, W), dtype=torch.int32, device="cuda:0")
out = torch.empty_like(lc)
mb = H * W * 8 / 1e6
tl = t(lambda: eqc.compositor_depth([lc, lc], [ld, ld], out))
tr = t(lambda: eqc.compositor_depth([lc, rc_], [ld, rd_], out))
trr = t(lambda: eqc.compositor_depth([rc_], [rd_], out))
buf = torch.empty((2, H, W), dtype=torch.int32, device="cuda:0")
src = torch.stack([rc_, rd_])
tc = t(lambda: buf.copy_(src, non_blocking=True))
print(f"local 2 sources: {tl*1e3:.1f} us; local+remote: {tr*1e3:.1f} us; remote only (1 source): {trr*1e3:.1f} us "
      f"-> kernel pull {mb / (trr*1e-3) / 1e3:.0f} GB/s; copy-engine peer copy {mb / (tc*1e-3) / 1e3:.0f} GB/s")
