"""GPU test helpers: move seeded numpy frames to device buffers with a chosen
row pitch and back.  No method arithmetic lives here."""
import numpy as np
import torch


def to_dev(a: np.ndarray, pitch: int | None = None, offset: int = 0) -> torch.Tensor:
    """[H, W] uint32 numpy -> CUDA [H, W] view of an [H, pitch] buffer
    (starting `offset` words into it, to exercise misaligned pointers)."""
    h, w = a.shape
    P = pitch or w
    buf = torch.full((h * P + offset + 4,), 0x7E7E7E7E, dtype=torch.int64).to(torch.int32)
    buf = buf.cuda()
    view = buf[offset:offset + h * P].view(h, P)[:, :w]
    view.copy_(torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda())
    return view


def out_frame(h: int, w: int, pitch: int | None = None, offset: int = 0) -> torch.Tensor:
    P = pitch or w
    buf = torch.full((h * P + offset + 4,), 0x13579BDF, dtype=torch.int64).to(torch.int32).cuda()
    return buf[offset:offset + h * P].view(h, P)[:, :w]


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().cpu().numpy().view(np.uint32)


def stream_dev(b: bytes, pad: int = 0) -> torch.Tensor:
    arr = np.frombuffer(bytes(b) + bytes(pad), dtype=np.uint8).copy()
    return torch.from_numpy(arr).cuda()


def bytes_of(t: torch.Tensor, n: int) -> bytes:
    return t[:n].cpu().numpy().tobytes()
