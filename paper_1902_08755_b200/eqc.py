"""Thin ctypes binding of libeqc (include/eqc.h).  Argument marshalling only:
every step of the path runs in the CUDA kernels of libeqc.so.

Functions keep the C names.  Pixel buffers are passed as torch CUDA tensors
(uint32 frames [H, pitch] viewed through [:, :W], or uint8 streams) or as raw
device addresses (int).  ``stream`` is a torch.cuda.Stream, a raw handle (int)
or None (= torch's current stream).  A negative return code raises EqcError.
There is no CPU fallback: if libeqc.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# EQC_LIB selects a tuning variant built by build.build(out=..., defines=...)
LIB_PATH = os.environ.get("EQC_LIB") or os.path.join(_HERE, "libeqc.so")

OK = 0
E_INVALID, E_CAPACITY, E_CORRUPT, E_UNSUPPORTED, E_CUDA, E_NCCL = -1, -2, -3, -4, -5, -6
MAX_SOURCES = 64
KIND_RGBA8, KIND_DEPTH32 = 0, 1
FLAG_SWIZZLE = 1
FLAG_RLE64 = 2
UNIQUE_ID_BYTES = 128
OP_DEPTH = 0
OP_BLEND = 1
OP_AVERAGE = 2
FLAG_RLE = 1
FLAG_NCCL = 2
FLAG_ROI = 4
FLAG_OVERLAP = 8  # the compose overlaps other GPU work: peer pulls use <= 1 CTA per SM
P2P_PLAIN, P2P_PIPELINED, P2P_SLOTS = 0, 1, 2  # compose_direct_send_p2p_local modes


class EqcError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} ({code})")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libeqc.so not found at {LIB_PATH}: build it with "
            "`python -m paper_1902_08755_b200.build` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
    sig = {
        "eqc_strerror": ([i32], ctypes.c_char_p),
        "eqc_version": ([], i32),
        "compositor_depth": ([i32, P, P, i32, i32, i64, P, P, i64, P], i32),
        "compositor_blend_ordered": ([i32, P, P, i32, i32, i64, u32, P, i64, P], i32),
        "image_roi": ([i32, P, i32, i32, i64, u32, P, P], i32),
        "compositor_average": ([i32, P, i32, i32, i64, P, i64, P], i32),
        "compositor_depth_roi": ([i32, P, P, P, i32, i32, i64, P, P, i64, P], i32),
        "compositor_blend_ordered_roi": ([i32, P, P, P, i32, i32, i64, u32, P, i64, P], i32),
        "image_rle_max_size": ([i32, i32], i64),
        "image_rle_workspace_size": ([i32, i32], sz),
        "image_rle_workspace_size_batch": ([i32, i32, i32], sz),
        "image_compress_rle": ([P, i32, i32, i64, i32, i32, P, i64, P, P, sz, P], i32),
        "image_decompress_rle": ([P, i64, P, i64, i32, i32, P, P], i32),
        "image_compress_rle_batch": ([i32, P, i32, i32, i64, P, P, P, i64, P, P, sz, P], i32),
        "image_decompress_rle_batch": ([i32, P, P, P, i64, i32, i32, P, P], i32),
        "compositor_depth_rle": ([i32, P, P, P, P, i32, i32, P, P, i64, P, P], i32),
        # eqc_comm.h
        "eqc_comm_get_unique_id": ([P], i32),
        "eqc_comm_init": ([P, i32, i32, P], i32),
        "eqc_comm_destroy": ([P], i32),
        "eqc_comm_stats": ([P, P], i32),
        "eqc_comm_frame_buffers": ([P, i32, i32, i32, P, P, P, P], i32),
        "eqc_comm_stream_buffers": ([P, i32, i64, i32, P, P], i32),
        "compose_direct_send_rle_pull": ([P, i32, i32, i32, i32, i32, P, i64, P, P], i32),
        "compositor_depth_rle_scatter": ([P, i32, P, P, P, P, i32, i32, i32, P, P], i32),
        "compose_direct_send_scattered": ([P, i32, i32, i32, i32, P, i64, i32, P], i32),
        "compose_direct_send_scatter_local": ([i32, i32, P, P, P, P, i32, i32, i32, P, i64, P, P, P], i32),
        "compose_direct_send_p2p_local": ([i32, i32, P, P, i32, i32, i64, i32, i32, i32, i32, P, i64, P, P], i32),
        "compose_direct_send_rle_pull_local": ([i32, i32, P, i64, i32, i32, i32, P, i64, P, P, P], i32),
        "compose_binary_swap_p2p_local": ([i32, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P, P], i32),
        "compose_swap23_p2p_local": ([i32, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P, P], i32),
        "compose_tiles": ([P, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P], i32),
        "compose_tiles_local": ([i32, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P, P], i32),
        "eqc_plan_tiles": ([i32, i32, i32, i32, i32, i32, P], i32),
        "eqc_comm_check": ([P, P], i32),
        "eqc_comm_abort": ([P], i32),
        "eqc_plan_bands": ([i32, i32, P], i32),
        "eqc_plan_bands_gather": ([i32, i32, i32, P], i32),
        "eqc_plan_binary_swap": ([i32, i32, i32, P, i32], i32),
        "compose_direct_send": ([P, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P], i32),
        "compose_binary_swap": ([P, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P], i32),
        "compose_direct_send_local": ([i32, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P, P], i32),
        "compose_binary_swap_local": ([i32, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P, P], i32),
        "compose_swap23": ([P, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P], i32),
        "compose_swap23_local": ([i32, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P, P], i32),
        "eqc_plan_swap23": ([i32, i32, i32, P, i32], i32),
        "compose_stream": ([P, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P], i32),
        "compose_direct_send_roi": ([P, i32, P, P, P, i32, i32, i64, i32, i32, P, i64, P], i32),
        "compose_direct_send_roi_local": ([i32, i32, P, P, P, i32, i32, i64, i32, i32, P, i64, P, P], i32),
        "compose_stream_local": ([i32, i32, P, P, i32, i32, i64, i32, i32, i32, P, i64, P, P], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


_lib = _load()


def lib():
    return _lib


def strerror(code: int) -> str:
    return _lib.eqc_strerror(int(code)).decode()


def version() -> int:
    return int(_lib.eqc_version())


def _check(rc: int, where: str) -> int:
    if rc < 0:
        raise EqcError(rc, where)
    return rc


def _addr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _stream(s) -> int | None:
    if s is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    if isinstance(s, int):
        return s
    return int(s.cuda_stream)


def _ptrs(xs):
    return (ctypes.c_void_p * len(xs))(*[_addr(x) for x in xs])


def _frame_geom(t):
    """(w, h, pitch) of a uint32 frame tensor [H, W] with row stride pitch."""
    h, w = t.shape
    assert t.stride(1) == 1, "frames must be row-major with unit column stride"
    return w, h, t.stride(0)


def compositor_depth(colors, depths, out_color, out_depth=None, stream=None):
    n = len(colors)
    w, h, pitch = _frame_geom(colors[0])
    _, _, opitch = _frame_geom(out_color)
    rc = _lib.compositor_depth(n, _ptrs(colors), _ptrs(depths), w, h, pitch, _addr(out_color),
                               _addr(out_depth), opitch, _stream(stream))
    return _check(rc, "compositor_depth")


def compositor_blend_ordered(colors, out_color, order=None, background: int = 0, stream=None):
    n = len(colors)
    w, h, pitch = _frame_geom(colors[0])
    _, _, opitch = _frame_geom(out_color)
    ordp = None
    if order is not None:
        ordp = (ctypes.c_int32 * n)(*[int(v) for v in order])
    rc = _lib.compositor_blend_ordered(n, _ptrs(colors), ordp, w, h, pitch, int(background) & 0xFFFFFFFF,
                                       _addr(out_color), opitch, _stream(stream))
    return _check(rc, "compositor_blend_ordered")


def compositor_average(colors, out_color, stream=None):
    """Subpixel accumulation + averaging: per-channel mean, rounded half up."""
    n = len(colors)
    w, h, pitch = _frame_geom(colors[0])
    _, _, opitch = _frame_geom(out_color)
    rc = _lib.compositor_average(n, _ptrs(colors), w, h, pitch, _addr(out_color), opitch, _stream(stream))
    return _check(rc, "compositor_average")


def image_roi(frames, d_roi, background: int, stream=None):
    """ROI {x, y, w, h} of each frame's pixels != background into the device
    int32 tensor d_roi [n, 4]."""
    n = len(frames)
    w, h, pitch = _frame_geom(frames[0])
    rc = _lib.image_roi(n, _ptrs(frames), w, h, pitch, int(background) & 0xFFFFFFFF, _addr(d_roi), _stream(stream))
    return _check(rc, "image_roi")


def compositor_depth_roi(colors, depths, d_roi, out_color, out_depth=None, stream=None):
    """compositor_depth over sources holding data only inside their ROI
    (device int32 [n, 4] {x, y, w, h})."""
    n = len(colors)
    w, h, pitch = _frame_geom(colors[0])
    _, _, opitch = _frame_geom(out_color)
    rc = _lib.compositor_depth_roi(n, _ptrs(colors), _ptrs(depths), _addr(d_roi), w, h, pitch, _addr(out_color),
                                   _addr(out_depth), opitch, _stream(stream))
    return _check(rc, "compositor_depth_roi")


def compositor_blend_ordered_roi(colors, d_roi, out_color, order=None, background: int = 0, stream=None):
    n = len(colors)
    w, h, pitch = _frame_geom(colors[0])
    _, _, opitch = _frame_geom(out_color)
    ordp = None
    if order is not None:
        ordp = (ctypes.c_int32 * n)(*[int(v) for v in order])
    rc = _lib.compositor_blend_ordered_roi(n, _ptrs(colors), ordp, _addr(d_roi), w, h, pitch,
                                           int(background) & 0xFFFFFFFF, _addr(out_color), opitch, _stream(stream))
    return _check(rc, "compositor_blend_ordered_roi")


def image_rle_max_size(w: int, h: int) -> int:
    return _check(int(_lib.image_rle_max_size(w, h)), "image_rle_max_size")


def image_rle_workspace_size(w: int, h: int) -> int:
    return int(_lib.image_rle_workspace_size(w, h))


def image_rle_workspace_size_batch(count: int, w: int, h: int) -> int:
    return int(_lib.image_rle_workspace_size_batch(count, w, h))


def image_compress_rle(src, kind: int, flags: int, dst, d_size, workspace, stream=None):
    w, h, pitch = _frame_geom(src)
    rc = _lib.image_compress_rle(_addr(src), w, h, pitch, kind, flags, _addr(dst), dst.numel(),
                                 _addr(d_size), _addr(workspace), workspace.numel() * workspace.element_size(),
                                 _stream(stream))
    return _check(rc, "image_compress_rle")


def image_decompress_rle(src, dst, d_status, src_bytes: int | None = None, stream=None):
    w, h, pitch = _frame_geom(dst)
    nb = src.numel() if src_bytes is None else src_bytes
    rc = _lib.image_decompress_rle(_addr(src), nb, _addr(dst), pitch, w, h, _addr(d_status), _stream(stream))
    return _check(rc, "image_decompress_rle")


def image_compress_rle_batch(srcs, kinds, flags, dsts, d_sizes, workspace, stream=None):
    n = len(srcs)
    w, h, pitch = _frame_geom(srcs[0])
    k = (ctypes.c_int * n)(*kinds)
    f = (ctypes.c_int * n)(*flags)
    cap = min(d.numel() for d in dsts)
    rc = _lib.image_compress_rle_batch(n, _ptrs(srcs), w, h, pitch, k, f, _ptrs(dsts), cap, _addr(d_sizes),
                                       _addr(workspace), workspace.numel() * workspace.element_size(),
                                       _stream(stream))
    return _check(rc, "image_compress_rle_batch")


def _i64s(vals):
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])


def image_decompress_rle_batch(srcs, dsts, d_status, src_bytes=None, stream=None):
    """src_bytes: per-stream readable bytes (default: each tensor's numel)."""
    n = len(srcs)
    w, h, pitch = _frame_geom(dsts[0])
    nb = [s.numel() for s in srcs] if src_bytes is None else src_bytes
    rc = _lib.image_decompress_rle_batch(n, _ptrs(srcs), _i64s(nb), _ptrs(dsts), pitch, w, h, _addr(d_status),
                                         _stream(stream))
    return _check(rc, "image_decompress_rle_batch")


def compositor_depth_rle(color_streams, depth_streams, out_color, out_depth, d_status,
                         color_bytes=None, depth_bytes=None, stream=None):
    """color_bytes / depth_bytes: per-stream readable bytes (default: numel)."""
    n = len(color_streams)
    w, h, opitch = _frame_geom(out_color)
    cb = [s.numel() for s in color_streams] if color_bytes is None else color_bytes
    db = [s.numel() for s in depth_streams] if depth_bytes is None else depth_bytes
    rc = _lib.compositor_depth_rle(n, _ptrs(color_streams), _ptrs(depth_streams), _i64s(cb), _i64s(db), w, h,
                                   _addr(out_color), _addr(out_depth), opitch, _addr(d_status), _stream(stream))
    return _check(rc, "compositor_depth_rle")


# ---------------------------------------------------------------- eqc_comm.h
def eqc_plan_bands(h: int, n: int):
    """Row boundaries of the n direct-send bands (R-C13): [row0[0] .. row0[n]]."""
    row0 = (ctypes.c_int * (n + 1))()
    _check(_lib.eqc_plan_bands(h, n, row0), "eqc_plan_bands")
    return list(row0)


def eqc_plan_bands_gather(h: int, n: int, dest: int):
    """Row boundaries of the peer-memory direct send's gather-aware bands."""
    row0 = (ctypes.c_int * (n + 1))()
    _check(_lib.eqc_plan_bands_gather(h, n, dest, row0), "eqc_plan_bands_gather")
    return list(row0)


def eqc_plan_binary_swap(h: int, n: int, rank: int):
    """Rounds of rank's binary-swap plan: [(partner, low, keep_y0, keep_y1, send_y0, send_y1), ...]."""
    buf = (ctypes.c_int * (6 * 32))()
    k = _check(_lib.eqc_plan_binary_swap(h, n, rank, buf, 32), "eqc_plan_binary_swap")
    return [tuple(buf[6 * i:6 * i + 6]) for i in range(k)]


class _DeviceView:
    """A [h, w] int32 view of device memory owned by the library
    (__cuda_array_interface__, so torch.as_tensor wraps it without a copy)."""

    def __init__(self, ptr: int, h: int, w: int, typestr: str = "<i4"):
        self.__cuda_array_interface__ = {"shape": (h, w), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


class Comm:
    """An eqc_comm: NCCL clique of one process per GPU (current device)."""

    def __init__(self, nranks: int, rank: int, unique_id: bytes):
        assert len(unique_id) == UNIQUE_ID_BYTES
        self.nranks, self.rank = nranks, rank
        self._h = ctypes.c_void_p()
        idbuf = (ctypes.c_uint8 * UNIQUE_ID_BYTES)(*unique_id)
        _check(_lib.eqc_comm_init(ctypes.byref(self._h), nranks, rank, idbuf), "eqc_comm_init")

    @staticmethod
    def get_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * UNIQUE_ID_BYTES)()
        _check(_lib.eqc_comm_get_unique_id(buf), "eqc_comm_get_unique_id")
        return bytes(buf)

    @classmethod
    def from_torch_distributed(cls, group=None):
        """Bootstrap the NCCL unique id over an initialised torch.distributed group."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        del torch
        return cls(world, rank, obj[0])

    @property
    def handle(self):
        return self._h

    def check(self, stream=None):
        """eqc_comm_check: synchronise, then raise on an NCCL async error, a
        peer-memory wait that timed out, or mismatched frame slots."""
        return _check(_lib.eqc_comm_check(self._h, _stream(stream)), "eqc_comm_check")

    def abort(self):
        return _check(_lib.eqc_comm_abort(self._h), "eqc_comm_abort")

    def stats(self):
        out = (ctypes.c_int64 * 4)()
        _check(_lib.eqc_comm_stats(self._h, out), "eqc_comm_stats")
        return list(out)

    def frame_buffers(self, w: int, h: int, slot: int, stream=None):
        """eqc_comm_frame_buffers: slot `slot`'s peer-mapped (color, depth)
        partial-frame buffers and the comm's gather buffer, as [h, w] int32
        tensor views of comm-owned memory (collective); None when the ranks
        cannot map each other's memory (E_UNSUPPORTED)."""
        import torch
        c, d, f = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        rc = _lib.eqc_comm_frame_buffers(self._h, w, h, slot, ctypes.byref(c), ctypes.byref(d), ctypes.byref(f),
                                         _stream(stream))
        if rc == E_UNSUPPORTED:
            return None
        _check(rc, "eqc_comm_frame_buffers")
        dev = torch.cuda.current_device()
        return tuple(torch.as_tensor(_DeviceView(x.value, h, w), device=f"cuda:{dev}") for x in (c, d, f))

    def stream_buffers(self, n_streams: int, cap_bytes: int, slot: int, stream=None):
        """eqc_comm_stream_buffers: slot `slot`'s peer-mapped RLE stream
        buffers as uint8 tensor views of comm-owned memory (collective);
        None when the ranks cannot map each other's memory."""
        import torch
        ptrs = (ctypes.c_void_p * n_streams)()
        rc = _lib.eqc_comm_stream_buffers(self._h, n_streams, cap_bytes, slot, ptrs, _stream(stream))
        if rc == E_UNSUPPORTED:
            return None
        _check(rc, "eqc_comm_stream_buffers")
        dev = torch.cuda.current_device()
        return [torch.as_tensor(_DeviceView(p, cap_bytes, 1, "|u1"), device=f"cuda:{dev}").view(-1) for p in ptrs]

    def destroy(self):
        if self._h:
            _check(_lib.eqc_comm_destroy(self._h), "eqc_comm_destroy")
            self._h = ctypes.c_void_p()


def _compose(fn, name, comm, colors, depths, out_color, dest_rank, flags, op, stream):
    n = len(colors)
    w, h, pitch = _frame_geom(colors[0])
    opitch = _frame_geom(out_color)[2] if out_color is not None else w
    rc = fn(comm.handle, n, _ptrs(colors), _ptrs(depths) if depths is not None else None, w, h, pitch, op, flags,
            dest_rank, _addr(out_color),
            opitch, _stream(stream))
    return _check(rc, name)


def compose_direct_send_rle_pull(comm, n_local: int, w: int, h: int, slot: int, out_color=None, status=None,
                                 dest_rank: int = 0, stream=None):
    """compose_direct_send_rle_pull: direct send of the RLE streams in stream
    slot `slot` (decoder pulls the peers' records over NVLink)."""
    opitch = _frame_geom(out_color)[2] if out_color is not None else w
    return _check(_lib.compose_direct_send_rle_pull(comm.handle, n_local, w, h, slot, dest_rank, _addr(out_color),
                                                    opitch, _addr(status), _stream(stream)),
                  "compose_direct_send_rle_pull")


def compositor_depth_rle_scatter(comm, color_streams, depth_streams, w: int, h: int, slot: int, d_status,
                                 color_bytes=None, depth_bytes=None, stream=None):
    """compositor_depth_rle_scatter: fused decode + depth composite of this
    rank's sources, band j stored into rank j's frame slot `slot`."""
    n = len(color_streams)
    cb = [s.numel() for s in color_streams] if color_bytes is None else color_bytes
    db = [s.numel() for s in depth_streams] if depth_bytes is None else depth_bytes
    return _check(_lib.compositor_depth_rle_scatter(comm.handle, n, _ptrs(color_streams), _ptrs(depth_streams),
                                                    _i64s(cb), _i64s(db), w, h, slot, _addr(d_status),
                                                    _stream(stream)), "compositor_depth_rle_scatter")


def compose_direct_send_scattered(comm, w: int, h: int, slot: int, out_color=None, dest_rank: int = 0,
                                  flags: int = 0, stream=None):
    """compose_direct_send_scattered: band composite of the copies the peers
    scattered into frame slot `slot`; colour to dest_rank's out_color."""
    opitch = _frame_geom(out_color)[2] if out_color is not None else w
    return _check(_lib.compose_direct_send_scattered(comm.handle, w, h, slot, dest_rank, _addr(out_color), opitch,
                                                     flags, _stream(stream)), "compose_direct_send_scattered")


def compose_direct_send(comm, colors, depths, out_color=None, dest_rank: int = 0, flags: int = 0,
                        op: int = OP_DEPTH, stream=None):
    return _compose(_lib.compose_direct_send, "compose_direct_send", comm, colors, depths, out_color, dest_rank,
                    flags, op, stream)


def compose_binary_swap(comm, colors, depths, out_color=None, dest_rank: int = 0, flags: int = 0,
                        op: int = OP_DEPTH, stream=None):
    return _compose(_lib.compose_binary_swap, "compose_binary_swap", comm, colors, depths, out_color, dest_rank,
                    flags, op, stream)


def _compose_local(fn, name, nranks, colors, depths, out_color, dest_rank, flags, op, stream):
    total = len(colors)
    assert total % nranks == 0
    w, h, pitch = _frame_geom(colors[0])
    opitch = _frame_geom(out_color)[2]
    stats = (ctypes.c_int64 * 4)()
    rc = fn(nranks, total // nranks, _ptrs(colors), _ptrs(depths) if depths is not None else None, w, h, pitch, op,
            flags, dest_rank,
            _addr(out_color), opitch, stats, _stream(stream))
    _check(rc, name)
    return list(stats)


def compose_direct_send_local(nranks, colors, depths, out_color, dest_rank: int = 0, flags: int = 0,
                              op: int = OP_DEPTH, stream=None):
    """Virtual-rank direct send on one GPU; returns summed traffic counters."""
    return _compose_local(_lib.compose_direct_send_local, "compose_direct_send_local", nranks, colors, depths,
                          out_color, dest_rank, flags, op, stream)


def compose_direct_send_p2p_local(nranks, colors, depths, out_color, dest_rank: int = 0, flags: int = 0,
                                  op: int = OP_DEPTH, mode: int = P2P_PLAIN, stream=None):
    """The peer-memory direct send for virtual ranks on one GPU (same host code
    and kernels as the multi-process path); returns summed traffic counters."""
    total = len(colors)
    assert total % nranks == 0
    w, h, pitch = _frame_geom(colors[0])
    opitch = _frame_geom(out_color)[2]
    stats = (ctypes.c_int64 * 4)()
    rc = _lib.compose_direct_send_p2p_local(nranks, total // nranks, _ptrs(colors),
                                            _ptrs(depths) if depths is not None else None, w, h, pitch, op, flags,
                                            mode, dest_rank, _addr(out_color), opitch, stats, _stream(stream))
    _check(rc, "compose_direct_send_p2p_local")
    return list(stats)


def plan_tiles(w: int, h: int, tiles_x: int, tiles_y: int, nranks: int, tile: int):
    """(x0, y0, w, h, owner) of a display-wall tile (eqc_plan_tiles)."""
    r = (ctypes.c_int * 5)()
    _check(_lib.eqc_plan_tiles(w, h, tiles_x, tiles_y, nranks, tile, r), "eqc_plan_tiles")
    return tuple(r)


def compose_tiles(comm, colors, depths, out_color, tiles_x: int = 6, tiles_y: int = 4, flags: int = FLAG_RLE,
                  stream=None):
    """Display-wall direct send (c5): every rank writes the tiles it owns into out_color."""
    w, h, pitch = _frame_geom(colors[0])
    opitch = _frame_geom(out_color)[2]
    return _check(_lib.compose_tiles(comm.handle, len(colors), _ptrs(colors), _ptrs(depths), w, h, pitch, tiles_x,
                                     tiles_y, flags, _addr(out_color), opitch, _stream(stream)), "compose_tiles")


def compose_tiles_local(nranks, colors, depths, out_color, tiles_x: int = 6, tiles_y: int = 4,
                        flags: int = FLAG_RLE, stream=None):
    """compose_tiles for virtual ranks on one GPU; returns summed traffic counters."""
    total = len(colors)
    assert total % nranks == 0
    w, h, pitch = _frame_geom(colors[0])
    opitch = _frame_geom(out_color)[2]
    stats = (ctypes.c_int64 * 4)()
    rc = _lib.compose_tiles_local(nranks, total // nranks, _ptrs(colors), _ptrs(depths), w, h, pitch, tiles_x,
                                  tiles_y, flags, _addr(out_color), opitch, stats, _stream(stream))
    _check(rc, "compose_tiles_local")
    return list(stats)


def compose_binary_swap_p2p_local(nranks, colors, depths, out_color, dest_rank: int = 0, flags: int = 0,
                                  op: int = OP_DEPTH, stream=None):
    """The peer-memory binary swap for virtual ranks on one GPU."""
    return _compose_local(_lib.compose_binary_swap_p2p_local, "compose_binary_swap_p2p_local", nranks, colors,
                          depths, out_color, dest_rank, flags, op, stream)


def compose_swap23_p2p_local(nranks, colors, depths, out_color, dest_rank: int = 0, flags: int = 0,
                             op: int = OP_DEPTH, stream=None):
    """The peer-memory 2-3 swap for virtual ranks on one GPU."""
    return _compose_local(_lib.compose_swap23_p2p_local, "compose_swap23_p2p_local", nranks, colors, depths,
                          out_color, dest_rank, flags, op, stream)


def compose_direct_send_rle_pull_local(nranks, n_local, rank_streams, cap_bytes, w, h, out_color, status,
                                       dest_rank: int = 0, stream=None):
    """compose_direct_send_rle_pull for virtual ranks on one GPU: rank q's
    2*n_local streams lie contiguously (cap_bytes apart) at rank_streams[q]."""
    opitch = _frame_geom(out_color)[2]
    stats = (ctypes.c_int64 * 4)()
    rc = _lib.compose_direct_send_rle_pull_local(nranks, n_local, _ptrs(rank_streams), cap_bytes, w, h, dest_rank,
                                                 _addr(out_color), opitch, _addr(status), stats, _stream(stream))
    _check(rc, "compose_direct_send_rle_pull_local")
    return list(stats)


def compose_direct_send_scatter_local(nranks, color_streams, depth_streams, w, h, out_color, status,
                                      dest_rank: int = 0, color_bytes=None, depth_bytes=None, stream=None):
    """compositor_depth_rle_scatter + compose_direct_send_scattered for
    virtual ranks on one GPU: rank q's streams are
    color_streams[q * n_local : (q + 1) * n_local] (and depth)."""
    total = len(color_streams)
    assert total % nranks == 0 and len(depth_streams) == total
    cb = [x.numel() for x in color_streams] if color_bytes is None else color_bytes
    db = [x.numel() for x in depth_streams] if depth_bytes is None else depth_bytes
    opitch = _frame_geom(out_color)[2]
    stats = (ctypes.c_int64 * 4)()
    rc = _lib.compose_direct_send_scatter_local(nranks, total // nranks, _ptrs(color_streams), _ptrs(depth_streams),
                                                _i64s(cb), _i64s(db), w, h, dest_rank, _addr(out_color), opitch,
                                                _addr(status), stats, _stream(stream))
    _check(rc, "compose_direct_send_scatter_local")
    return list(stats)


def compose_binary_swap_local(nranks, colors, depths, out_color, dest_rank: int = 0, flags: int = 0,
                              op: int = OP_DEPTH, stream=None):
    return _compose_local(_lib.compose_binary_swap_local, "compose_binary_swap_local", nranks, colors, depths,
                          out_color, dest_rank, flags, op, stream)


def compose_swap23(comm, colors, depths, out_color=None, dest_rank: int = 0, flags: int = 0,
                   op: int = OP_DEPTH, stream=None):
    """2-3 swap (any number of ranks; R-C21)."""
    return _compose(_lib.compose_swap23, "compose_swap23", comm, colors, depths, out_color, dest_rank,
                    flags, op, stream)


def compose_swap23_local(nranks, colors, depths, out_color, dest_rank: int = 0, flags: int = 0,
                         op: int = OP_DEPTH, stream=None):
    return _compose_local(_lib.compose_swap23_local, "compose_swap23_local", nranks, colors, depths,
                          out_color, dest_rank, flags, op, stream)


def eqc_plan_swap23(h: int, n: int, rank: int):
    """Plan of `rank`: dict(fold_role, fold_partner, final=(y0, y1), rounds=[dict(k, t, members, bounds)])."""
    buf = (ctypes.c_int * (5 + 9 * 64))()
    k = _check(_lib.eqc_plan_swap23(h, n, rank, buf, len(buf)), "eqc_plan_swap23")
    v = list(buf)
    rounds = []
    for i in range(k):
        o = v[5 + 9 * i: 14 + 9 * i]
        rounds.append({"k": o[0], "t": o[1], "members": [m for m in o[2:5] if m >= 0][:o[0]],
                       "bounds": o[5:6 + o[0]]})
    return {"fold_role": v[0], "fold_partner": v[1], "final": (v[3], v[4]), "rounds": rounds}


def compose_stream(comm, colors, depths, out_color=None, dest_rank: int = 0, flags: int = 0,
                   op: int = OP_DEPTH, stream=None):
    """Streaming sort-last chain 0 -> 1 -> ... -> n-1."""
    return _compose(_lib.compose_stream, "compose_stream", comm, colors, depths, out_color, dest_rank,
                    flags, op, stream)


def compose_stream_local(nranks, colors, depths, out_color, dest_rank: int = 0, flags: int = 0,
                         op: int = OP_DEPTH, stream=None):
    return _compose_local(_lib.compose_stream_local, "compose_stream_local", nranks, colors, depths,
                          out_color, dest_rank, flags, op, stream)


def compose_direct_send_roi(comm, colors, depths, d_src_roi, out_color=None, dest_rank: int = 0, flags: int = 0,
                            stream=None):
    """Direct send with application-provided source ROIs (device int32 [n_local, 4])."""
    n = len(colors)
    w, h, pitch = _frame_geom(colors[0])
    opitch = _frame_geom(out_color)[2] if out_color is not None else w
    rc = _lib.compose_direct_send_roi(comm.handle, n, _ptrs(colors), _ptrs(depths), _addr(d_src_roi), w, h, pitch,
                                      flags, dest_rank, _addr(out_color), opitch, _stream(stream))
    return _check(rc, "compose_direct_send_roi")


def compose_direct_send_roi_local(nranks, colors, depths, d_src_roi, out_color, dest_rank: int = 0, flags: int = 0,
                                  stream=None):
    total = len(colors)
    w, h, pitch = _frame_geom(colors[0])
    opitch = _frame_geom(out_color)[2]
    stats = (ctypes.c_int64 * 4)()
    rc = _lib.compose_direct_send_roi_local(nranks, total // nranks, _ptrs(colors), _ptrs(depths), _addr(d_src_roi),
                                            w, h, pitch, flags, dest_rank, _addr(out_color), opitch, stats,
                                            _stream(stream))
    _check(rc, "compose_direct_send_roi_local")
    return list(stats)
