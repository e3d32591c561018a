"""CPU oracle for the sort-last compositing + RLE transport hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_1902_08755_b200`` never imports it, and
this package imports nothing from the product.

The arithmetic lives in ``eqc_oracle.c`` (plain single-threaded C, one function
per definition in the thesis, each citing the passage it follows).  This module
only compiles it with gcc and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eqc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, E_INVALID, E_CAPACITY, E_CORRUPT, E_UNSUPPORTED = 0, -1, -2, -3, -4
KIND_RGBA8, KIND_DEPTH32 = 0, 1
FLAG_SWIZZLE = 1


def build(force: bool = False) -> str:
    """Compile eqc_oracle.c -> liboracle.so (gcc, -O2, no vectorisation tricks)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-Wall", "-Wextra", "-shared", "-fPIC",
             "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u32 = ctypes.c_int, ctypes.c_int64, ctypes.c_uint32
        L.or_depth_composite.argtypes = [i32, P, P, i32, i32, i64, P, P, i64]
        L.or_depth_composite.restype = None
        L.or_blend_ordered.argtypes = [i32, P, P, i32, i32, i64, u32, P, i64]
        L.or_blend_ordered.restype = None
        L.or_swizzle.argtypes = [u32]
        L.or_swizzle.restype = u32
        L.or_unswizzle.argtypes = [u32]
        L.or_unswizzle.restype = u32
        L.or_rle_max_size.argtypes = [i32, i32, i32]
        L.or_rle_max_size.restype = i64
        L.or_rle_encode_plane.argtypes = [P, i32, P]
        L.or_rle_encode_plane.restype = i32
        L.or_rle_decode_plane.argtypes = [P, i32, i32, P]
        L.or_rle_decode_plane.restype = i32
        L.or_rle_encode.argtypes = [P, i32, i32, i64, i32, i32, i32, P, i64]
        L.or_rle_encode.restype = i64
        L.or_rle_decode.argtypes = [P, i64, P, i64, i32, i32]
        L.or_rle_decode.restype = i32
        L.or_roi.argtypes = [P, i32, i32, i64, u32, P]
        L.or_roi.restype = None
        L.or_depth_composite_roi.argtypes = [i32, P, P, P, i32, i32, i64, P, P, i64]
        L.or_depth_composite_roi.restype = i32
        L.or_blend_ordered_roi.argtypes = [i32, P, P, P, i32, i32, i64, u32, P, i64]
        L.or_blend_ordered_roi.restype = i32
        L.or_average.argtypes = [i32, P, i32, i32, i64, P, i64]
        L.or_average.restype = None
        L.or_rle64_encode_chunk.argtypes = [P, i32, P]
        L.or_rle64_encode_chunk.restype = i32
        L.or_rle64_encode.argtypes = [P, i32, i32, i64, i32, P, i64]
        L.or_rle64_encode.restype = i64
        L.or_rle64_decode.argtypes = [P, i64, P, i64, i32, i32]
        L.or_rle64_decode.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _ptr_array(arrs):
    return (ctypes.c_void_p * len(arrs))(*[_ptr(a) for a in arrs])


def _as_u32_frames(frames):
    out = []
    for f in frames:
        f = np.ascontiguousarray(f, dtype=np.uint32) if f.dtype != np.uint32 or f.strides[-1] != 4 else f
        out.append(f)
    return out


def depth_composite(colors, depths, want_depth: bool = True):
    """O1: per pixel, colour/depth of the source with the smallest (depth, index).

    colors, depths: sequences of [H, W] (or [H, pitch] views) uint32 arrays.
    Returns (out_color [H, W], out_depth [H, W] or None).
    """
    n = len(colors)
    assert n == len(depths) and n >= 1
    colors = _as_u32_frames(colors)
    depths = _as_u32_frames(depths)
    h, w = colors[0].shape
    pitch = colors[0].strides[0] // 4
    for a in list(colors) + list(depths):
        assert a.shape == (h, w) and a.strides == colors[0].strides
    oc = np.empty((h, w), np.uint32)
    od = np.empty((h, w), np.uint32) if want_depth else None
    lib().or_depth_composite(n, _ptr_array(colors), _ptr_array(depths), w, h, pitch,
                             _ptr(oc), _ptr(od) if od is not None else None, w)
    return oc, od


def blend_ordered(colors, order=None, background: int = 0):
    """O2: exact back-to-front premultiplied 'over' with one final rounding."""
    n = len(colors)
    colors = _as_u32_frames(colors)
    h, w = colors[0].shape
    pitch = colors[0].strides[0] // 4
    for a in colors:
        assert a.shape == (h, w) and a.strides == colors[0].strides
    oc = np.empty((h, w), np.uint32)
    ordp = None
    if order is not None:
        order = np.ascontiguousarray(order, dtype=np.int32)
        assert order.shape == (n,)
        ordp = _ptr(order)
    lib().or_blend_ordered(n, _ptr_array(colors), ordp, w, h, pitch,
                           int(background) & 0xFFFFFFFF, _ptr(oc), w)
    return oc


def swizzle(v: int) -> int:
    return int(lib().or_swizzle(int(v) & 0xFFFFFFFF))


def unswizzle(v: int) -> int:
    return int(lib().or_unswizzle(int(v) & 0xFFFFFFFF))


def rle_max_size(w: int, h: int, log2c: int = 7) -> int:
    return int(lib().or_rle_max_size(w, h, log2c))


def rle_encode_plane(b: bytes) -> bytes:
    buf = np.frombuffer(bytes(b), np.uint8).copy()
    out = np.zeros(len(b) + 2, np.uint8)
    n = lib().or_rle_encode_plane(_ptr(buf), len(b), _ptr(out))
    return out[:n].tobytes()


def rle_decode_plane(rec: bytes, L: int):
    buf = np.frombuffer(bytes(rec), np.uint8).copy() if len(rec) else np.zeros(1, np.uint8)
    out = np.zeros(max(L, 1), np.uint8)
    rc = lib().or_rle_decode_plane(_ptr(buf), len(rec), L, _ptr(out))
    return rc, out[:L].tobytes()


def rle_encode(img: np.ndarray, kind: int = KIND_RGBA8, flags: int = 0, log2c: int = 7) -> bytes:
    """Encode a [H, W] uint32 image (or row-pitched view) into an RLE-BP v1 stream."""
    assert img.dtype == np.uint32 and img.ndim == 2 and img.strides[1] == 4
    h, w = img.shape
    pitch = img.strides[0] // 4
    cap = rle_max_size(w, h, log2c)
    out = np.empty(cap, np.uint8)
    n = lib().or_rle_encode(_ptr(img), w, h, pitch, kind, flags, log2c, _ptr(out), cap)
    if n < 0:
        raise ValueError(f"or_rle_encode failed: {n}")
    return out[:n].tobytes()


def rle_decode(stream: bytes, w: int, h: int):
    """Decode; returns (rc, [H, W] uint32 image)."""
    buf = np.frombuffer(bytes(stream), np.uint8).copy() if len(stream) else np.zeros(1, np.uint8)
    out = np.zeros((h, w), np.uint32)
    rc = lib().or_rle_decode(_ptr(buf), len(stream), _ptr(out), w, w, h)
    return rc, out


def roi(frame: np.ndarray, background: int) -> tuple:
    """Bounding box (x, y, w, h) of the pixels != background; (0, 0, 0, 0) if none."""
    f = _as_u32_frames([frame])[0]
    h, w = f.shape
    out = np.zeros(4, np.int32)
    lib().or_roi(_ptr(f), w, h, f.strides[0] // 4, int(background) & 0xFFFFFFFF, _ptr(out))
    return tuple(int(v) for v in out)


def _rois(rois, n):
    r = np.ascontiguousarray(np.asarray(rois, dtype=np.int32).reshape(n, 4))
    return r


def depth_composite_roi(colors, depths, rois, want_depth: bool = True):
    """O1 over sources that hold data only inside their ROI (x, y, w, h)."""
    n = len(colors)
    colors = _as_u32_frames(colors)
    depths = _as_u32_frames(depths)
    h, w = colors[0].shape
    pitch = colors[0].strides[0] // 4
    r = _rois(rois, n)
    oc = np.empty((h, w), np.uint32)
    od = np.empty((h, w), np.uint32) if want_depth else None
    rc = lib().or_depth_composite_roi(n, _ptr_array(colors), _ptr_array(depths), _ptr(r), w, h, pitch,
                                      _ptr(oc), _ptr(od) if od is not None else None, w)
    if rc:
        raise ValueError(f"or_depth_composite_roi: {rc}")
    return oc, od


def blend_ordered_roi(colors, rois, order=None, background: int = 0):
    """O2 over layers that are transparent outside their ROI (x, y, w, h)."""
    n = len(colors)
    colors = _as_u32_frames(colors)
    h, w = colors[0].shape
    pitch = colors[0].strides[0] // 4
    r = _rois(rois, n)
    ordp = None
    if order is not None:
        order = np.ascontiguousarray(order, dtype=np.int32)
        ordp = _ptr(order)
    oc = np.empty((h, w), np.uint32)
    rc = lib().or_blend_ordered_roi(n, _ptr_array(colors), ordp, _ptr(r), w, h, pitch,
                                    int(background) & 0xFFFFFFFF, _ptr(oc), w)
    if rc:
        raise ValueError(f"or_blend_ordered_roi: {rc}")
    return oc


def average(colors):
    """Subpixel accumulation + averaging: per channel round-half-up mean."""
    n = len(colors)
    colors = _as_u32_frames(colors)
    h, w = colors[0].shape
    pitch = colors[0].strides[0] // 4
    oc = np.empty((h, w), np.uint32)
    lib().or_average(n, _ptr_array(colors), w, h, pitch, _ptr(oc), w)
    return oc


FLAG_RLE64 = 2


def rle64_encode_chunk(pixels) -> bytes:
    """RLE-64 record of one chunk of L <= 128 uint32 pixels (R-C17)."""
    px = np.ascontiguousarray(np.asarray(pixels, dtype=np.uint32))
    out = np.zeros(1 + 64 + 8 * 64, np.uint8)
    n = lib().or_rle64_encode_chunk(_ptr(px), len(px), _ptr(out))
    return out[:n].tobytes()


def rle64_encode(img: np.ndarray, kind: int = KIND_RGBA8) -> bytes:
    assert img.dtype == np.uint32 and img.ndim == 2 and img.strides[1] == 4
    h, w = img.shape
    cap = rle_max_size(w, h, 7)
    out = np.empty(cap, np.uint8)
    n = lib().or_rle64_encode(_ptr(img), w, h, img.strides[0] // 4, kind, _ptr(out), cap)
    if n < 0:
        raise ValueError(f"or_rle64_encode failed: {n}")
    return out[:n].tobytes()


def rle64_decode(stream: bytes, w: int, h: int):
    buf = np.frombuffer(bytes(stream), np.uint8).copy() if len(stream) else np.zeros(1, np.uint8)
    out = np.zeros((h, w), np.uint32)
    rc = lib().or_rle64_decode(_ptr(buf), len(stream), _ptr(out), w, w, h)
    return rc, out
