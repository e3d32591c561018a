"""CPU-side checks of the C ABI (no GPU needed): libeqc.so builds for sm_100a,
loads, exports every function include/*.h declares, and rejects invalid
arguments on the host before touching the device."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libeqc():
    from paper_1902_08755_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M):
            name = m.group(1)
            if name not in ("if", "while", "return", "sizeof"):
                names.append(name)
    return sorted(set(names))


def test_header_declares_the_six_calls():
    names = declared_functions()
    for n in ["compositor_depth", "compositor_blend_ordered", "image_compress_rle",
              "image_decompress_rle", "compose_direct_send", "compose_binary_swap"]:
        assert n in names, n


def test_every_declared_symbol_is_exported(libeqc):
    from paper_1902_08755_b200 import build
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_sm100a_code_only(libeqc):
    from paper_1902_08755_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_binding_and_strerror():
    from paper_1902_08755_b200 import eqc
    assert eqc.strerror(0) == "EQC_OK"
    assert "CORRUPT" in eqc.strerror(-3)
    assert eqc.version() >= 0x000100


def test_max_size_matches_format_bound():
    """32 + 16*ceil(w/128)*h + 4*w*h; equals the oracle's bound."""
    import oracle
    from paper_1902_08755_b200 import eqc
    for w, h in [(1, 1), (64, 64), (1920, 1080), (3840, 2160), (129, 3)]:
        assert eqc.image_rle_max_size(w, h) == oracle.rle_max_size(w, h, 7)
    with pytest.raises(eqc.EqcError):
        eqc.image_rle_max_size(0, 5)
    assert eqc.image_rle_workspace_size(3840, 2160) > 0


def test_host_validation_rejects_before_launch(libeqc):
    L = libeqc
    P = ctypes.c_void_p
    L.compositor_depth.argtypes = [ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, P, P,
                                   ctypes.c_int64, P]
    fake = (ctypes.c_void_p * 2)(0x1000, 0x2000)
    # n out of range, w <= 0, pitch < w, null output
    assert L.compositor_depth(0, fake, fake, 4, 4, 4, 0x3000, None, 4, None) == -1
    assert L.compositor_depth(65, fake, fake, 4, 4, 4, 0x3000, None, 4, None) == -1
    assert L.compositor_depth(2, fake, fake, 0, 4, 4, 0x3000, None, 4, None) == -1
    assert L.compositor_depth(2, fake, fake, 8, 4, 4, 0x3000, None, 8, None) == -1
    assert L.compositor_depth(2, fake, fake, 4, 4, 4, None, None, 4, None) == -1
    L.compositor_blend_ordered.argtypes = [ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                           ctypes.c_uint32, P, ctypes.c_int64, P]
    bad_order = (ctypes.c_int32 * 2)(0, 0)
    assert L.compositor_blend_ordered(2, fake, bad_order, 4, 4, 4, 0, 0x3000, 4, None) == -1
    L.image_compress_rle.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                     P, ctypes.c_int64, P, P, ctypes.c_size_t, P]
    # swizzle on depth is unsupported (R-C11); too-small destination is a capacity error
    assert L.image_compress_rle(0x1000, 4, 4, 4, 1, 1, 0x2000, 1 << 20, 0x3000, 0x4000, 1 << 20, None) == -4
    assert L.image_compress_rle(0x1000, 4, 4, 4, 0, 0, 0x2000, 10, 0x3000, 0x4000, 1 << 20, None) == -2
    assert L.image_compress_rle(0x1000, 4, 4, 4, 2, 0, 0x2000, 1 << 20, 0x3000, 0x4000, 1 << 20, None) == -1


def test_comm_frame_buffers_and_flags_validation(libeqc):
    """eqc_comm_frame_buffers rejects a null comm / bad slot / null outputs on
    the host; compose rejects unknown flag bits (EQC_FLAG_OVERLAP = 8 is known)."""
    L = libeqc
    P = ctypes.c_void_p
    L.eqc_comm_frame_buffers.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P]
    c, d, f = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    refs = [ctypes.byref(c), ctypes.byref(d), ctypes.byref(f)]
    assert L.eqc_comm_frame_buffers(None, 64, 64, 0, *refs, None) == -1
    assert L.eqc_comm_frame_buffers(0x1000, 64, 64, 2, *refs, None) == -1
    assert L.eqc_comm_frame_buffers(0x1000, 0, 64, 0, *refs, None) == -1
    assert L.eqc_comm_frame_buffers(0x1000, 64, 64, 0, None, refs[1], refs[2], None) == -1
    L.compose_direct_send_local.argtypes = [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P,
                                            ctypes.c_int64, P, P]
    fake = (ctypes.c_void_p * 2)(0x1000, 0x2000)
    assert L.compose_direct_send_local(2, 1, fake, fake, 4, 4, 4, 0, 16, 0, 0x3000, 4, None, None) == -1
    from paper_1902_08755_b200 import eqc
    assert eqc.FLAG_OVERLAP == 8
