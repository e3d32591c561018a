"""GPU parity of the region-of-interest calls against the
oracle: image_roi bit-exact (bounding boxes), compositor_depth_roi bit-exact,
compositor_blend_ordered_roi within 1/255.  Cases: compact and scattered
sort-last scenes, ROIs straight from image_roi (device, no host sync), random
and unaligned rectangles, empty / full / out-of-frame (clipped) rectangles,
pitch > width, misaligned pointers, ragged widths."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import out_frame, to_dev, to_host  # noqa: E402

BG = 0xFFFFFFFF


@pytest.fixture(scope="module")
def eqc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1902_08755_b200 import eqc as m
    return m


def roi_tensor(rois):
    return torch.tensor(np.asarray(rois, np.int32).reshape(-1, 4), dtype=torch.int32, device="cuda")


ROI_CASES = [
    ("compact_8x640x360", 8, 640, 360, None, 0, "compact"),
    ("scattered_4x300x77", 4, 300, 77, None, 0, "scattered"),
    ("pitch_3x129x40_p136", 3, 129, 40, 136, 0, "compact"),
    ("misaligned_5x64x9", 5, 64, 9, 64, 1, "compact"),
    ("sparse_6x257x33", 6, 257, 33, None, 0, "sparse"),
]


def _scene(kind, n, w, h, seed):
    if kind in ("compact", "scattered"):
        return synth.depth_sources(seed, n, w, h, mode=kind)
    rng = np.random.default_rng(seed)
    c = [np.zeros((h, w), np.uint32) for _ in range(n)]
    d = [np.full((h, w), BG, np.uint32) for _ in range(n)]
    for i in range(1, n):  # source 0 stays empty; others get 0..4 random pixels
        for _ in range(i % 5):
            y, x = int(rng.integers(0, h)), int(rng.integers(0, w))
            d[i][y, x] = int(rng.integers(0, BG))
            c[i][y, x] = int(rng.integers(1, 1 << 32))
    return c, d


@pytest.mark.parametrize("case", ROI_CASES, ids=[c[0] for c in ROI_CASES])
def test_image_roi_bit_exact(eqc, case):
    name, n, w, h, pitch, offset, kind = case
    c, d = _scene(kind, n, w, h, synth.SEED_BASE + 60 + n)
    dd = [to_dev(x, pitch, offset) for x in d]
    dc = [to_dev(x, pitch, offset) for x in c]
    r = torch.full((n, 4), -7, dtype=torch.int32, device="cuda")
    eqc.image_roi(dd, r, BG)
    want = [oracle.roi(x, BG) for x in d]
    assert [tuple(v) for v in r.cpu().tolist()] == want
    eqc.image_roi(dc, r, 0)  # colour buffers against background colour 0
    assert [tuple(v) for v in r.cpu().tolist()] == [oracle.roi(x, 0) for x in c]


@pytest.mark.parametrize("case", ROI_CASES, ids=[c[0] for c in ROI_CASES])
def test_depth_roi_from_image_roi(eqc, case):
    # ROI computed on the device feeds the composite with no host round trip
    name, n, w, h, pitch, offset, kind = case
    c, d = _scene(kind, n, w, h, synth.SEED_BASE + 61 + n)
    dc = [to_dev(x, pitch, offset) for x in c]
    dd = [to_dev(x, pitch, offset) for x in d]
    r = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
    eqc.image_roi(dd, r, BG)
    oc, od = out_frame(h, w, pitch, offset), out_frame(h, w, pitch, offset)
    eqc.compositor_depth_roi(dc, dd, r, oc, od)
    rois = [oracle.roi(x, BG) for x in d]
    want_c, want_d = oracle.depth_composite_roi(c, d, rois)
    np.testing.assert_array_equal(to_host(oc), want_c)
    np.testing.assert_array_equal(to_host(od), want_d)
    # and (the ROI premise) the full-frame composite is unchanged
    full_c, full_d = oracle.depth_composite(c, d)
    np.testing.assert_array_equal(to_host(oc), full_c)


@pytest.mark.parametrize("w,h,pitch,offset", [(97, 31, None, 0), (256, 20, 260, 0), (64, 8, 64, 3)])
def test_depth_roi_random_rects(eqc, w, h, pitch, offset):
    rng = np.random.default_rng(w * h)
    n = 6
    c, d = synth.random_frames(synth.SEED_BASE + 62, n, w, h, depth_alphabet=[0, 3, 3, 8, BG])
    rois = []
    for i in range(n):
        x0, x1 = sorted(int(v) for v in rng.integers(-3, w + 4, size=2))
        y0, y1 = sorted(int(v) for v in rng.integers(-3, h + 4, size=2))
        rois.append((x0, y0, x1 - x0, y1 - y0))  # partly outside -> clipped (R-C19)
    rois[1] = (0, 0, 0, 0)
    rois[2] = (0, 0, w, h)
    dc = [to_dev(x, pitch, offset) for x in c]
    dd = [to_dev(x, pitch, offset) for x in d]
    oc, od = out_frame(h, w, pitch, offset), out_frame(h, w, pitch, offset)
    eqc.compositor_depth_roi(dc, dd, roi_tensor(rois), oc, od)
    want_c, want_d = oracle.depth_composite_roi(c, d, rois)
    np.testing.assert_array_equal(to_host(oc), want_c)
    np.testing.assert_array_equal(to_host(od), want_d)
    eqc.compositor_depth_roi(dc, dd, roi_tensor(rois), oc)  # colour only
    np.testing.assert_array_equal(to_host(oc), want_c)


def test_depth_roi_cropped_buffers(eqc):
    # cropped buffers holding only the ROI, passed as crop - (y * pitch + x)
    n, w, h = 4, 512, 200
    c, d = synth.depth_sources(synth.SEED_BASE + 63, n, w, h, mode="compact")
    rois = [oracle.roi(x, BG) for x in d]
    pitch = 520
    crops_c, crops_d, views_c, views_d = [], [], [], []
    for (x, y, rw, rh), ci, di in zip(rois, c, d):
        for src, crops, views in ((ci, crops_c, views_c), (di, crops_d, views_d)):
            buf = torch.zeros((max(rh, 1) * pitch + 8,), dtype=torch.int32, device="cuda")
            blk = buf[:rh * pitch].view(rh, pitch)[:, :rw] if rh else buf[:0].view(0, pitch)[:, :0]
            if rh and rw:
                blk.copy_(torch.from_numpy(np.ascontiguousarray(src[y:y + rh, x:x + rw]).view(np.int32)).cuda())
            crops.append(buf)
            views.append(buf.data_ptr() - 4 * (y * pitch + x))
    oc = out_frame(h, w)
    import ctypes
    arr = lambda v: (ctypes.c_void_p * n)(*v)  # noqa: E731
    r = roi_tensor(rois)
    rc = eqc._lib.compositor_depth_roi(n, arr(views_c), arr(views_d), r.data_ptr(), w, h, pitch,
                                       oc.data_ptr(), None, w, None)
    assert rc == 0
    np.testing.assert_array_equal(to_host(oc), oracle.depth_composite(c, d)[0])


@pytest.mark.parametrize("n,w,h,pitch,offset", [(16, 640, 360, None, 0), (5, 131, 29, 136, 0), (3, 64, 7, 64, 2)])
def test_blend_roi_within_one_lsb(eqc, n, w, h, pitch, offset):
    layers = synth.volume_bricks(synth.SEED_BASE + 64, n, w, h)
    rng = np.random.default_rng(n)
    order = rng.permutation(n).astype(np.int32)
    dl = [to_dev(x, pitch, offset) for x in layers]
    r = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
    eqc.image_roi(dl, r, 0)
    assert [tuple(v) for v in r.cpu().tolist()] == [oracle.roi(x, 0) for x in layers]
    out = out_frame(h, w, pitch, offset)
    eqc.compositor_blend_ordered_roi(dl, r, out, order=order, background=0x20000000)
    want = oracle.blend_ordered_roi(layers, [oracle.roi(x, 0) for x in layers], order=order,
                                    background=0x20000000)
    got = to_host(out)
    diff = np.abs(got.view(np.uint8).astype(int) - want.view(np.uint8).astype(int))
    assert diff.max() <= 1
    # random rectangles (layers partly masked)
    rois = [(int(rng.integers(-2, w)), int(rng.integers(-2, h)), int(rng.integers(0, w + 3)),
             int(rng.integers(0, h + 3))) for _ in range(n)]
    eqc.compositor_blend_ordered_roi(dl, roi_tensor(rois), out, order=order)
    want = oracle.blend_ordered_roi(layers, rois, order=order)
    diff = np.abs(to_host(out).view(np.uint8).astype(int) - want.view(np.uint8).astype(int))
    assert diff.max() <= 1


def test_roi_host_validation(eqc):
    c = [torch.zeros((4, 4), dtype=torch.int32, device="cuda")]
    r = torch.zeros((1, 4), dtype=torch.int32, device="cuda")
    out = torch.zeros((4, 4), dtype=torch.int32, device="cuda")
    with pytest.raises(eqc.EqcError):
        eqc.image_roi(c, r[:, 1:], 0)  # misaligned ROI array
    with pytest.raises(eqc.EqcError):
        eqc.compositor_blend_ordered_roi(c * 2, torch.zeros((2, 4), dtype=torch.int32, device="cuda"), out,
                                         order=[0, 0])  # not a permutation


@pytest.mark.parametrize("nr,nl,w,h,loose,dest", [(2, 2, 640, 360, 0, 0), (3, 1, 300, 41, 5, 2), (4, 2, 257, 77, 0, 1)])
def test_direct_send_with_application_rois_virtual_ranks(eqc, nr, nl, w, h, loose, dest):
    # application-provided ROIs: exact or loose boxes around each
    # source's rendered pixels; the result equals the full composite
    N = nr * nl
    c, d = synth.depth_sources(synth.SEED_BASE + 68 + N, N, w, h, mode="compact")
    rois = []
    for x in d:
        rx, ry, rw, rh = oracle.roi(x, BG)
        rois.append((rx - loose, ry - loose, rw + 2 * loose, rh + 2 * loose) if rw else (0, 0, 0, 0))
    out = out_frame(h, w)
    for flags in (0, eqc.FLAG_RLE):
        eqc.compose_direct_send_roi_local(nr, [to_dev(x) for x in c], [to_dev(x) for x in d], roi_tensor(rois), out,
                                          dest_rank=dest, flags=flags)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(to_host(out), oracle.depth_composite(c, d)[0])
