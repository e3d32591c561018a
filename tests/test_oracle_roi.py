"""Oracle pins for the region of interest (SURVEY 8(f) row f1, P:2259-2271,
P:2296-2299): or_roi against numpy's nonzero bounding box, and the ROI
composites reduced to O1 / O2 on frames masked outside their rectangles."""
import numpy as np
import pytest

import oracle
import synth

BG = 0xFFFFFFFF


def np_bbox(frame, bg):
    ys, xs = np.nonzero(frame != np.uint32(bg))
    if ys.size == 0:
        return (0, 0, 0, 0)
    return (int(xs.min()), int(ys.min()), int(xs.max() - xs.min() + 1), int(ys.max() - ys.min() + 1))


@pytest.mark.parametrize("density", [0.0, 1e-4, 0.01, 0.3, 1.0])
def test_roi_matches_numpy_bbox(density):
    rng = np.random.default_rng(int(density * 1e4) + 7)
    for h, w in [(1, 1), (3, 17), (64, 64), (37, 131)]:
        f = np.full((h, w), BG, np.uint32)
        m = rng.random((h, w)) < density
        f[m] = rng.integers(0, BG, size=int(m.sum()), dtype=np.uint64).astype(np.uint32)
        assert oracle.roi(f, BG) == np_bbox(f, BG)


def test_roi_special_cases():
    f = np.zeros((20, 30), np.uint32)
    assert oracle.roi(f, 0) == (0, 0, 0, 0)  # empty frame
    f[7, 11] = 3
    assert oracle.roi(f, 0) == (11, 7, 1, 1)  # one pixel
    f[0, 0] = f[19, 29] = 1
    assert oracle.roi(f, 0) == (0, 0, 30, 20)  # corners: the whole frame
    # a pitched view: the padding never counts
    buf = np.full((20, 40), 9, np.uint32)
    buf[:, :30] = 0
    buf[5, 3] = 1
    assert oracle.roi(buf[:, :30], 0) == (3, 5, 1, 1)


def _masked(frames, rois, bg):
    out = []
    for f, (x, y, w, h) in zip(frames, rois):
        g = np.full_like(f, bg)
        g[y:y + h, x:x + w] = f[y:y + h, x:x + w]
        out.append(g)
    return out


def _random_rois(rng, n, w, h):
    r = []
    for _ in range(n):
        x0, x1 = sorted(rng.integers(0, w + 1, size=2))
        y0, y1 = sorted(rng.integers(0, h + 1, size=2))
        r.append((int(x0), int(y0), int(x1 - x0), int(y1 - y0)))
    return r


def test_depth_roi_reduces_to_o1_on_masked_frames():
    rng = np.random.default_rng(11)
    for n, w, h in [(1, 9, 5), (3, 40, 23), (6, 67, 31)]:
        c, d = synth.random_frames(100 + n, n, w, h, depth_alphabet=[0, 5, 5, 9, BG])
        rois = _random_rois(rng, n, w, h)
        rois[0] = (0, 0, 0, 0) if n > 1 else rois[0]  # an empty ROI contributes nothing
        got_c, got_d = oracle.depth_composite_roi(c, d, rois)
        want_c, want_d = oracle.depth_composite(_masked(c, rois, 0), _masked(d, rois, BG))
        np.testing.assert_array_equal(got_c, want_c)
        np.testing.assert_array_equal(got_d, want_d)


def test_depth_roi_full_rect_and_exact_crop_are_o1():
    c, d = synth.depth_sources(synth.SEED_BASE + 50, 4, 96, 64)
    want_c, want_d = oracle.depth_composite(c, d)
    full = [(0, 0, 96, 64)] * 4
    got = oracle.depth_composite_roi(c, d, full)
    np.testing.assert_array_equal(got[0], want_c)
    np.testing.assert_array_equal(got[1], want_d)
    # the ROI premise: cropping each source to the bounding box
    # of its rendered pixels changes nothing
    exact = [oracle.roi(x, BG) for x in d]
    got = oracle.depth_composite_roi(c, d, exact)
    np.testing.assert_array_equal(got[0], want_c)
    np.testing.assert_array_equal(got[1], want_d)


def test_blend_roi_reduces_to_o2_on_masked_layers():
    rng = np.random.default_rng(12)
    for n, w, h in [(1, 8, 3), (4, 33, 17), (7, 50, 20)]:
        layers = synth.premultiplied_noise(200 + n, n, w, h)
        rois = _random_rois(rng, n, w, h)
        order = rng.permutation(n).astype(np.int32)
        got = oracle.blend_ordered_roi(layers, rois, order=order, background=0x10203040)
        want = oracle.blend_ordered(_masked(layers, rois, 0), order=order, background=0x10203040)
        np.testing.assert_array_equal(got, want)
    bricks = synth.volume_bricks(synth.SEED_BASE + 51, 8, 80, 48)
    exact = [oracle.roi(b, 0) for b in bricks]
    np.testing.assert_array_equal(oracle.blend_ordered_roi(bricks, exact), oracle.blend_ordered(bricks))


def test_roi_rects_are_clipped_to_the_frame():
    # R-C19: the part of a rectangle outside the frame holds no pixels
    c, d = synth.random_frames(1, 2, 8, 8, depth_alphabet=[1, 2, BG])
    for bad, clipped in [((-1, 0, 3, 2), (0, 0, 2, 2)), ((0, 0, 9, 1), (0, 0, 8, 1)),
                         ((7, 7, 2, 1), (7, 7, 1, 1)), ((0, 0, -1, 3), (0, 0, 0, 0)),
                         ((9, 2, 4, 4), (0, 0, 0, 0))]:
        a = oracle.depth_composite_roi(c, d, [bad, (0, 0, 8, 8)])
        b = oracle.depth_composite_roi(c, d, [clipped, (0, 0, 8, 8)])
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
        np.testing.assert_array_equal(oracle.blend_ordered_roi(c, [(0, 0, 8, 8), bad]),
                                      oracle.blend_ordered_roi(c, [(0, 0, 8, 8), clipped]))
