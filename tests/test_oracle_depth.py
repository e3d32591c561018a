"""Pins for oracle O1 (depth-sorted compositing; ties R-C2).

Each check is independent of the oracle's own formulation (argmin of the
(depth, index) pair): hand-worked example D, the sequential keep-destination
fold of S:299 (a different algorithm), numpy's min/argmin library routines,
exhaustive tiny cases, and invariants (identity, permutation with travelling
labels -- the out-of-order assembly of P:2492-2498 -- and monotone transforms).
"""
import itertools

import numpy as np
import pytest

import synth
from helpers import read_golden_lines

MAX = 0xFFFFFFFF


def _parse_example_d():
    rec = {}
    for line in read_golden_lines("depth_example_d.txt"):
        k, v = line.split(":")
        base = 10 if "depth" in k else 16
        rec[k.strip()] = np.array([int(t, base) for t in v.split()], np.uint64).astype(np.uint32).reshape(2, 2)
    return rec


def test_worked_example_d(oracle_lib):
    r = _parse_example_d()
    oc, od = oracle_lib.depth_composite([r["color0"], r["color1"]], [r["depth0"], r["depth1"]])
    np.testing.assert_array_equal(oc, r["out_color"])
    np.testing.assert_array_equal(od, r["out_depth"])


def test_single_source_is_identity(oracle_lib):
    c, d = synth.random_frames(1, 1, 37, 11)
    oc, od = oracle_lib.depth_composite(c, d)
    np.testing.assert_array_equal(oc, c[0])
    np.testing.assert_array_equal(od, d[0])


def _keep_dst_fold(colors, depths):
    """S:299 z_composite(dst, src): copy src iff src.depth < dst.depth (keep dst
    on ties), folded over sources in index order -- a different algorithm."""
    oc = colors[0].copy()
    od = depths[0].copy()
    for c, d in zip(colors[1:], depths[1:]):
        take = d < od
        oc[take] = c[take]
        od[take] = d[take]
    return oc, od


@pytest.mark.parametrize("n", [1, 2, 3])
def test_exhaustive_single_pixel_small_alphabet(oracle_lib, n):
    alphabet = [0, 1, 2, MAX]
    combos = list(itertools.product(alphabet, repeat=n))
    w = len(combos)
    depths = [np.array([[c[i] for c in combos]], np.uint64).astype(np.uint32) for i in range(n)]
    colors = [np.full((1, w), 0x01010101 * (i + 1), np.uint32) for i in range(n)]
    oc, od = oracle_lib.depth_composite(colors, depths)
    for x, combo in enumerate(combos):
        m = min(combo)
        first = combo.index(m)  # lowest index among the minima
        assert od[0, x] == m
        assert oc[0, x] == 0x01010101 * (first + 1)


@pytest.mark.parametrize("n,alphabet", [(2, None), (5, [0, 7, MAX]), (8, [3, MAX]), (16, None)])
def test_matches_fold_and_numpy_min(oracle_lib, n, alphabet):
    c, d = synth.random_frames(100 + n, n, 23, 9, depth_alphabet=alphabet)
    oc, od = oracle_lib.depth_composite(c, d)
    fc, fd = _keep_dst_fold(c, d)
    np.testing.assert_array_equal(oc, fc)
    np.testing.assert_array_equal(od, fd)
    D = np.stack(d)
    np.testing.assert_array_equal(od, D.min(axis=0))
    k = D.argmin(axis=0)  # numpy: first occurrence of the minimum
    np.testing.assert_array_equal(oc, np.take_along_axis(np.stack(c), k[None], 0)[0])


def test_permutation_with_travelling_labels(oracle_lib):
    """Out-of-order assembly: any processing order gives the same
    image when the (depth, index) label travels with the data.  We emulate the
    label by making depths unique per index (depth*n + index), permute the
    sources, and compare."""
    n = 6
    c, d = synth.random_frames(7, n, 17, 13, depth_alphabet=[0, 5, 9, MAX >> 4])
    lab = [(x.astype(np.uint64) * n + i).astype(np.uint32) for i, x in enumerate(d)]
    oc0, od0 = oracle_lib.depth_composite(c, lab)
    rng = np.random.default_rng(1)
    for _ in range(5):
        perm = rng.permutation(n)
        oc, od = oracle_lib.depth_composite([c[i] for i in perm], [lab[i] for i in perm])
        np.testing.assert_array_equal(oc, oc0)
        np.testing.assert_array_equal(od, od0)


def test_strictly_increasing_depth_transform(oracle_lib):
    n = 5
    c, d = synth.random_frames(8, n, 19, 7, depth_alphabet=[0, 1, 2, 3, 100, 1000])
    oc, _ = oracle_lib.depth_composite(c, d)
    d2 = [(x.astype(np.uint64) * 3 + 11).astype(np.uint32) for x in d]
    oc2, _ = oracle_lib.depth_composite(c, d2)
    np.testing.assert_array_equal(oc, oc2)


def test_pitch_and_colour_only(oracle_lib):
    c, d = synth.depth_sources(20190214, 3, 50, 20, pitch=64)
    assert c[0].strides[0] == 64 * 4
    oc, od = oracle_lib.depth_composite(c, d)
    oc2, od2 = oracle_lib.depth_composite([np.ascontiguousarray(x) for x in c],
                                          [np.ascontiguousarray(x) for x in d])
    np.testing.assert_array_equal(oc, oc2)
    oc3, od3 = oracle_lib.depth_composite(c, d, want_depth=False)
    assert od3 is None
    np.testing.assert_array_equal(oc3, oc)


def test_all_background_resolves_to_source0(oracle_lib):
    n = 4
    c = [np.full((3, 5), 0x10 + i, np.uint32) for i in range(n)]
    d = [np.full((3, 5), MAX, np.uint32) for _ in range(n)]
    oc, od = oracle_lib.depth_composite(c, d)
    assert (oc == 0x10).all() and (od == MAX).all()
