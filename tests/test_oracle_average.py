"""Oracle pins for subpixel accumulation + averaging (SURVEY 8(f) f4,
P:1855-1858, reading R-C22: per-channel mean rounded half up)."""
import numpy as np

import oracle
import synth


def np_mean_half_up(frames):
    a = np.stack([f.view(np.uint8).reshape(f.shape + (4,)).astype(np.int64) for f in frames])
    n = len(frames)
    s = a.sum(axis=0)
    m = (2 * s + n) // (2 * n)  # floor(mean + 1/2)
    return m.astype(np.uint8).reshape(frames[0].shape + (4,)).view(np.uint32).reshape(frames[0].shape)


def test_average_matches_numpy_half_up():
    for n, w, h in [(1, 5, 3), (2, 17, 9), (3, 33, 7), (8, 64, 16), (64, 9, 5)]:
        c, _ = synth.random_frames(300 + n, n, w, h)
        np.testing.assert_array_equal(oracle.average(c), np_mean_half_up(c))


def test_average_special_cases():
    c, _ = synth.random_frames(5, 1, 20, 4)
    np.testing.assert_array_equal(oracle.average(c), c[0])  # n = 1: identity
    f = np.full((3, 4), 0x80402010, np.uint32)
    np.testing.assert_array_equal(oracle.average([f] * 7), f)  # equal sources
    # exact .5 means round up: (1 + 2) / 2 = 1.5 -> 2 ; (0 + 255) / 2 = 127.5 -> 128
    a = np.full((1, 1), 0x00FF0001, np.uint32)
    b = np.full((1, 1), 0x00000002, np.uint32)
    assert int(oracle.average([a, b])[0, 0]) == 0x00800002
    # permutation invariance
    c, _ = synth.random_frames(9, 5, 13, 6)
    np.testing.assert_array_equal(oracle.average(c), oracle.average(c[::-1]))
