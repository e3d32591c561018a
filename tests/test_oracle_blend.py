"""Pins for oracle O2 (ordered back-to-front 'over'; R-C3, R-C4).

Independent of the oracle's recursive double-precision chain:
* worked example B and the closed form of N identical layers (geometric series);
* the EXPANDED exact-rational form out = bg*prod_j(1-a_j) + sum_k s_k prod_{j>k}(1-a_j)
  evaluated with fractions.Fraction (a different formula, exact);
* special cases a = 255 (front layer wins) and the all-zero layer.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import synth
from helpers import read_golden_lines


def pack(r, g, b, a):
    return (r & 255) | ((g & 255) << 8) | ((b & 255) << 16) | ((a & 255) << 24)


def unpack(v):
    return [(int(v) >> (8 * c)) & 255 for c in range(4)]


def exact_expanded(layers, bg):
    """Exact value of each channel, in units of 1/255 of full scale * 255."""
    out = []
    for c in range(4):
        # sum_k s_k * prod_{j>k} (1 - a_j/255)  +  bg * prod_j (1 - a_j/255)
        total = Fraction(0)
        for k in range(len(layers)):
            prod = Fraction(1)
            for j in range(k + 1, len(layers)):
                prod *= Fraction(255 - layers[j][3], 255)
            total += Fraction(layers[k][c]) * prod
        trans = Fraction(1)
        for j in range(len(layers)):
            trans *= Fraction(255 - layers[j][3], 255)
        total += Fraction(bg[c]) * trans
        out.append(total)
    return out


def round_half_up(fr: Fraction) -> int:
    return max(0, min(255, math.floor(fr + Fraction(1, 2))))


def test_worked_example_b(oracle_lib):
    recs = {}
    for line in read_golden_lines("blend_example_b.txt"):
        if line.startswith("const16"):
            lhs, rhs = line.split(":", 1)[1].split("->")
            recs["const16"] = ([int(t) for t in lhs.split()], [int(t) for t in rhs.split()])
            continue
        k, v = line.split(":")
        recs[k.strip()] = [int(t) for t in v.split()]
    l0 = np.array([[pack(*recs["layer0"])]], np.uint32)
    l1 = np.array([[pack(*recs["layer1"])]], np.uint32)
    out = oracle_lib.blend_ordered([l0, l1], background=pack(*recs["background"]))
    assert unpack(out[0, 0]) == recs["out"]
    lay, want = recs["const16"]
    layers = [np.array([[pack(*lay)]], np.uint32) for _ in range(16)]
    out = oracle_lib.blend_ordered(layers)
    assert unpack(out[0, 0]) == want


@pytest.mark.parametrize("c,a,n", [(51, 51, 16), (10, 20, 5), (200, 255, 3), (0, 0, 4), (7, 9, 64), (128, 128, 2)])
def test_closed_form_identical_layers(oracle_lib, c, a, n):
    """x = c * (1 - (1 - a/255)^n) / (a/255) for a > 0 (geometric series); n*c for a = 0."""
    layers = [np.array([[pack(c, c, c, a)]], np.uint32) for _ in range(n)]
    out = oracle_lib.blend_ordered(layers)
    if a == 0:
        xc = Fraction(c * n)
        xa = Fraction(0)
    else:
        q = Fraction(255 - a, 255)
        xc = Fraction(c) * (1 - q ** n) / Fraction(a, 255)
        xa = Fraction(a) * (1 - q ** n) / Fraction(a, 255)
    got = unpack(out[0, 0])
    assert got[:3] == [round_half_up(xc)] * 3
    assert got[3] == round_half_up(xa)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_random_against_expanded_exact(oracle_lib, n):
    layers = synth.premultiplied_noise(500 + n, n, 9, 7)
    bg = pack(3, 0, 200, 255)
    out = oracle_lib.blend_ordered(layers, background=bg)
    bgl = unpack(bg)
    for y in range(7):
        for x in range(9):
            lay = [unpack(L[y, x]) for L in layers]
            ex = exact_expanded(lay, bgl)
            got = unpack(out[y, x])
            for c in range(4):
                want = round_half_up(ex[c])
                frac = ex[c] - math.floor(ex[c])
                if abs(frac - Fraction(1, 2)) < Fraction(1, 10 ** 9):
                    assert abs(got[c] - want) <= 1  # double cannot resolve (R-C4)
                else:
                    assert got[c] == want, (y, x, c, lay, float(ex[c]))


def test_order_permutation_argument(oracle_lib):
    layers = synth.premultiplied_noise(77, 4, 6, 5)
    order = [2, 0, 3, 1]
    a = oracle_lib.blend_ordered(layers, order=order)
    b = oracle_lib.blend_ordered([layers[i] for i in order])
    np.testing.assert_array_equal(a, b)


def test_opaque_front_layer_wins(oracle_lib):
    layers = synth.premultiplied_noise(78, 3, 8, 8)
    front = layers[-1].copy()
    front |= np.uint32(0xFF000000)  # a = 255 (premultiplied: any RGB <= 255 is valid)
    out = oracle_lib.blend_ordered(layers[:-1] + [front], background=pack(9, 9, 9, 9))
    np.testing.assert_array_equal(out, front)


def test_zero_layer_is_identity(oracle_lib):
    layers = synth.premultiplied_noise(79, 3, 8, 8)
    z = np.zeros_like(layers[0])
    a = oracle_lib.blend_ordered(layers)
    b = oracle_lib.blend_ordered([z] + layers[:2] + [z] + layers[2:] + [z])
    np.testing.assert_array_equal(a, b)
    one = oracle_lib.blend_ordered([layers[0]])
    np.testing.assert_array_equal(one, layers[0])  # N = 1, bg = 0
