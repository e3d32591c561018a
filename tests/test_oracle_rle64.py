"""Oracle pins for the RLE-64 codec (reading
R-C17): hand-derived records, round trips, canonical form (maximal runs of
units), the size bound and corrupt-stream rejection."""
import numpy as np
import pytest

import oracle
import synth
from helpers import read_golden_lines


def test_rle64_golden_records():
    n = 0
    for line in read_golden_lines("rle64_records.txt"):
        px, rec = line.split("|")
        pixels = [int(v, 16) for v in px.strip().split(",")]
        want = bytes.fromhex(rec.replace(" ", ""))
        assert oracle.rle64_encode_chunk(pixels) == want, line
        n += 1
    assert n >= 7


def _parse(rec: bytes, L: int):
    ntok = rec[0]
    ctrl = rec[1:1 + ntok]
    p = 1 + ntok
    toks = []
    for c in ctrl:
        ln = (c & 0x7F) + 1
        if c & 0x80:
            toks.append(("R", ln, [rec[p:p + 8]]))
            p += 8
        else:
            toks.append(("L", ln, [rec[p + 8 * q:p + 8 * q + 8] for q in range(ln)]))
            p += 8 * ln
    assert p == len(rec)
    return toks


def _canonical(toks):
    # REPEAT >= 2; no two adjacent LITERALs; a LITERAL holds no two equal
    # neighbours; adjacent REPEATs differ; a LITERAL's edge unit differs from
    # the neighbouring REPEAT's unit (else the run was not maximal)
    for i, (k, ln, units) in enumerate(toks):
        if k == "R":
            assert ln >= 2
        else:
            assert all(units[q] != units[q + 1] for q in range(ln - 1))
        if i:
            pk, _, pu = toks[i - 1]
            assert not (pk == "L" and k == "L")
            assert pu[-1] != units[0]


def test_rle64_round_trip_and_canonical():
    rng = np.random.default_rng(64)
    for trial in range(3000):
        L = int(rng.integers(1, 129))
        alpha = rng.integers(0, 1 << 32, size=int(rng.integers(1, 4)), dtype=np.uint64).astype(np.uint32)
        px = alpha[rng.integers(0, len(alpha), size=L)]
        if trial % 3 == 0:  # long runs of pixel pairs
            px = np.repeat(px[: (L + 1) // 2], 2)[:L] if trial % 2 else np.tile(px[:2], L)[:L]
        rec = oracle.rle64_encode_chunk(px)
        U = (L + 1) // 2
        assert len(rec) <= 2 + 8 * U  # size bound (literal-only worst case)
        toks = _parse(rec, L)
        assert sum(t[1] for t in toks) == U
        _canonical(toks)


@pytest.mark.parametrize("w,h", [(1, 1), (3, 2), (128, 4), (129, 3), (300, 7)])
def test_rle64_stream_round_trip(w, h):
    c, d = synth.depth_sources(synth.SEED_BASE + 65, 1, w, h)
    for img, kind in ((c[0], 0), (d[0], 1)):
        s = oracle.rle64_encode(img, kind)
        assert len(s) <= oracle.rle_max_size(w, h)
        rc, out = oracle.rle64_decode(s, w, h)
        assert rc == 0
        np.testing.assert_array_equal(out, img)
        # the v1 per-component decoder rejects an RLE-64 stream
        assert oracle.rle_decode(s, w, h)[0] == oracle.E_CORRUPT


def test_rle64_compresses_only_equal_pixel_pairs():
    # "it can only compress adjacent pixels of the same colour"
    flat = np.full((4, 256), 0x11223344, np.uint32)
    grad = (np.arange(256, dtype=np.uint32)[None, :] * 0x01010101 + np.zeros((4, 1), np.uint32)).astype(np.uint32)
    assert len(oracle.rle64_encode(flat)) < 32 + 8 * 8 + 8 * 10 + 1
    raw = 4 * grad.size
    assert len(oracle.rle64_encode(grad)) > raw  # no equal pairs: no gain


def test_rle64_corrupt_streams_rejected():
    img = synth.random_frames(3, 1, 130, 5, depth_alphabet=[1, 2])[1][0]
    s = bytearray(oracle.rle64_encode(img, 1))
    for pos, val in [(6, 0), (6, 3), (16, 99), (32 + 4, 255), (len(s) - 1, None)]:
        t = bytearray(s)
        if val is None:
            t = t[:-1]
        else:
            t[pos] = val
        assert oracle.rle64_decode(bytes(t), 130, 5)[0] != 0


def golden_rle64_streams():
    """Hand-derived whole RLE-64 streams (tests/golden/rle64_streams.txt):
    yields (name, kind, image [H, W] uint32, stream bytes)."""
    for line in read_golden_lines("rle64_streams.txt"):
        name, kind, w, h, px, hexs = (f.strip() for f in line.split("|"))
        w, h = int(w), int(h)
        if "*" in px:
            v, cnt = px.split("*")
            vals = [int(v, 16)] * int(cnt)
        else:
            vals = [int(v, 16) for v in px.split(",")]
        img = np.array(vals, dtype=np.uint32).reshape(h, w)
        yield name, int(kind), img, bytes.fromhex(hexs.replace(" ", ""))


def test_rle64_golden_streams():
    """Pins the RLE-64 stream framing (header flags = 2, table word 2 = record
    size, records in chunk order) against hand-derived bytes, both ways."""
    seen = 0
    for name, kind, img, want in golden_rle64_streams():
        h, w = img.shape
        assert oracle.rle64_encode(img, kind) == want, name
        rc, out = oracle.rle64_decode(want, w, h)
        assert rc == 0, name
        np.testing.assert_array_equal(out, img)
        seen += 1
    assert seen == 2
