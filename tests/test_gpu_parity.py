"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (north_star): bit-exact for depth compositing and RLE bytes / decode;
ordered blend within 1/255 (1 LSB of RGBA8) of the exact-chain oracle.
Shapes span several 128-pixel chunks / 4-pixel vectors and ragged tails,
odd widths, pitch > width, misaligned pointers (scalar path), N in
{1, 2, 3, 8, 16, 64}, all-background, heavy depth ties and uniform noise.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import bytes_of, out_frame, stream_dev, to_dev, to_host  # noqa: E402

SEED = synth.SEED_BASE


@pytest.fixture(scope="module")
def eqc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1902_08755_b200 import eqc as m
    return m


# ---------------------------------------------------------------- depth ----
DEPTH_CASES = [
    # (name, n, w, h, pitch, offset, generator)
    ("c1_2x64x64", 2, 64, 64, None, 0, "scene"),
    ("c2_8x1920x1080", 8, 1920, 1080, None, 0, "scene"),
    ("one_px", 1, 1, 1, None, 0, "noise"),
    ("odd_3x5", 2, 3, 5, None, 0, "noise"),
    ("ragged_67x13", 3, 67, 13, None, 0, "ties"),
    ("pitch_129x7_p136", 8, 129, 7, 136, 0, "scene"),
    ("n16_1000x3", 16, 1000, 3, None, 0, "noise"),
    ("n64_37x9_p40", 64, 37, 9, 40, 0, "ties"),
    ("misaligned", 5, 64, 6, 64, 1, "ties"),
    ("allbg", 4, 100, 4, None, 0, "background"),
]


def _frames(kind, n, w, h, seed):
    if kind == "scene":
        return synth.depth_sources(seed, n, w, h)
    if kind == "noise":
        return synth.random_frames(seed, n, w, h)
    if kind == "ties":
        return synth.random_frames(seed, n, w, h, depth_alphabet=[0, 1, 5, 0xFFFFFFFF])
    c = [np.full((h, w), 0x01010101 * (i + 1), np.uint32) for i in range(n)]
    d = [np.full((h, w), 0xFFFFFFFF, np.uint32) for _ in range(n)]
    return c, d


@pytest.mark.parametrize("case", DEPTH_CASES, ids=[c[0] for c in DEPTH_CASES])
def test_depth_composite_bit_exact(eqc, case):
    name, n, w, h, pitch, offset, kind = case
    c, d = _frames(kind, n, w, h, SEED + 1 + n + w)
    oc, od = oracle.depth_composite(c, d)
    dc = [to_dev(x, pitch, offset) for x in c]
    dd = [to_dev(x, pitch, offset) for x in d]
    out_c = out_frame(h, w, pitch, offset)
    out_d = out_frame(h, w, pitch, offset)
    eqc.compositor_depth(dc, dd, out_c, out_d)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out_c), oc)
    np.testing.assert_array_equal(to_host(out_d), od)
    # colour-only output
    out_c2 = out_frame(h, w, pitch, offset)
    eqc.compositor_depth(dc, dd, out_c2, None)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out_c2), oc)


def test_depth_composite_target_4k_sampled_rows(eqc):
    """Full 8 x 3840x2160 in bench.py's launch configuration; oracle on sampled rows."""
    n, w, h = 8, 3840, 2160
    c, d = synth.depth_sources(SEED + 2, n, w, h)
    dc = [to_dev(x) for x in c]
    dd = [to_dev(x) for x in d]
    out_c, out_d = out_frame(h, w), out_frame(h, w)
    eqc.compositor_depth(dc, dd, out_c, out_d)
    torch.cuda.synchronize()
    gc, gd = to_host(out_c), to_host(out_d)
    rows = np.random.default_rng(0).choice(h, 24, replace=False)
    for y in rows:
        oc, od = oracle.depth_composite([x[y:y + 1] for x in c], [x[y:y + 1] for x in d])
        np.testing.assert_array_equal(gc[y:y + 1], oc)
        np.testing.assert_array_equal(gd[y:y + 1], od)
    # properties at every pixel: output depth is the minimum over sources
    np.testing.assert_array_equal(gd, np.minimum.reduce(d))


# ---------------------------------------------------------------- blend ----
BLEND_CASES = [
    ("c3_small_16x512x288", 16, 512, 288, None, 0, "bricks"),
    ("n1", 1, 33, 7, None, 0, "noise"),
    ("n2_odd", 2, 5, 3, None, 0, "noise"),
    ("n3_pitch", 3, 130, 9, 136, 0, "noise"),
    ("n64", 64, 70, 5, None, 0, "noise"),
    ("misaligned", 7, 64, 4, 64, 3, "noise"),
]


def _assert_within_one_lsb(got, want):
    g = got.view(np.uint8).astype(np.int32)
    o = want.view(np.uint8).astype(np.int32)
    diff = np.abs(g - o)
    assert diff.max() <= 1, (diff.max(), np.argwhere(diff > 1)[:5])


@pytest.mark.parametrize("case", BLEND_CASES, ids=[c[0] for c in BLEND_CASES])
def test_blend_within_one_lsb(eqc, case):
    name, n, w, h, pitch, offset, kind = case
    if kind == "bricks":
        layers = synth.volume_bricks(SEED + 3, n, w, h)
    else:
        layers = synth.premultiplied_noise(SEED + n + w, n, w, h)
    rng = np.random.default_rng(n)
    order = rng.permutation(n)
    bg = 0x20101008 if n % 2 else 0
    want = oracle.blend_ordered(layers, order=order, background=bg)
    dl = [to_dev(x, pitch, offset) for x in layers]
    out = out_frame(h, w, pitch, offset)
    eqc.compositor_blend_ordered(dl, out, order=list(order), background=bg)
    torch.cuda.synchronize()
    _assert_within_one_lsb(to_host(out), want)


def test_blend_c3_4k_sampled_rows(eqc):
    n, w, h = 16, 3840, 2160
    layers = synth.volume_bricks(SEED + 2, n, w, h)
    dl = [to_dev(x) for x in layers]
    out = out_frame(h, w)
    eqc.compositor_blend_ordered(dl, out)
    torch.cuda.synchronize()
    got = to_host(out)
    for y in np.random.default_rng(1).choice(h, 16, replace=False):
        want = oracle.blend_ordered([x[y:y + 1] for x in layers])
        _assert_within_one_lsb(got[y:y + 1], want)


def test_blend_opaque_and_transparent_special_cases(eqc):
    layers = synth.premultiplied_noise(9, 3, 64, 4)
    front = layers[2] | np.uint32(0xFF000000)
    out = out_frame(4, 64)
    eqc.compositor_blend_ordered([to_dev(layers[0]), to_dev(layers[1]), to_dev(front)], out, background=0x12345678)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out), front)
    z = np.zeros((4, 64), np.uint32)
    eqc.compositor_blend_ordered([to_dev(z), to_dev(layers[0]), to_dev(z)], out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out), layers[0])


# ------------------------------------------------------------------ RLE ----
RLE_CASES = [
    # (name, w, h, pitch, kind, flags, generator)
    ("c1_colour_swz", 64, 64, None, 0, 1, "scene"),
    ("c1_depth", 64, 64, None, 1, 0, "scene"),
    ("c2_colour_swz", 1920, 1080, None, 0, 1, "scene"),
    ("c2_depth", 1920, 1080, None, 1, 0, "scene"),
    ("c2_colour_plain", 1920, 1080, None, 0, 0, "scene"),
    ("noise_colour", 300, 7, None, 0, 1, "noise"),
    ("noise_depth", 257, 5, 264, 1, 0, "noise"),
    ("narrow_w1", 1, 9, None, 0, 1, "noise"),
    ("narrow_w2", 2, 3, None, 1, 0, "noise"),
    ("w130_ragged", 130, 11, 131, 0, 1, "scene"),
    ("constant", 512, 4, None, 0, 1, "const"),
    ("smallalpha", 200, 6, None, 1, 0, "ties"),
    ("runs", 384, 8, None, 0, 0, "runs"),
]


def _rle_image(kind_gen, w, h, seed, depth):
    if kind_gen == "scene":
        c, d = synth.depth_sources(seed, 1, w, h)
        return d[0] if depth else c[0]
    if kind_gen == "noise":
        c, d = synth.random_frames(seed, 1, w, h)
        return d[0] if depth else c[0]
    if kind_gen == "ties":
        c, d = synth.random_frames(seed, 1, w, h, depth_alphabet=[0, 1, 0xFFFFFFFF])
        return d[0]
    if kind_gen == "const":
        return np.full((h, w), 0x80FF0011, np.uint32)
    # runs of random lengths of a few values, per byte plane
    rng = np.random.default_rng(seed)
    vals = np.array([0x00000000, 0xFF000000, 0xFF102030, 0x01010101], np.uint32)
    flat = np.repeat(vals[rng.integers(0, 4, size=w * h)], rng.integers(1, 6, size=w * h))[: w * h]
    return flat.reshape(h, w)


def _workspace(eqc, count, w, h):
    return torch.zeros(eqc.image_rle_workspace_size_batch(count, w, h), dtype=torch.uint8, device="cuda")


@pytest.mark.parametrize("case", RLE_CASES, ids=[c[0] for c in RLE_CASES])
def test_rle_encode_bytes_exact_and_decode(eqc, case):
    name, w, h, pitch, kind, flags, gen = case
    img = _rle_image(gen, w, h, SEED + w + h, kind == 1)
    want = oracle.rle_encode(img, kind=kind, flags=flags)
    src = to_dev(img, pitch)
    cap = eqc.image_rle_max_size(w, h)
    dst = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    d_size = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = _workspace(eqc, 1, w, h)
    for rep in range(3):  # the workspace is reusable without a reset
        dst.fill_(0xAB)
        eqc.image_compress_rle(src, kind, flags, dst, d_size, ws)
        torch.cuda.synchronize()
        n = int(d_size.item())
        assert n == len(want), (rep, n, len(want))
        assert bytes_of(dst, n) == want, rep
    # decode the GPU stream on the GPU
    out = out_frame(h, w, pitch)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.image_decompress_rle(dst, out, status, src_bytes=n)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    np.testing.assert_array_equal(to_host(out), img)


@pytest.mark.parametrize("log2c", [5, 6, 7])
def test_rle_decode_oracle_streams_any_chunk_size(eqc, log2c):
    w, h = 333, 6
    c, d = synth.depth_sources(SEED + log2c, 1, w, h)
    for img, kind, flags in [(c[0], 0, 1), (d[0], 1, 0), (c[0], 0, 0)]:
        s = oracle.rle_encode(img, kind=kind, flags=flags, log2c=log2c)
        out = out_frame(h, w)
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        eqc.image_decompress_rle(stream_dev(s), out, status)
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        np.testing.assert_array_equal(to_host(out), img)


def test_rle_decode_flags_corruption(eqc):
    w, h = 200, 4
    c, _ = synth.depth_sources(SEED + 9, 1, w, h)
    s = bytearray(oracle.rle_encode(c[0], kind=0, flags=1))
    for pos, val in [(0, 0x00), (8, 0x07), (36, 0x77), (40, 0x05), (24, 0x01)]:
        t = bytearray(s)
        t[pos] = (t[pos] + val) & 0xFF if pos != 0 else 0x00
        out = out_frame(h, w)
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        eqc.image_decompress_rle(stream_dev(bytes(t)), out, status)
        torch.cuda.synchronize()
        assert int(status.item()) == -3, pos
    # a plane record claiming zero tokens
    pay0 = 32 + 8 * 2 * h
    t = bytearray(s)
    t[pay0] = 0  # ntok of chunk 0 plane 0
    out = out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.image_decompress_rle(stream_dev(bytes(t)), out, status)
    torch.cuda.synchronize()
    assert int(status.item()) == -3


def test_rle_batch_16_streams(eqc):
    n, w, h = 8, 640, 360
    c, d = synth.depth_sources(SEED + 11, n, w, h)
    imgs = c + d
    kinds = [0] * n + [1] * n
    flags = [1] * n + [0] * n
    srcs = [to_dev(x) for x in imgs]
    cap = eqc.image_rle_max_size(w, h)
    dsts = [torch.zeros(cap, dtype=torch.uint8, device="cuda") for _ in imgs]
    sizes = torch.zeros(len(imgs), dtype=torch.int64, device="cuda")
    ws = _workspace(eqc, len(imgs), w, h)
    for _ in range(2):
        eqc.image_compress_rle_batch(srcs, kinds, flags, dsts, sizes, ws)
    torch.cuda.synchronize()
    for i, img in enumerate(imgs):
        want = oracle.rle_encode(img, kind=kinds[i], flags=flags[i])
        assert int(sizes[i].item()) == len(want)
        assert bytes_of(dsts[i], len(want)) == want
    outs = [out_frame(h, w) for _ in imgs]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.image_decompress_rle_batch(dsts, outs, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    for o, img in zip(outs, imgs):
        np.testing.assert_array_equal(to_host(o), img)


@pytest.mark.parametrize("n,w,h", [(2, 64, 64), (8, 1920, 1080), (3, 300, 5), (16, 130, 3),
                                   (32, 384, 6), (33, 200, 5), (64, 130, 4)])
def test_fused_decode_depth_composite(eqc, n, w, h):
    """n <= 32: descriptors + one prefetch round trip per position (n = 32 at
    384 px overflows the per-warp prefetch buffer: the staging fallback);
    n > 32: every record staged when decoded."""
    c, d = synth.depth_sources(SEED + n + w, n, w, h)
    oc, od = oracle.depth_composite(c, d)
    cs = [stream_dev(oracle.rle_encode(x, kind=0, flags=1)) for x in c]
    ds = [stream_dev(oracle.rle_encode(x, kind=1, flags=0)) for x in d]
    out_c, out_d = out_frame(h, w), out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.compositor_depth_rle(cs, ds, out_c, out_d, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    np.testing.assert_array_equal(to_host(out_c), oc)
    np.testing.assert_array_equal(to_host(out_d), od)


@pytest.mark.parametrize("n,w,h,ties,mode", [(8, 1920, 1080, True, "scattered"), (5, 333, 77, True, "scattered"),
                                              (8, 1024, 512, False, "compact"), (2, 128, 9, True, "compact")])
def test_fused_decode_significance_first(eqc, n, w, h, ties, mode):
    """The fused decode skips a depth record's low byte planes when its most
    significant plane already loses at every pixel; quantised depths (many
    equal high bytes and exact ties) and compact sources exercise both the
    skip and the full decode: still bit-exact against O1."""
    c, d = synth.depth_sources(SEED + 40 + n + w, n, w, h, ties=ties, mode=mode)
    oc, od = oracle.depth_composite(c, d)
    cs = [stream_dev(oracle.rle_encode(x, kind=0, flags=1)) for x in c]
    ds = [stream_dev(oracle.rle_encode(x, kind=1, flags=0)) for x in d]
    out_c, out_d = out_frame(h, w), out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.compositor_depth_rle(cs, ds, out_c, out_d, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    np.testing.assert_array_equal(to_host(out_c), oc)
    np.testing.assert_array_equal(to_host(out_d), od)


def test_target_pipeline_4k_one_image_exact(eqc):
    """One full 3840x2160 colour (swizzled) and depth image, in bench.py's
    launch configuration, byte-exact against the oracle stream."""
    w, h = 3840, 2160
    c, d = synth.depth_sources(SEED + 2, 1, w, h)
    for img, kind, flags in [(c[0], 0, 1), (d[0], 1, 0)]:
        want = oracle.rle_encode(img, kind=kind, flags=flags)
        dst = torch.zeros(eqc.image_rle_max_size(w, h), dtype=torch.uint8, device="cuda")
        sz = torch.zeros(1, dtype=torch.int64, device="cuda")
        eqc.image_compress_rle(to_dev(img), kind, flags, dst, sz, _workspace(eqc, 1, w, h))
        torch.cuda.synchronize()
        assert int(sz.item()) == len(want)
        assert bytes_of(dst, len(want)) == want


def test_display_wall_tile_64_sources_rle_transport(eqc):
    """Config c5 on one wall tile: 64 sources of 2560x1440, 70 % background
    (F = 0.3), every source shipped as RLE streams (two batched encodes of 64)
    and decoded + composited by the fused kernel (64 sources: two passes of
    32 lanes).  Oracle on sampled rows; depth = min over sources everywhere."""
    n, w, h = 64, 2560, 1440
    c, d = synth.depth_sources(SEED + 4, n, w, h, F=0.3)
    dc = [to_dev(x) for x in c]
    dd = [to_dev(x) for x in d]
    cap = eqc.image_rle_max_size(w, h)
    cs = [torch.empty(cap, dtype=torch.uint8, device="cuda") for _ in range(n)]
    ds = [torch.empty(cap, dtype=torch.uint8, device="cuda") for _ in range(n)]
    sizes = torch.zeros(n, dtype=torch.int64, device="cuda")
    ws = _workspace(eqc, n, w, h)
    eqc.image_compress_rle_batch(dc, [0] * n, [1] * n, cs, sizes, ws)
    eqc.image_compress_rle_batch(dd, [1] * n, [0] * n, ds, sizes, ws)
    out_c, out_d = out_frame(h, w), out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.compositor_depth_rle(cs, ds, out_c, out_d, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    gc, gd = to_host(out_c), to_host(out_d)
    np.testing.assert_array_equal(gd, np.minimum.reduce(d))
    for y in np.random.default_rng(5).choice(h, 12, replace=False):
        oc, od = oracle.depth_composite([x[y:y + 1] for x in c], [x[y:y + 1] for x in d])
        np.testing.assert_array_equal(gc[y:y + 1], oc)
        np.testing.assert_array_equal(gd[y:y + 1], od)
    # and the streams decode exactly (spot-check three sources)
    for i in (0, 31, 63):
        o = out_frame(h, w)
        eqc.image_decompress_rle(cs[i], o, status)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(to_host(o), c[i])


def test_bench_step_8x4k_exact(eqc):
    """bench.py's exact step on its exact inputs: image_compress_rle_batch of
    the 16 images of synth.depth_sources(SEED + 10, 8, 3840, 2160) (colour
    swizzled, depth plain) in one launch, then compositor_depth_rle.  Every
    stream byte-for-byte against oracle.rle_encode; every output colour and
    depth pixel against oracle.depth_composite."""
    n, w, h = 8, 3840, 2160
    c, d = synth.depth_sources(SEED + 10, n, w, h)
    imgs = c + d
    kinds = [eqc.KIND_RGBA8] * n + [eqc.KIND_DEPTH32] * n
    flags = [eqc.FLAG_SWIZZLE] * n + [0] * n
    srcs = [to_dev(x) for x in imgs]
    cap = eqc.image_rle_max_size(w, h)
    streams = [torch.empty(cap, dtype=torch.uint8, device="cuda") for _ in imgs]
    sizes = torch.zeros(len(imgs), dtype=torch.int64, device="cuda")
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(len(imgs), w, h), dtype=torch.uint8, device="cuda")
    out_c, out_d = out_frame(h, w), out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(2):  # as in the bench: the workspace is reused without a reset
        eqc.image_compress_rle_batch(srcs, kinds, flags, streams, sizes, ws)
        eqc.compositor_depth_rle(streams[:n], streams[n:], out_c, out_d, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    got_sizes = sizes.tolist()
    for i, img in enumerate(imgs):
        want = oracle.rle_encode(img, kind=kinds[i], flags=flags[i])
        assert got_sizes[i] == len(want), i
        assert bytes_of(streams[i], len(want)) == want, i
    oc, od = oracle.depth_composite(c, d)
    np.testing.assert_array_equal(to_host(out_c), oc)
    np.testing.assert_array_equal(to_host(out_d), od)


def _fused_status(eqc, cs, ds, w, h):
    out_c, out_d = out_frame(h, w), out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.compositor_depth_rle([stream_dev(s) for s in cs], [stream_dev(s) for s in ds], out_c, out_d, status)
    torch.cuda.synchronize()
    return int(status.item())


def test_fused_decode_corruption(eqc):
    """compositor_depth_rle flags a corrupt header field, a broken table offset
    and a malformed record it decodes (one noise source: every chunk of both
    streams is non-constant and decoded)."""
    w, h = 300, 3
    c, d = synth.random_frames(SEED + 77, 1, w, h)
    cs = bytearray(oracle.rle_encode(c[0], kind=0, flags=1))
    ds = bytearray(oracle.rle_encode(d[0], kind=1, flags=0))
    assert _fused_status(eqc, [bytes(cs)], [bytes(ds)], w, h) == 0
    S = (w + 127) // 128
    pay0 = 32 + 8 * S * h
    cases = []
    t = bytearray(ds); t[8] ^= 0x01; cases.append(("depth header W", bytes(cs), bytes(t)))
    t = bytearray(cs); t[12] ^= 0x02; cases.append(("colour header H", bytes(t), bytes(ds)))
    t = bytearray(cs); t[32 + 8 * 2] ^= 0x04; cases.append(("colour table offset", bytes(t), bytes(ds)))
    t = bytearray(ds); t[32 + 8 * 4] ^= 0x01; cases.append(("depth table offset", bytes(cs), bytes(t)))
    t = bytearray(ds); t[pay0] = 0; cases.append(("depth record ntok = 0", bytes(cs), bytes(t)))
    t = bytearray(cs); t[pay0] = 0; cases.append(("colour record ntok = 0", bytes(t), bytes(ds)))
    t = bytearray(ds); t[pay0 + 1] = 0x80 | 3; cases.append(("depth token lengths", bytes(cs), bytes(t)))
    for name, a, b in cases:
        assert _fused_status(eqc, [a], [b], w, h) == eqc.E_CORRUPT, name


@pytest.mark.parametrize("n", [3, 20])  # phase A lane per stream (n <= 16) / lane per source
def test_decoders_survive_random_corruption(eqc, n):
    """Random byte corruption of the payload (ntok bytes, ctrl bytes, values)
    and of plane sizes in the table: the fused decode and the plain decoder
    must never fault (their reads stay inside the staged records + slack) and
    must report EQC_E_CORRUPT whenever the output could be wrong; a stream
    they accept decodes exactly like the oracle's decoder of the same bytes
    when that one accepts it too."""
    rng = np.random.default_rng(SEED + 79 + n)
    w, h = 333, 6
    c, d = synth.depth_sources(SEED + 79, n, w, h)
    cs = [bytearray(oracle.rle_encode(x, kind=0, flags=1)) for x in c]
    ds = [bytearray(oracle.rle_encode(x, kind=1, flags=0)) for x in d]
    S = (w + 127) // 128
    pay0 = 32 + 8 * S * h
    for trial in range(int(os.environ.get("EQC_FUZZ_TRIALS", "60"))):
        tc = [bytearray(x) for x in cs]
        td = [bytearray(x) for x in ds]
        for _ in range(1 + trial % 4):
            tgt = (tc if rng.integers(2) else td)[int(rng.integers(n))]
            if rng.integers(5) == 0:  # a plane size of a table entry
                k = 32 + 8 * int(rng.integers(S * h)) + 4 + int(rng.integers(4))
            else:  # any payload byte
                k = pay0 + int(rng.integers(len(tgt) - pay0))
            tgt[k] = int(rng.integers(256))
        st = _fused_status(eqc, [bytes(x) for x in tc], [bytes(x) for x in td], w, h)
        assert st in (0, eqc.E_CORRUPT), (trial, st)
        for x in tc + td:
            out = out_frame(h, w)
            status = torch.zeros(1, dtype=torch.int32, device="cuda")
            eqc.image_decompress_rle(stream_dev(bytes(x)), out, status)
            torch.cuda.synchronize()
            st = int(status.item())
            assert st in (0, eqc.E_CORRUPT), trial
            rc, want = oracle.rle_decode(bytes(x), w, h)
            # the plain decoder decodes every record: it accepts exactly the
            # streams the oracle accepts, and then decodes them identically
            assert (st == 0) == (rc == 0), (trial, st, rc)
            if st == 0:
                np.testing.assert_array_equal(to_host(out), want)
    torch.cuda.synchronize()  # no sticky CUDA error


def test_encoder_workspace_any_8_byte_alignment(eqc):
    """The encoder workspace need only be 8-byte aligned (eqc.h): a workspace
    starting 8 bytes into an allocation gives the same, exact streams."""
    n, w, h = 4, 900, 40
    c, d = synth.depth_sources(SEED + 78, n, w, h)
    imgs = c[:2] + d[:2]
    kinds, flags = [0, 0, 1, 1], [1, 1, 0, 0]
    srcs = [to_dev(x) for x in imgs]
    cap = eqc.image_rle_max_size(w, h)
    streams = [torch.empty(cap, dtype=torch.uint8, device="cuda") for _ in imgs]
    sizes = torch.zeros(len(imgs), dtype=torch.int64, device="cuda")
    need = eqc.image_rle_workspace_size_batch(len(imgs), w, h)
    for off in (8, 24, 136):
        base = torch.full((need + off,), 0x5A, dtype=torch.uint8, device="cuda")
        eqc.image_compress_rle_batch(srcs, kinds, flags, streams, sizes, base[off:])
        torch.cuda.synchronize()
        for i, img in enumerate(imgs):
            want = oracle.rle_encode(img, kind=kinds[i], flags=flags[i])
            assert int(sizes[i].item()) == len(want), (off, i)
            assert bytes_of(streams[i], len(want)) == want, (off, i)


def test_rle_large_image_offsets_beyond_2_30(eqc):
    """A 16384 x 16384 noise image (1 GiB raw, incompressible: payload offsets
    pass 2^30 and the table holds 2 M chunks) on the v1 path: the stream
    decodes back to the image exactly, its size equals the oracle's size
    formula for all-literal chunks, and sampled row bands re-encoded by the
    oracle give the same table entries (rebased) and records."""
    w = h = 16384
    free = torch.cuda.mem_get_info()[0]
    if free < 8 << 30:
        pytest.skip("needs ~8 GB of free device memory")
    g = torch.Generator(device="cuda")
    g.manual_seed(SEED + 80)
    img = torch.randint(-(1 << 31), (1 << 31) - 1, (h, w), generator=g, device="cuda", dtype=torch.int64)
    img = img.to(torch.int32)
    cap = eqc.image_rle_max_size(w, h)
    dst = torch.empty(cap, dtype=torch.uint8, device="cuda")
    d_size = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(eqc.image_rle_workspace_size(w, h), dtype=torch.uint8, device="cuda")
    eqc.image_compress_rle(img, eqc.KIND_DEPTH32, 0, dst, d_size, ws)
    torch.cuda.synchronize()
    n = int(d_size.item())
    S = (w + 127) // 128
    nch = S * h
    assert n > (1 << 30) + 32 + 8 * nch
    out = torch.empty_like(img)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.image_decompress_rle(dst, out, status, src_bytes=n)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert torch.equal(out, img)
    del out
    table = dst[32:32 + 8 * nch].view(torch.int32).view(nch, 2)
    for y in (0, 1, h // 2, h - 1):
        band = img[y:y + 1].cpu().numpy().view(np.uint32)
        want = oracle.rle_encode(np.ascontiguousarray(band), kind=1, flags=0)
        wtab = np.frombuffer(want[32:32 + 8 * S], dtype=np.uint32).reshape(S, 2)
        gtab = table[y * S:(y + 1) * S].cpu().numpy().view(np.uint32)
        base = int(gtab[0, 0])
        np.testing.assert_array_equal(gtab[:, 1], wtab[:, 1])
        np.testing.assert_array_equal(gtab[:, 0] - base, wtab[:, 0])
        payload = 32 + 8 * nch + base
        rec = bytes_of(dst[payload:], len(want) - 32 - 8 * S)
        assert rec == want[32 + 8 * S:], y
