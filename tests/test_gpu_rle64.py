"""GPU parity of the RLE-64 codec:
GPU streams byte-identical to the oracle's, GPU decode of oracle streams
exact, corrupt streams flagged, codec mixing rejected on the host."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import bytes_of, out_frame, stream_dev, to_dev, to_host  # noqa: E402


@pytest.fixture(scope="module")
def eqc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1902_08755_b200 import eqc as m
    return m


CASES = [("scene_640x64", 640, 64, None, 0, "scene"), ("odd_129x7", 129, 7, None, 0, "scene"),
         ("pitch_300x9_p304", 300, 9, 304, 0, "pairs"), ("one_px", 1, 1, None, 0, "noise"),
         ("misaligned_131x5", 131, 5, 136, 1, "pairs"), ("noise_256x8", 256, 8, None, 0, "noise"),
         ("flat_384x3", 384, 3, None, 0, "flat"), ("c2_1920x1080", 1920, 1080, None, 0, "scene")]


def _img(kind, w, h, seed):
    rng = np.random.default_rng(seed)
    if kind == "scene":
        c, d = synth.depth_sources(seed, 1, w, h)
        return [c[0], d[0]]
    if kind == "pairs":  # runs of equal pixel pairs, odd run lengths, small alphabet
        a = rng.integers(0, 3, size=(h, (w + 1) // 2)).astype(np.uint32) * np.uint32(0x01010101)
        a = np.repeat(a, 2, axis=1)[:, :w]
        a[:, ::7] ^= np.uint32(1)
        return [np.ascontiguousarray(a)]
    if kind == "flat":
        return [np.full((h, w), 0x12345678, np.uint32)]
    return [rng.integers(0, 1 << 32, size=(h, w), dtype=np.uint64).astype(np.uint32)]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_rle64_encode_bytes_exact_and_decode(eqc, case):
    name, w, h, pitch, offset, kind = case
    imgs = _img(kind, w, h, synth.SEED_BASE + 66 + w)
    dev = [to_dev(x, pitch, offset) for x in imgs]
    cap = eqc.image_rle_max_size(w, h)
    streams = [torch.zeros(cap, dtype=torch.uint8, device="cuda") for _ in imgs]
    sizes = torch.zeros(len(imgs), dtype=torch.int64, device="cuda")
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(len(imgs), w, h), dtype=torch.uint8, device="cuda")
    kinds = [0, 1][:len(imgs)]
    eqc.image_compress_rle_batch(dev, kinds, [eqc.FLAG_RLE64] * len(imgs), streams, sizes, ws)
    torch.cuda.synchronize()
    for img, k, st, n in zip(imgs, kinds, streams, sizes.tolist()):
        want = oracle.rle64_encode(img, k)
        assert n == len(want)
        assert bytes_of(st, n) == want
    outs = [out_frame(h, w, pitch, offset) for _ in imgs]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.image_decompress_rle_batch(streams, outs, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    for img, o in zip(imgs, outs):
        np.testing.assert_array_equal(to_host(o), img)


def test_rle64_decode_oracle_streams_and_mixed_batch(eqc):
    w, h = 515, 11
    c, d = synth.depth_sources(synth.SEED_BASE + 67, 2, w, h)
    streams = [oracle.rle64_encode(c[0], 0), oracle.rle_encode(c[1], 0, 1), oracle.rle64_encode(d[0], 1)]
    srcs = [stream_dev(s, pad=5) for s in streams]
    outs = [out_frame(h, w) for _ in streams]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.image_decompress_rle_batch(srcs, outs, status)  # the decoder takes either codec per stream
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    for img, o in zip([c[0], c[1], d[0]], outs):
        np.testing.assert_array_equal(to_host(o), img)


def test_rle64_corruption_flagged(eqc):
    w, h = 260, 6
    img = _img("pairs", w, h, 5)[0]
    good = bytearray(oracle.rle64_encode(img, 0))
    for pos, val in [(6, 3), (32 + 4, 250), (32 + 8 * 3, 7), (32 + 8 * 3 * 6, 1), (len(good) - 3, 0x55)]:
        t = bytearray(good)
        t[pos] = val
        rc_oracle = oracle.rle64_decode(bytes(t), w, h)[0]
        out = out_frame(h, w)
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        eqc.image_decompress_rle_batch([stream_dev(bytes(t))], [out], status)
        torch.cuda.synchronize()
        if rc_oracle != 0:
            assert int(status.item()) == eqc.E_CORRUPT, pos
        else:  # still a valid stream: identical decode
            np.testing.assert_array_equal(to_host(out), oracle.rle64_decode(bytes(t), w, h)[1])


def test_rle64_host_validation(eqc):
    w, h = 64, 4
    a = to_dev(np.zeros((h, w), np.uint32))
    cap = eqc.image_rle_max_size(w, h)
    st = [torch.zeros(cap, dtype=torch.uint8, device="cuda") for _ in range(2)]
    sz = torch.zeros(2, dtype=torch.int64, device="cuda")
    ws = torch.zeros(eqc.image_rle_workspace_size_batch(2, w, h), dtype=torch.uint8, device="cuda")
    with pytest.raises(eqc.EqcError):  # one codec per batch
        eqc.image_compress_rle_batch([a, a], [0, 0], [eqc.FLAG_RLE64, 0], st, sz, ws)
    with pytest.raises(eqc.EqcError) as e:  # swizzle + 64-bit tokens
        eqc.image_compress_rle_batch([a], [0], [eqc.FLAG_RLE64 | eqc.FLAG_SWIZZLE], st[:1], sz, ws)
    assert e.value.code == eqc.E_UNSUPPORTED


def test_fused_decode_rejects_rle64(eqc):
    w, h = 128, 2
    c, d = synth.depth_sources(3, 1, w, h)
    cs, ds = stream_dev(oracle.rle64_encode(c[0], 0)), stream_dev(oracle.rle_encode(d[0], 1))
    oc = out_frame(h, w)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    eqc.compositor_depth_rle([cs], [ds], oc, None, status)
    torch.cuda.synchronize()
    assert int(status.item()) == eqc.E_CORRUPT  # the fused path takes per-component streams only


def test_rle64_golden_streams_on_gpu(eqc):
    """The hand-derived RLE-64 streams (tests/golden/rle64_streams.txt): the
    GPU encoder emits them byte for byte and the GPU decoder inverts them."""
    from test_oracle_rle64 import golden_rle64_streams
    for name, kind, img, want in golden_rle64_streams():
        h, w = img.shape
        cap = eqc.image_rle_max_size(w, h)
        st = torch.zeros(cap, dtype=torch.uint8, device="cuda")
        sz = torch.zeros(1, dtype=torch.int64, device="cuda")
        ws = torch.zeros(eqc.image_rle_workspace_size_batch(1, w, h), dtype=torch.uint8, device="cuda")
        eqc.image_compress_rle_batch([to_dev(img)], [kind], [eqc.FLAG_RLE64], [st], sz, ws)
        torch.cuda.synchronize()
        assert int(sz.item()) == len(want), name
        assert bytes_of(st, len(want)) == want, name
        out = out_frame(h, w)
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        eqc.image_decompress_rle_batch([stream_dev(want)], [out], status)
        torch.cuda.synchronize()
        assert int(status.item()) == 0, name
        np.testing.assert_array_equal(to_host(out), img)
