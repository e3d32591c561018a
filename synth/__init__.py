"""Seeded synthetic frame-buffer generators (shared by tests and bench.py).

This module holds NONE of the method's arithmetic (no compositing, no blending,
no RLE, no swizzle): it only draws deterministic synthetic sort-last source
frames shaped like the thesis's workloads.  Both the oracle harness and the
CUDA harness consume its output; neither side's results feed back into it.

Recipes:

* ``depth_sources`` -- sort-last polygonal sources.
  Background = colour 0x00000000, depth 0xFFFFFFFF.  A model footprint is the
  union of 6 random ellipses sized to cover about ``F`` of the screen.  Each
  source draws 32 fragment ellipses whose centres lie in the footprint, whose
  total area is ``cover_i`` x footprint area with ``cover_i ~ U[1/sqrt(N), 1]``,
  clipped to the footprint ("scattered" round-robin allocation).
  Fragment depth is a plane z0 + gx*dx + gy*dy (z0 ~ U[2^28, 0xE0000000),
  |gx|, |gy| <= 2^16), clamped to [0, 0xFFFFFFFE]; within a source the nearer
  fragment wins.  Colour = per-fragment base RGB x a smooth radial shade,
  A = 255, plus ``noise_bits`` random low bits per channel.  ``ties=True``
  quantises depth (depth &= 0xFFFF0000) to force many equal depths.
* ``volume_bricks`` -- DB / volume decomposition: 16 bricks in a
  2x2x4 arrangement, emitted back to front; each brick covers a screen
  rectangle of ~30 % of the screen with ~50 % mutual overlap; inside,
  alpha = 16 + smooth polynomial in [16, 160], RGB = floor(base*alpha/255)
  (valid premultiplied) with 1 low noise bit clamped to <= alpha; outside 0.

Seeds: ``seed = 20190213 + config_index`` (the thesis approval date) by
convention of bench.py and the tests.
"""
from __future__ import annotations

import math

import numpy as np

BG_DEPTH = 0xFFFFFFFF
SEED_BASE = 20190213


def _ellipse_mask(h, w, cx, cy, rx, ry):
    """Return (y0, y1, x0, x1, mask) of the ellipse restricted to its bbox."""
    x0 = max(0, int(math.floor(cx - rx)))
    x1 = min(w, int(math.ceil(cx + rx)) + 1)
    y0 = max(0, int(math.floor(cy - ry)))
    y1 = min(h, int(math.ceil(cy + ry)) + 1)
    if x0 >= x1 or y0 >= y1:
        return y0, y0, x0, x0, np.zeros((0, 0), bool), None, None
    ys = (np.arange(y0, y1, dtype=np.float64)[:, None] + 0.5 - cy) / max(ry, 1e-9)
    xs = (np.arange(x0, x1, dtype=np.float64)[None, :] + 0.5 - cx) / max(rx, 1e-9)
    r2 = xs * xs + ys * ys
    return y0, y1, x0, x1, r2 <= 1.0, r2, (xs, ys)


def footprint(seed: int, w: int, h: int, F: float = 0.5) -> np.ndarray:
    """Union of 6 random ellipses covering roughly F of the screen (F >= 1:
    the whole screen)."""
    if F >= 1.0:
        return np.ones((h, w), bool)
    rng = np.random.default_rng([seed, 0xF00])
    fp = np.zeros((h, w), bool)
    area = F * w * h / 6.0 * 1.35  # overlap compensation
    for _ in range(6):
        aspect = float(rng.uniform(0.5, 2.0))
        rx = math.sqrt(area * aspect / math.pi)
        ry = math.sqrt(area / aspect / math.pi)
        cx = float(rng.uniform(0.2, 0.8)) * w
        cy = float(rng.uniform(0.2, 0.8)) * h
        y0, y1, x0, x1, m, _, _ = _ellipse_mask(h, w, cx, cy, rx, ry)
        if m.size:
            fp[y0:y1, x0:x1] |= m
    if not fp.any():
        fp[h // 2, w // 2] = True
    return fp


def kd_cells(n: int, x0: int, y0: int, x1: int, y1: int):
    """Split the rectangle [x0, x1) x [y0, y1) into n cells by recursive
    halving of the longer side (proportional to the cell counts)."""
    if n == 1:
        return [(x0, y0, x1, y1)]
    a = n // 2
    if x1 - x0 >= y1 - y0:
        xm = x0 + (x1 - x0) * a // n
        return kd_cells(a, x0, y0, xm, y1) + kd_cells(n - a, xm, y0, x1, y1)
    ym = y0 + (y1 - y0) * a // n
    return kd_cells(a, x0, y0, x1, ym) + kd_cells(n - a, x0, ym, x1, y1)


def depth_sources(seed: int, n: int, w: int, h: int, F: float = 0.5,
                  noise_bits: int = 1, ties: bool = False, pitch: int | None = None,
                  mode: str = "scattered", cover: float | None = None):
    """N sort-last source frames: (colors, depths), each a list of [H, W] uint32.

    ``mode="scattered"`` (default): every source's fragments fall anywhere in
    the footprint (round-robin allocation).  ``mode="compact"``:
    source i's fragment centres fall in the i-th kD cell of the footprint's
    bounding box (spatially compact allocation),
    so each source covers a small screen region -- the case the ROI targets.

    ``cover`` (default: drawn per source from U[1/sqrt(N), 1]) fixes every
    source's fragment area as a fraction of the footprint; with ``F`` >= 1,
    ``cover`` = 1 and more ``noise_bits`` the frames compress less (the
    compression-ratio anchors of DESIGN.md section 6).

    If ``pitch`` > W the arrays are [H, pitch] buffers and the returned frames
    are [H, W] views into them (row pitch = ``pitch`` words); the padding holds
    a recognisable garbage pattern so a kernel reading it would be caught.
    """
    fp = footprint(seed, w, h, F)
    fp_idx = np.flatnonzero(fp)
    fp_area = float(fp_idx.size)
    cells = None
    if mode == "compact":
        ys, xs = np.nonzero(fp)
        cells = kd_cells(n, int(xs.min()), int(ys.min()), int(xs.max()) + 1, int(ys.max()) + 1)
    elif mode != "scattered":
        raise ValueError(mode)
    colors, depths = [], []
    for i in range(n):
        rng = np.random.default_rng([seed, 1, i])
        src_idx, src_area = fp_idx, fp_area
        if cells is not None:
            cx0, cy0, cx1, cy1 = cells[i]
            sub = np.zeros_like(fp)
            sub[cy0:cy1, cx0:cx1] = fp[cy0:cy1, cx0:cx1]
            if sub.any():
                src_idx = np.flatnonzero(sub)
                src_area = float(src_idx.size)
        P = pitch if pitch is not None else w
        cbuf = np.full((h, P), 0xDEADBEEF, np.uint32)
        dbuf = np.full((h, P), 0x5A5A5A5A, np.uint32)
        col = cbuf[:, :w]
        dep = dbuf[:, :w]
        col[:] = 0
        dep[:] = BG_DEPTH
        cov = float(rng.uniform(1.0 / math.sqrt(max(n, 1)), 1.0))
        if cover is not None:
            cov = float(cover)
        frag_area = cov * src_area / 32.0 * 1.2
        for _f in range(32):
            c = int(src_idx[int(rng.integers(0, src_idx.size))])
            cy, cx = c // w + 0.5, c % w + 0.5
            aspect = float(rng.uniform(0.4, 2.5))
            rx = max(math.sqrt(frag_area * aspect / math.pi), 1.0)
            ry = max(math.sqrt(frag_area / aspect / math.pi), 1.0)
            y0, y1, x0, x1, m, r2, (xs, ys) = _ellipse_mask(h, w, cx, cy, rx, ry)
            if not m.size:
                continue
            m = m & fp[y0:y1, x0:x1]
            if not m.any():
                continue
            z0 = int(rng.integers(1 << 28, 0xE0000000))
            gx = int(rng.integers(-(1 << 16), (1 << 16) + 1))
            gy = int(rng.integers(-(1 << 16), (1 << 16) + 1))
            dx = (np.arange(x0, x1, dtype=np.int64)[None, :] - int(cx))
            dy = (np.arange(y0, y1, dtype=np.int64)[:, None] - int(cy))
            z = np.clip(z0 + gx * dx + gy * dy, 0, 0xFFFFFFFE).astype(np.uint32)
            if ties:
                z &= np.uint32(0xFFFF0000)
            base = rng.integers(32, 256, size=3)
            shade = 1.0 - 0.5 * np.clip(r2, 0.0, 1.0)
            rgb = [np.clip(np.floor(b * shade), 0, 255).astype(np.uint32) for b in base]
            if noise_bits:
                nmask = (1 << noise_bits) - 1
                nz = rng.integers(0, 1 << 30, size=(y1 - y0, x1 - x0), dtype=np.int64).astype(np.uint32)
                rgb = [(ch & ~np.uint32(nmask)) | ((nz >> np.uint32(8 * k)) & np.uint32(nmask))
                       for k, ch in enumerate(rgb)]
            pix = rgb[0] | (rgb[1] << np.uint32(8)) | (rgb[2] << np.uint32(16)) | np.uint32(0xFF000000)
            sub_d = dep[y0:y1, x0:x1]
            sub_c = col[y0:y1, x0:x1]
            win = m & (z < sub_d)  # the source's own z-buffer: nearer fragment wins
            sub_d[win] = z[win]
            sub_c[win] = pix[win]
        colors.append(col)
        depths.append(dep)
    return colors, depths


def volume_bricks(seed: int, n: int, w: int, h: int, pitch: int | None = None):
    """N premultiplied RGBA8 brick images, back to front (list of [H, W] uint32)."""
    rng = np.random.default_rng([seed, 2])
    out = []
    for k in range(n):
        bx, by, bz = k % 2, (k // 2) % 2, k // 4  # 2x2xN/4 arrangement
        P = pitch if pitch is not None else w
        buf = np.full((h, P), 0xDEADBEEF, np.uint32)
        img = buf[:, :w]
        img[:] = 0
        fw, fh = 0.55 * w, 0.55 * h  # ~30 % of the screen each
        x0 = int((0.05 + 0.40 * bx) * w + rng.uniform(-0.03, 0.03) * w + bz * 0.01 * w)
        y0 = int((0.05 + 0.40 * by) * h + rng.uniform(-0.03, 0.03) * h + bz * 0.01 * h)
        x1 = min(w, max(x0 + 1, int(x0 + fw)))
        y1 = min(h, max(y0 + 1, int(y0 + fh)))
        x0, y0 = max(0, x0), max(0, y0)
        if x0 >= x1 or y0 >= y1:
            out.append(img)
            continue
        u = (np.arange(x0, x1, dtype=np.float64)[None, :] + 0.5 - x0) / (x1 - x0)
        v = (np.arange(y0, y1, dtype=np.float64)[:, None] + 0.5 - y0) / (y1 - y0)
        ph = float(rng.uniform(0, 2 * math.pi))
        poly = (16.0 * u * (1 - u) * v * (1 - v)) * (0.75 + 0.25 * np.sin(6.0 * u + 4.0 * v + ph))
        alpha = np.clip(np.floor(16.0 + 144.0 * np.clip(poly, 0.0, 1.0)), 16, 160).astype(np.uint32)
        base = rng.integers(40, 256, size=3)
        chans = []
        nz = rng.integers(0, 1 << 30, size=alpha.shape, dtype=np.int64).astype(np.uint32)
        for c in range(3):
            ch = (np.uint32(base[c]) * alpha) // np.uint32(255)
            ch = (ch & ~np.uint32(1)) | ((nz >> np.uint32(c)) & np.uint32(1))
            ch = np.minimum(ch, alpha)
            chans.append(ch.astype(np.uint32))
        img[y0:y1, x0:x1] = chans[0] | (chans[1] << np.uint32(8)) | (chans[2] << np.uint32(16)) | (alpha << np.uint32(24))
        out.append(img)
    return out


def random_frames(seed: int, n: int, w: int, h: int, depth_alphabet=None):
    """Uniform-noise frames for fuzz tests: colours uniform u32, depths either
    uniform u32 or drawn from a small alphabet (to force ties)."""
    rng = np.random.default_rng([seed, 3])
    colors = [rng.integers(0, 1 << 32, size=(h, w), dtype=np.uint64).astype(np.uint32) for _ in range(n)]
    if depth_alphabet is None:
        depths = [rng.integers(0, 1 << 32, size=(h, w), dtype=np.uint64).astype(np.uint32) for _ in range(n)]
    else:
        alpha = np.asarray(depth_alphabet, dtype=np.uint64)
        depths = [alpha[rng.integers(0, len(alpha), size=(h, w))].astype(np.uint32) for _ in range(n)]
    return colors, depths


def premultiplied_noise(seed: int, n: int, w: int, h: int):
    """Random valid premultiplied RGBA8 layers (each RGB <= A) for blend fuzzing."""
    rng = np.random.default_rng([seed, 4])
    out = []
    for _ in range(n):
        a = rng.integers(0, 256, size=(h, w), dtype=np.int64)
        a[rng.random((h, w)) < 0.15] = 0
        a[rng.random((h, w)) < 0.15] = 255
        rgb = [np.floor(rng.random((h, w)) * (a + 1)).astype(np.int64) for _ in range(3)]
        rgb = [np.minimum(c, a) for c in rgb]
        out.append((rgb[0] | (rgb[1] << 8) | (rgb[2] << 16) | (a << 24)).astype(np.uint32))
    return out


def structured_planes(seed: int, count: int, max_len: int = 128):
    """Byte planes with runs, alternations and noise for RLE round-trip fuzzing."""
    rng = np.random.default_rng([seed, 5])
    out = []
    for _ in range(count):
        L = int(rng.integers(1, max_len + 1))
        kind = int(rng.integers(0, 5))
        if kind == 0:
            b = rng.integers(0, 256, size=L)
        elif kind == 1:
            b = np.full(L, int(rng.integers(0, 256)))
        elif kind == 2:  # runs of random length
            vals = []
            while len(vals) < L:
                vals += [int(rng.integers(0, 4))] * int(rng.integers(1, 7))
            b = np.array(vals[:L])
        elif kind == 3:  # alternations
            b = np.array([int(x) for x in (np.arange(L) % int(rng.integers(1, 4)))])
        else:  # small alphabet noise
            b = rng.integers(0, 2, size=L)
        out.append(bytes(np.asarray(b, dtype=np.uint8).tolist()))
    return out


def depth_sources_torch(seed: int, n: int, w: int, h: int, F: float = 0.3, noise_bits: int = 1,
                        device="cuda", indices=None):
    """The depth_sources recipe ("scattered" mode) generated ON THE GPU with
    torch, for the display-wall workload (config c5: 64 sources of
    15360x5760, 45 GB -- too large to draw on the host).  Same structure and
    parameter draws (footprint of 6 ellipses covering ~F, 32 fragment ellipses
    per source with planar depth and shaded colour, source-local z-buffer);
    the per-pixel noise comes from a torch generator seeded per fragment, so
    the frames differ from depth_sources' bit for bit but are a deterministic
    function of (seed, n, w, h, F, noise_bits).  Returns (colors, depths):
    lists of [H, W] int32 CUDA tensors (uint32 bit patterns) for the sources in
    `indices` (default all n).
    """
    import torch
    fp_np = footprint(seed, w, h, F)
    fp_idx = np.flatnonzero(fp_np)
    fp_area = float(fp_idx.size)
    fp = torch.from_numpy(fp_np).to(device)
    colors, depths = [], []
    for i in (range(n) if indices is None else indices):
        rng = np.random.default_rng([seed, 1, i])
        dep = torch.full((h, w), 0xFFFFFFFF, dtype=torch.int64, device=device)
        col = torch.zeros((h, w), dtype=torch.int64, device=device)
        cov = float(rng.uniform(1.0 / math.sqrt(max(n, 1)), 1.0))
        frag_area = cov * fp_area / 32.0 * 1.2
        for f in range(32):
            c = int(fp_idx[int(rng.integers(0, fp_idx.size))])
            cy, cx = c // w + 0.5, c % w + 0.5
            aspect = float(rng.uniform(0.4, 2.5))
            rx = max(math.sqrt(frag_area * aspect / math.pi), 1.0)
            ry = max(math.sqrt(frag_area / aspect / math.pi), 1.0)
            x0 = max(0, int(math.floor(cx - rx)))
            x1 = min(w, int(math.ceil(cx + rx)) + 1)
            y0 = max(0, int(math.floor(cy - ry)))
            y1 = min(h, int(math.ceil(cy + ry)) + 1)
            z0 = int(rng.integers(1 << 28, 0xE0000000))
            gx = int(rng.integers(-(1 << 16), (1 << 16) + 1))
            gy = int(rng.integers(-(1 << 16), (1 << 16) + 1))
            base = rng.integers(32, 256, size=3)
            nseed = int(rng.integers(0, 1 << 62))
            if x0 >= x1 or y0 >= y1:
                continue
            ys = (torch.arange(y0, y1, device=device, dtype=torch.float64)[:, None] + 0.5 - cy) / ry
            xs = (torch.arange(x0, x1, device=device, dtype=torch.float64)[None, :] + 0.5 - cx) / rx
            r2 = xs * xs + ys * ys
            m = (r2 <= 1.0) & fp[y0:y1, x0:x1]
            dx = torch.arange(x0, x1, device=device, dtype=torch.int64)[None, :] - int(cx)
            dy = torch.arange(y0, y1, device=device, dtype=torch.int64)[:, None] - int(cy)
            z = torch.clamp(z0 + gx * dx + gy * dy, 0, 0xFFFFFFFE)
            shade = 1.0 - 0.5 * torch.clamp(r2, 0.0, 1.0)
            rgb = [torch.clamp(torch.floor(float(b) * shade), 0, 255).to(torch.int64) for b in base]
            if noise_bits:
                nmask = (1 << noise_bits) - 1
                g = torch.Generator(device=device)
                g.manual_seed(nseed)
                nz = torch.randint(0, 1 << 30, (y1 - y0, x1 - x0), generator=g, device=device, dtype=torch.int64)
                rgb = [(ch & ~nmask) | ((nz >> (8 * k)) & nmask) for k, ch in enumerate(rgb)]
            pix = rgb[0] | (rgb[1] << 8) | (rgb[2] << 16) | 0xFF000000
            sub_d = dep[y0:y1, x0:x1]
            win = m & (z < sub_d)
            sub_d.copy_(torch.where(win, z, sub_d))
            sub_c = col[y0:y1, x0:x1]
            sub_c.copy_(torch.where(win, pix, sub_c))
        colors.append((col - ((col >> 31) << 32)).to(torch.int32))  # uint32 bit patterns as int32
        depths.append((dep - ((dep >> 31) << 32)).to(torch.int32))
        del dep, col
    return colors, depths
