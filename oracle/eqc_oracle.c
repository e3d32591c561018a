/*
 * eqc_oracle.c -- plain, slow, single-threaded CPU oracle for the sort-last
 * compositing + RLE transport hot path of Eilemann, "Parallel Rendering and
 * Large Data Visualization" (arxiv 1902.08755, PhD thesis UZH 2019).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1902_08755_b200/, libeqc.so) never links, calls or
 * includes anything from here, and this file includes nothing from there.
 *
 * Citation keys: "P:n" = line n of the thesis text; "S:n" = line n
 * of SPEC.md (used for test ideas only); "R-Cn" = reading Cn of the ambiguity
 * register in DESIGN.md section 3 (= SURVEY.md section 8(c)).
 *
 * Pin status (see DESIGN.md section 4 and tests/test_oracle_*.py):
 *   or_depth_composite   pinned: exhaustive brute force, worked example D,
 *                        permutation/monotone-transform invariants.
 *   or_blend_ordered     pinned: closed form for identical layers, expanded
 *                        (non-recursive) exact-rational sum, a in {0,255}
 *                        special cases, worked example B.
 *   or_swizzle/unswizzle pinned: hand bit traces, bijection.
 *   or_rle_encode/decode pinned: hand-derived byte strings (tests/golden),
 *                        round trip, size bound, brute-force token
 *                        minimality properties.  Compression MAGNITUDES vs the
 *                        paper's 10/25/40 % are "parity unpinned" (the paper's
 *                        dataset is unavailable).
 *   or_roi               pinned: numpy nonzero bounding boxes, empty / single
 *                        pixel / full frames.
 *   or_rle64_*           pinned: hand-derived record bytes (tests/golden),
 *                        round trips, canonical-form checker (maximal runs,
 *                        literal spans never hold a run of 2), size bound,
 *                        corrupt-stream rejection.
 *   or_average           pinned: numpy integer mean with explicit half-up
 *                        rounding, n = 1 identity, equal sources, permutation
 *                        invariance, exact .5 ties rounding up.
 *   or_*_roi             pinned: reduction to O1 / O2 on frames masked outside
 *                        the rectangle (the definition of ROI placement), and
 *                        invariance under cropping to the exact bounding box.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define OR_OK 0
#define OR_E_INVALID (-1)
#define OR_E_CAPACITY (-2)
#define OR_E_CORRUPT (-3)
#define OR_E_UNSUPPORTED (-4)

/* ------------------------------------------------------------------------ */
/* O1 depth-sorted sort-last compositing                                      */
/* ------------------------------------------------------------------------ */
/*
 * "assigns the final pixel to the colour of the source with the
 * front-most depth buffer values".  R-C1: depth is u32, smaller = nearer.
 * R-C2: ties go to the lower source index.  Written as the plain definition:
 * k* = argmin over i of the pair (depth_i[p], i), compared lexicographically.
 * out_depth may be NULL (colour-only output, R-C15).
 */
void or_depth_composite(int n, const uint32_t *const *color,
                        const uint32_t *const *depth, int w, int h,
                        int64_t pitch, uint32_t *out_color,
                        uint32_t *out_depth, int64_t out_pitch) {
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      int64_t p = (int64_t)y * pitch + x;
      int best = 0;
      for (int i = 1; i < n; ++i) {
        uint32_t di = depth[i][p], db = depth[best][p];
        /* lexicographic (depth, index): i > best always, so only a strictly
           smaller depth makes i the new minimum */
        if (di < db || (di == db && i < best)) best = i;
      }
      int64_t q = (int64_t)y * out_pitch + x;
      out_color[q] = color[best][p];
      if (out_depth) out_depth[q] = depth[best][p];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* O2 ordered (spatial) back-to-front alpha compositing                       */
/* ------------------------------------------------------------------------ */
/*
 * partial images are depth-sorted and "composited in order,
 * typically with alpha-blending"; the application supplies the order
 * (P:1598-1600).  R-C3: premultiplied Porter-Duff "over".  R-C4: the chain is
 * evaluated exactly (double here) and rounded ONCE at the end, half up.
 *   x_{-1} = bg_c / 255
 *   x_k    = s_{k,c} / 255 + x_{k-1} * (1 - a_k / 255)     k = 0..n-1
 *   out_c  = clamp(floor(255 * x_{n-1} + 1/2), 0, 255)
 * Position k = 0 is the farthest layer; order[k] names the source drawn k-th
 * (NULL = identity).  Byte c of a pixel is channel c (R-C7: R = byte 0,
 * A = byte 3).
 */
void or_blend_ordered(int n, const uint32_t *const *color,
                      const int32_t *order, int w, int h, int64_t pitch,
                      uint32_t background, uint32_t *out_color,
                      int64_t out_pitch) {
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      int64_t p = (int64_t)y * pitch + x;
      double xc[4];
      for (int c = 0; c < 4; ++c) xc[c] = (double)((background >> (8 * c)) & 0xFFu) / 255.0;
      for (int k = 0; k < n; ++k) {
        int src = order ? order[k] : k;
        uint32_t s = color[src][p];
        double a = (double)(s >> 24) / 255.0;
        for (int c = 0; c < 4; ++c) {
          double sc = (double)((s >> (8 * c)) & 0xFFu) / 255.0;
          xc[c] = sc + xc[c] * (1.0 - a);
        }
      }
      uint32_t o = 0;
      for (int c = 0; c < 4; ++c) {
        double v = floor(255.0 * xc[c] + 0.5);
        if (v < 0.0) v = 0.0;
        if (v > 255.0) v = 255.0;
        o |= ((uint32_t)v) << (8 * c);
      }
      out_color[(int64_t)y * out_pitch + x] = o;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Swizzle preconditioner                                                     */
/* ------------------------------------------------------------------------ */
/*
 * "reorders and interleaves the per-component bits ... by
 * grouping them by significance".  The figure is missing;
 * R-C9 takes S:429: output bit 4b + (3 - c) = bit b of channel c, channels
 * c = 0 R, 1 G, 2 B, 3 A (bit 31 = R7, 30 = G7, 29 = B7, 28 = A7, ...,
 * 0 = A0).  Written as the bit-by-bit definition.
 */
uint32_t or_swizzle(uint32_t v) {
  uint32_t o = 0;
  for (int c = 0; c < 4; ++c)
    for (int b = 0; b < 8; ++b)
      if ((v >> (8 * c + b)) & 1u) o |= 1u << (4 * b + (3 - c));
  return o;
}

uint32_t or_unswizzle(uint32_t v) {
  uint32_t o = 0;
  for (int c = 0; c < 4; ++c)
    for (int b = 0; b < 8; ++b)
      if ((v >> (4 * b + (3 - c))) & 1u) o |= 1u << (8 * c + b);
  return o;
}

/* ------------------------------------------------------------------------ */
/* RLE-BP v1: per-component (byte-plane) RLE, chunked by row segments         */
/* ------------------------------------------------------------------------ */
/*
 * "treat each colour component separately by producing four
 * independent RLE-compressed output streams".  P:2427-2430: "All RLE
 * compressors perform a data decomposition on the input image" (chunks).
 * The bit stream is reading R-C8:
 *   chunk = C = 2^log2c pixels of one row (last chunk of a row may be short);
 *   plane p of a chunk = byte p of each (optionally swizzled) word, x order;
 *   plane record = [ntok u8][ctrl u8 x ntok][payloads], where each maximal
 *   run of >= 3 equal bytes is a REPEAT token (ctrl 0x80|(len-1), payload =
 *   the byte) and each maximal span not covered by REPEAT tokens is a
 *   LITERAL token (ctrl len-1, payload = the bytes);
 *   stream = 32 B header, 8 B table entry per chunk {u32 payload offset,
 *   u8 plane_size[4]}, then chunk records in chunk-id order.
 */
#define RLE_MAGIC 0x4C525145u /* "EQRL" little-endian */
#define RLE_VERSION 1

static void put_u32(uint8_t *d, uint32_t v) {
  d[0] = (uint8_t)v; d[1] = (uint8_t)(v >> 8); d[2] = (uint8_t)(v >> 16); d[3] = (uint8_t)(v >> 24);
}
static void put_u64(uint8_t *d, uint64_t v) {
  put_u32(d, (uint32_t)v); put_u32(d + 4, (uint32_t)(v >> 32));
}
static uint32_t get_u32(const uint8_t *d) {
  return (uint32_t)d[0] | ((uint32_t)d[1] << 8) | ((uint32_t)d[2] << 16) | ((uint32_t)d[3] << 24);
}
static uint64_t get_u64(const uint8_t *d) {
  return (uint64_t)get_u32(d) | ((uint64_t)get_u32(d + 4) << 32);
}

int64_t or_rle_max_size(int w, int h, int log2c) {
  if (w <= 0 || h <= 0 || log2c < 5 || log2c > 7) return OR_E_INVALID;
  int64_t C = 1 << log2c;
  int64_t S = (w + C - 1) / C;
  return 32 + 16 * S * (int64_t)h + 4 * (int64_t)w * h;
}

/*
 * Encode one plane record of L bytes b[0..L) into out; returns its size.
 * Step 1: find maximal runs.  Step 2: runs of length >= 3 -> REPEAT.
 * Step 3: maximal spans of bytes not in a REPEAT -> one LITERAL each.
 * Step 4: record = [ntok][ctrl...][payload...].
 */
int or_rle_encode_plane(const uint8_t *b, int L, uint8_t *out) {
  uint8_t ctrl[256];
  uint8_t payload[256];
  int ntok = 0, npay = 0;
  int lit_start = -1; /* start of the open literal span, -1 if none */
  int i = 0;
  while (i < L) {
    int j = i + 1;
    while (j < L && b[j] == b[i]) ++j; /* maximal run [i, j) */
    int run = j - i;
    if (run >= 3) {
      if (lit_start >= 0) { /* close the pending literal span */
        int len = i - lit_start;
        ctrl[ntok++] = (uint8_t)(len - 1);
        for (int k = lit_start; k < i; ++k) payload[npay++] = b[k];
        lit_start = -1;
      }
      ctrl[ntok++] = (uint8_t)(0x80 | (run - 1));
      payload[npay++] = b[i];
    } else if (lit_start < 0) {
      lit_start = i;
    }
    i = j;
  }
  if (lit_start >= 0) {
    int len = L - lit_start;
    ctrl[ntok++] = (uint8_t)(len - 1);
    for (int k = lit_start; k < L; ++k) payload[npay++] = b[k];
  }
  out[0] = (uint8_t)ntok;
  memcpy(out + 1, ctrl, (size_t)ntok);
  memcpy(out + 1 + ntok, payload, (size_t)npay);
  return 1 + ntok + npay;
}

/*
 * Decode one plane record of exactly rec_size bytes into L bytes.
 * Returns 0 or OR_E_CORRUPT (ntok < 1, token lengths not summing to L,
 * payload size inconsistent with rec_size).
 */
int or_rle_decode_plane(const uint8_t *rec, int rec_size, int L, uint8_t *b) {
  if (rec_size < 1) return OR_E_CORRUPT;
  int ntok = rec[0];
  if (ntok < 1 || 1 + ntok > rec_size) return OR_E_CORRUPT;
  const uint8_t *ctrl = rec + 1;
  int pay = 1 + ntok;
  int pos = 0;
  for (int t = 0; t < ntok; ++t) {
    int len = (ctrl[t] & 0x7F) + 1;
    if (pos + len > L) return OR_E_CORRUPT;
    if (ctrl[t] & 0x80) {
      if (pay + 1 > rec_size) return OR_E_CORRUPT;
      for (int k = 0; k < len; ++k) b[pos + k] = rec[pay];
      pay += 1;
    } else {
      if (pay + len > rec_size) return OR_E_CORRUPT;
      for (int k = 0; k < len; ++k) b[pos + k] = rec[pay + k];
      pay += len;
    }
    pos += len;
  }
  if (pos != L || pay != rec_size) return OR_E_CORRUPT;
  return OR_OK;
}

/*
 * Encode a W x H image of 32-bit words (row pitch in words) into dst.
 * kind 0 = RGBA8 colour, 1 = depth u32; flags bit 0 = swizzle (colour only,
 * R-C11).  Returns the stream size in bytes, or a negative error.
 */
int64_t or_rle_encode(const uint32_t *src, int w, int h, int64_t pitch,
                      int kind, int flags, int log2c, uint8_t *dst,
                      int64_t cap) {
  if (!src || !dst || w <= 0 || h <= 0 || pitch < w) return OR_E_INVALID;
  if (kind != 0 && kind != 1) return OR_E_INVALID;
  if (flags & ~1) return OR_E_INVALID;
  if (kind == 1 && (flags & 1)) return OR_E_UNSUPPORTED;
  if (log2c < 5 || log2c > 7) return OR_E_INVALID;
  int C = 1 << log2c;
  int S = (w + C - 1) / C;
  int64_t nchunks = (int64_t)S * h;
  if (nchunks > 0xFFFFFFFFll) return OR_E_INVALID;
  int64_t table = 32, payload0 = 32 + 8 * nchunks;
  if (cap < payload0) return OR_E_CAPACITY;
  uint8_t plane[128];
  uint8_t rec[4][130];
  int64_t off = 0; /* payload offset of the current chunk */
  for (int y = 0; y < h; ++y) {
    for (int k = 0; k < S; ++k) {
      int x0 = k * C;
      int L = (w - x0 < C) ? (w - x0) : C;
      int sz[4];
      for (int p = 0; p < 4; ++p) {
        for (int i = 0; i < L; ++i) {
          uint32_t v = src[(int64_t)y * pitch + x0 + i];
          if (flags & 1) v = or_swizzle(v);
          plane[i] = (uint8_t)(v >> (8 * p));
        }
        sz[p] = or_rle_encode_plane(plane, L, rec[p]);
      }
      int64_t chunk_id = (int64_t)y * S + k;
      int64_t total = sz[0] + sz[1] + sz[2] + sz[3];
      if (off > 0xFFFFFFFFll) return OR_E_INVALID; /* u32 offset field */
      if (payload0 + off + total > cap) return OR_E_CAPACITY;
      uint8_t *te = dst + table + 8 * chunk_id;
      put_u32(te, (uint32_t)off);
      for (int p = 0; p < 4; ++p) te[4 + p] = (uint8_t)sz[p];
      uint8_t *o = dst + payload0 + off;
      for (int p = 0; p < 4; ++p) { memcpy(o, rec[p], (size_t)sz[p]); o += sz[p]; }
      off += total;
    }
  }
  put_u32(dst + 0, RLE_MAGIC);
  dst[4] = RLE_VERSION;
  dst[5] = (uint8_t)kind;
  dst[6] = (uint8_t)flags;
  dst[7] = (uint8_t)log2c;
  put_u32(dst + 8, (uint32_t)w);
  put_u32(dst + 12, (uint32_t)h);
  put_u32(dst + 16, (uint32_t)nchunks);
  put_u32(dst + 20, 0);
  put_u64(dst + 24, (uint64_t)off);
  return payload0 + off;
}

/*
 * Decode a stream into a W x H image (row pitch in words).  The caller states
 * the expected W and H; the header must agree.  Validation follows DESIGN.md
 * section 5: magic/version/kind/flags/log2c, W/H and chunk count, offsets
 * monotone and contiguous, each plane record well formed, total size.
 */
int or_rle_decode(const uint8_t *src, int64_t src_bytes, uint32_t *dst,
                  int64_t pitch, int w, int h) {
  if (!src || !dst || w <= 0 || h <= 0 || pitch < w) return OR_E_INVALID;
  if (src_bytes < 32) return OR_E_CORRUPT;
  if (get_u32(src) != RLE_MAGIC || src[4] != RLE_VERSION) return OR_E_CORRUPT;
  int kind = src[5], flags = src[6], log2c = src[7];
  if (kind > 1 || (flags & ~1) || (kind == 1 && flags) || log2c < 5 || log2c > 7)
    return OR_E_CORRUPT;
  if ((int64_t)get_u32(src + 8) != w || (int64_t)get_u32(src + 12) != h) return OR_E_CORRUPT;
  int C = 1 << log2c;
  int S = (w + C - 1) / C;
  int64_t nchunks = (int64_t)S * h;
  if ((int64_t)get_u32(src + 16) != nchunks || get_u32(src + 20) != 0) return OR_E_CORRUPT;
  uint64_t pbytes = get_u64(src + 24);
  int64_t payload0 = 32 + 8 * nchunks;
  if ((uint64_t)src_bytes < (uint64_t)payload0 || (uint64_t)(src_bytes - payload0) < pbytes)
    return OR_E_CORRUPT;
  uint8_t plane[128];
  uint64_t expect = 0;
  for (int y = 0; y < h; ++y) {
    for (int k = 0; k < S; ++k) {
      int x0 = k * C;
      int L = (w - x0 < C) ? (w - x0) : C;
      int64_t chunk_id = (int64_t)y * S + k;
      const uint8_t *te = src + 32 + 8 * chunk_id;
      uint64_t off = get_u32(te);
      if (off != expect) return OR_E_CORRUPT; /* monotone and contiguous */
      uint64_t total = (uint64_t)te[4] + te[5] + te[6] + te[7];
      if (off + total > pbytes) return OR_E_CORRUPT;
      const uint8_t *r = src + payload0 + off;
      for (int i = 0; i < L; ++i) dst[(int64_t)y * pitch + x0 + i] = 0;
      for (int p = 0; p < 4; ++p) {
        int rc = or_rle_decode_plane(r, te[4 + p], L, plane);
        if (rc) return rc;
        for (int i = 0; i < L; ++i)
          dst[(int64_t)y * pitch + x0 + i] |= (uint32_t)plane[i] << (8 * p);
        r += te[4 + p];
      }
      if (flags & 1)
        for (int i = 0; i < L; ++i)
          dst[(int64_t)y * pitch + x0 + i] = or_unswizzle(dst[(int64_t)y * pitch + x0 + i]);
      expect = off + total;
    }
  }
  if (expect != pbytes) return OR_E_CORRUPT;
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Region of interest                                    */
/* ------------------------------------------------------------------------ */
/*
 * "The ROI is the screen-space 2D bounding box fully enclosing
 * the data rendered by a single resource"; the ROI can be
 * computed automatically "by analysing the framebuffer".  Plain definition:
 * the smallest axis-aligned rectangle {x, y, w, h} containing every pixel
 * whose value differs from `background` (for a depth buffer: 0xFFFFFFFF,
 * R-C1); {0, 0, 0, 0} when there is no such pixel (R-C18).
 */
void or_roi(const uint32_t *frame, int w, int h, int64_t pitch, uint32_t background, int32_t out[4]) {
  int x0 = w, y0 = h, x1 = -1, y1 = -1;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x)
      if (frame[(int64_t)y * pitch + x] != background) {
        if (x < x0) x0 = x;
        if (x > x1) x1 = x;
        if (y < y0) y0 = y;
        if (y > y1) y1 = y;
      }
  if (x1 < 0) {
    out[0] = out[1] = out[2] = out[3] = 0;
    return;
  }
  out[0] = x0;
  out[1] = y0;
  out[2] = x1 - x0 + 1;
  out[3] = y1 - y0 + 1;
}

/* R-C19: a rectangle is clipped to the frame; no pixel lies outside it. */
static void roi_clip(const int32_t *r, int w, int h, int32_t *c) {
  int64_t x0 = r[0], y0 = r[1], x1 = (int64_t)r[0] + r[2], y1 = (int64_t)r[1] + r[3];
  if (x0 < 0) x0 = 0;
  if (y0 < 0) y0 = 0;
  if (x1 > w) x1 = w;
  if (y1 > h) y1 = h;
  if (r[2] <= 0 || r[3] <= 0 || x1 <= x0 || y1 <= y0) x0 = y0 = x1 = y1 = 0;
  c[0] = (int32_t)x0;
  c[1] = (int32_t)y0;
  c[2] = (int32_t)(x1 - x0);
  c[3] = (int32_t)(y1 - y0);
}

static int in_roi(const int32_t *r, int x, int y) {
  return x >= r[0] && x < r[0] + r[2] && y >= r[1] && y < r[1] + r[3];
}

/*
 * the ROI "is transmitted to all input frames together with the
 * pixel data.  On the input frame, the compositing code respects this
 * parameter to place the pixel data in the right position."  Source i
 * supplies pixel data only inside roi[4i..4i+3] = {x, y, w, h} (full-frame
 * coordinates, buffer indexed like a full frame); everywhere else it is
 * background (depth 0xFFFFFFFF, colour 0, R-C1).  The result is O1 over the
 * sources expanded that way.  Rectangles are clipped to the frame (R-C19).
 */
int or_depth_composite_roi(int n, const uint32_t *const *color, const uint32_t *const *depth,
                           const int32_t *roi, int w, int h, int64_t pitch, uint32_t *out_color,
                           uint32_t *out_depth, int64_t out_pitch) {
  int32_t rc[4 * 64];
  if (n < 1 || n > 64) return OR_E_INVALID;
  for (int i = 0; i < n; ++i) roi_clip(roi + 4 * i, w, h, rc + 4 * i);
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      int64_t p = (int64_t)y * pitch + x;
      int best = -1;
      uint32_t bd = 0, bc = 0;
      for (int i = 0; i < n; ++i) {
        int inside = in_roi(rc + 4 * i, x, y);
        uint32_t di = inside ? depth[i][p] : 0xFFFFFFFFu;
        uint32_t ci = inside ? color[i][p] : 0u;
        if (best < 0 || di < bd) { /* (depth, index) order: i > best */
          best = i;
          bd = di;
          bc = ci;
        }
      }
      int64_t q = (int64_t)y * out_pitch + x;
      out_color[q] = bc;
      if (out_depth) out_depth[q] = bd;
    }
  }
  return OR_OK;
}

/*
 * O2 over ROI-restricted layers: outside its rectangle a layer is fully
 * transparent (premultiplied 0), which leaves the running value unchanged.
 */
int or_blend_ordered_roi(int n, const uint32_t *const *color, const int32_t *order, const int32_t *roi,
                         int w, int h, int64_t pitch, uint32_t background, uint32_t *out_color,
                         int64_t out_pitch) {
  int32_t rc[4 * 64];
  if (n < 1 || n > 64) return OR_E_INVALID;
  for (int i = 0; i < n; ++i) roi_clip(roi + 4 * i, w, h, rc + 4 * i);
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      int64_t p = (int64_t)y * pitch + x;
      double xc[4];
      for (int c = 0; c < 4; ++c) xc[c] = (double)((background >> (8 * c)) & 0xFFu) / 255.0;
      for (int k = 0; k < n; ++k) {
        int src = order ? order[k] : k;
        uint32_t s = in_roi(rc + 4 * src, x, y) ? color[src][p] : 0u;
        double a = (double)(s >> 24) / 255.0;
        for (int c = 0; c < 4; ++c) {
          double sc = (double)((s >> (8 * c)) & 0xFFu) / 255.0;
          xc[c] = sc + xc[c] * (1.0 - a);
        }
      }
      uint32_t o = 0;
      for (int c = 0; c < 4; ++c) {
        double v = floor(255.0 * xc[c] + 0.5);
        if (v < 0.0) v = 0.0;
        if (v > 255.0) v = 255.0;
        o |= ((uint32_t)v) << (8 * c);
      }
      out_color[(int64_t)y * out_pitch + x] = o;
    }
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Subpixel compositing: accumulation and averaging      */
/* ------------------------------------------------------------------------ */
/*
 * subpixel compounds' "default compositing algorithm uses
 * accumulation and averaging of all computed fragments for a pixel".  Plain
 * definition per channel c: out_c = the mean of the n source values rounded
 * half up, i.e. floor((2 * sum_i s_ic + n) / (2 n)) in integers (R-C22).
 */
void or_average(int n, const uint32_t *const *color, int w, int h, int64_t pitch, uint32_t *out_color,
                int64_t out_pitch) {
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      int64_t p = (int64_t)y * pitch + x;
      uint32_t o = 0;
      for (int c = 0; c < 4; ++c) {
        uint64_t sum = 0;
        for (int i = 0; i < n; ++i) sum += (color[i][p] >> (8 * c)) & 0xFFu;
        uint64_t v = (2 * sum + (uint64_t)n) / (2 * (uint64_t)n);
        o |= (uint32_t)v << (8 * c);
      }
      out_color[(int64_t)y * out_pitch + x] = o;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* RLE-64: the basic 64-bit token codec (reading R-C17)   */
/* ------------------------------------------------------------------------ */
/*
 * "a fast 64-bit version comparing two pixels at the same time
 * (8 bit per channel RGBA format) ... it can only compress adjacent pixels of
 * the same colour".  Reading R-C17 (wire format in DESIGN.md section 5): the
 * stream is RLE-BP v1's (same header, chunking and table) with header flags
 * = EQC_FLAG_RLE64 (2).  A chunk of L pixels is U = ceil(L / 2) 64-bit units,
 * unit u = pixel 2u | pixel 2u+1 << 32 (for odd L the last unit's high half
 * is 0).  Maximal runs of >= 2 equal units become REPEAT tokens (ctrl = 0x80 |
 * (len - 1), payload = the unit, 8 bytes little-endian); each maximal span of
 * other units becomes one LITERAL token (ctrl = len - 1, payload = the
 * units).  Record = [ntok u8][ctrl x ntok][payloads]; the table entry's
 * second word is the record size (u32) instead of four plane sizes.
 */
static uint64_t unit64(const uint32_t *row, int L, int u) {
  uint64_t lo = row[2 * u];
  uint64_t hi = (2 * u + 1 < L) ? row[2 * u + 1] : 0u;
  return lo | (hi << 32);
}

static void put_u64le(uint8_t *d, uint64_t v) {
  for (int b = 0; b < 8; ++b) d[b] = (uint8_t)(v >> (8 * b));
}

/* Encode one chunk (row pointer, L pixels); returns the record size. */
int or_rle64_encode_chunk(const uint32_t *row, int L, uint8_t *out) {
  int U = (L + 1) / 2;
  uint8_t ctrl[64];
  uint8_t pay[8 * 64];
  int ntok = 0, np = 0, i = 0;
  while (i < U) {
    uint64_t v = unit64(row, L, i);
    int j = i + 1;
    while (j < U && unit64(row, L, j) == v) ++j;
    if (j - i >= 2) { /* REPEAT */
      ctrl[ntok++] = (uint8_t)(0x80 | (j - i - 1));
      put_u64le(pay + np, v);
      np += 8;
      i = j;
    } else { /* LITERAL: up to the start of the next run of >= 2 */
      int s = i;
      while (i < U && !(i + 1 < U && unit64(row, L, i + 1) == unit64(row, L, i))) {
        put_u64le(pay + np, unit64(row, L, i));
        np += 8;
        ++i;
      }
      ctrl[ntok++] = (uint8_t)(i - s - 1);
    }
  }
  out[0] = (uint8_t)ntok;
  memcpy(out + 1, ctrl, (size_t)ntok);
  memcpy(out + 1 + ntok, pay, (size_t)np);
  return 1 + ntok + np;
}

int64_t or_rle64_encode(const uint32_t *src, int w, int h, int64_t pitch, int kind, uint8_t *dst, int64_t cap) {
  if (!src || !dst || w <= 0 || h <= 0 || pitch < w) return OR_E_INVALID;
  if (kind != 0 && kind != 1) return OR_E_INVALID;
  const int C = 128, log2c = 7;
  int S = (w + C - 1) / C;
  int64_t nchunks = (int64_t)S * h;
  int64_t payload0 = 32 + 8 * nchunks;
  if (cap < payload0) return OR_E_CAPACITY;
  uint8_t rec[1 + 64 + 8 * 64];
  int64_t off = 0;
  for (int y = 0; y < h; ++y) {
    for (int k = 0; k < S; ++k) {
      int x0 = k * C;
      int L = (w - x0 < C) ? (w - x0) : C;
      int sz = or_rle64_encode_chunk(src + (int64_t)y * pitch + x0, L, rec);
      int64_t chunk_id = (int64_t)y * S + k;
      if (off > 0xFFFFFFFFll) return OR_E_INVALID;
      if (payload0 + off + sz > cap) return OR_E_CAPACITY;
      put_u32(dst + 32 + 8 * chunk_id, (uint32_t)off);
      put_u32(dst + 32 + 8 * chunk_id + 4, (uint32_t)sz);
      memcpy(dst + payload0 + off, rec, (size_t)sz);
      off += sz;
    }
  }
  put_u32(dst + 0, RLE_MAGIC);
  dst[4] = RLE_VERSION;
  dst[5] = (uint8_t)kind;
  dst[6] = 2; /* EQC_FLAG_RLE64 */
  dst[7] = (uint8_t)log2c;
  put_u32(dst + 8, (uint32_t)w);
  put_u32(dst + 12, (uint32_t)h);
  put_u32(dst + 16, (uint32_t)nchunks);
  put_u32(dst + 20, 0);
  put_u64(dst + 24, (uint64_t)off);
  return payload0 + off;
}

/* Exact inverse with validation (OR_E_CORRUPT on any inconsistency). */
int or_rle64_decode(const uint8_t *src, int64_t src_bytes, uint32_t *dst, int64_t pitch, int w, int h) {
  if (!src || !dst || w <= 0 || h <= 0 || pitch < w) return OR_E_INVALID;
  if (src_bytes < 32) return OR_E_CORRUPT;
  if (get_u32(src) != RLE_MAGIC || src[4] != RLE_VERSION || src[5] > 1 || src[6] != 2 || src[7] != 7)
    return OR_E_CORRUPT;
  if ((int64_t)get_u32(src + 8) != w || (int64_t)get_u32(src + 12) != h) return OR_E_CORRUPT;
  const int C = 128;
  int S = (w + C - 1) / C;
  int64_t nchunks = (int64_t)S * h;
  if ((int64_t)get_u32(src + 16) != nchunks || get_u32(src + 20) != 0) return OR_E_CORRUPT;
  uint64_t pbytes = get_u64(src + 24);
  int64_t payload0 = 32 + 8 * nchunks;
  if (src_bytes < payload0 || (uint64_t)(src_bytes - payload0) < pbytes) return OR_E_CORRUPT;
  uint64_t expect = 0;
  for (int y = 0; y < h; ++y) {
    for (int k = 0; k < S; ++k) {
      int x0 = k * C;
      int L = (w - x0 < C) ? (w - x0) : C;
      int U = (L + 1) / 2;
      int64_t chunk_id = (int64_t)y * S + k;
      uint64_t off = get_u32(src + 32 + 8 * chunk_id);
      uint64_t size = get_u32(src + 32 + 8 * chunk_id + 4);
      if (off != expect || size < 2 || off + size > pbytes) return OR_E_CORRUPT;
      const uint8_t *r = src + payload0 + off;
      int ntok = r[0];
      if (ntok < 1 || (uint64_t)(1 + ntok) > size) return OR_E_CORRUPT;
      uint64_t p = 1 + (uint64_t)ntok;
      int u = 0;
      uint32_t *row = dst + (int64_t)y * pitch + x0;
      for (int t = 0; t < ntok; ++t) {
        int c = r[1 + t];
        int len = (c & 0x7F) + 1;
        if (u + len > U) return OR_E_CORRUPT;
        for (int q = 0; q < len; ++q) {
          uint64_t pp = p + ((c & 0x80) ? 0 : 8 * (uint64_t)q);
          if (pp + 8 > size) return OR_E_CORRUPT;
          uint64_t v = 0;
          for (int b = 0; b < 8; ++b) v |= (uint64_t)r[pp + b] << (8 * b);
          int px = 2 * (u + q);
          row[px] = (uint32_t)v;
          if (px + 1 < L) row[px + 1] = (uint32_t)(v >> 32);
          else if ((v >> 32) != 0) return OR_E_CORRUPT; /* canonical padding */
        }
        p += (c & 0x80) ? 8 : 8 * (uint64_t)len;
        u += len;
      }
      if (u != U || p != size) return OR_E_CORRUPT;
      expect = off + size;
    }
  }
  if (expect != pbytes) return OR_E_CORRUPT;
  return OR_OK;
}
