// composite.cu -- per-pixel sort-last compositing kernels for sm_100a.
//
//  compositor_depth          depth-sorted compositing (R-C1, R-C2)
//  compositor_blend_ordered  ordered back-to-front "over" (R-C3, R-C4)
//
// Both are HBM-bound streaming reductions over N source frames:
// depth moves (8N + 8) B per output pixel (8N + 4 colour-only), blend (4N + 4).
// Design: one thread owns 4 consecutive pixels of a row and
// issues one 128-bit streaming load per source buffer (L1 no-allocate, L2
// evict-first: every input byte is read exactly once), keeps the running
// result in registers and writes one 128-bit streaming store per output buffer.
// No shared memory, no tensor cores: there is no reuse and no contraction.
#include "eqc_common.cuh"

// ROI kernels: one wave of resident CTAs (the rectangle staging is paid once
// per CTA) unless EQC_ROI_GRID16 asks for the 16-CTAs/SM grid
#ifdef EQC_ROI_GRID16
#define EQC_ROI_GRID(k) (16 * eqc_num_sms())
#else
#define EQC_ROI_GRID(k) ([] { static const int c = eqc_resident_ctas(k, 256); return c; }())
#endif
#ifndef EQC_ROI_MINB
#define EQC_ROI_MINB 3
#endif

namespace {

struct DepthParams {
  const uint32_t *color[EQC_MAX_SOURCES];
  const uint32_t *depth[EQC_MAX_SOURCES];
  uint32_t *out_color;
  uint32_t *out_depth;
  int4 *cta_box;  // BBOX: per-CTA bounding box {x0, y0, x1, y1} (inclusive) of the rendered output
  int64_t pitch, out_pitch;
  int n, w, h, groups_per_row;
};

// Running bounding box of rendered pixels (output depth != background),
// fused into the composite: the ROI of the composited frame
// at no extra HBM pass.  `m` bit j: pixel x + j is rendered.
struct BBox {
  int x0 = 0x7FFFFFFF, y0 = 0x7FFFFFFF, x1 = -1, y1 = -1;
  __device__ __forceinline__ void add(int x, int y, uint32_t m) {
    if (m) {
      x0 = min(x0, x + __ffs(m) - 1);
      x1 = max(x1, x + 31 - __clz(m));
      y0 = min(y0, y);
      y1 = max(y1, y);
    }
  }
  // CTA-wide reduction; thread 0 stores the CTA's box
  __device__ __forceinline__ void store_cta(int4 *out) {
    __shared__ int4 s_b[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int a = __reduce_min_sync(EQC_FULL, x0), b = __reduce_min_sync(EQC_FULL, y0);
    int c = __reduce_max_sync(EQC_FULL, x1), d = __reduce_max_sync(EQC_FULL, y1);
    if (lane == 0) s_b[warp] = make_int4(a, b, c, d);
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      const int4 v = lane < nw ? s_b[lane] : make_int4(0x7FFFFFFF, 0x7FFFFFFF, -1, -1);
      a = __reduce_min_sync(EQC_FULL, v.x);
      b = __reduce_min_sync(EQC_FULL, v.y);
      c = __reduce_max_sync(EQC_FULL, v.z);
      d = __reduce_max_sync(EQC_FULL, v.w);
      if (lane == 0) out[blockIdx.x] = make_int4(a, b, c, d);
    }
  }
};

__device__ __forceinline__ uint32_t rendered4(uint4 d) {
  return (d.x != 0xFFFFFFFFu) | ((d.y != 0xFFFFFFFFu) << 1) | ((d.z != 0xFFFFFFFFu) << 2) |
         ((d.w != 0xFFFFFFFFu) << 3);
}

// One running (depth, colour) minimum step per lane: strictly smaller depth
// replaces, so for equal depths the earlier (lower-index) source is kept.
__device__ __forceinline__ void zmin(uint32_t &bd, uint32_t &bc, uint32_t d, uint32_t c) {
  bool t = d < bd;
  bd = t ? d : bd;
  bc = t ? c : bc;
}

template <bool VEC, bool BBOX = false>
__global__ void __launch_bounds__(256) depth_composite_kernel(const __grid_constant__ DepthParams p) {
  BBox box;
  // 32-bit group index (the host guarantees groups_per_row * h < 2^31)
  const uint32_t total = (uint32_t)p.groups_per_row * (uint32_t)p.h;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int y = (int)(g / (uint32_t)p.groups_per_row);
    const int x = (int)(g - (uint32_t)y * (uint32_t)p.groups_per_row) * 4;
    const int64_t off = (int64_t)y * p.pitch + x;
    const int64_t ooff = (int64_t)y * p.out_pitch + x;
    if (VEC && x + 4 <= p.w) {
      uint4 bd = ld_stream_u4(p.depth[0] + off);
      uint4 bc = ld_stream_u4(p.color[0] + off);
      int i = 1;
      // batches of 4 sources: 8 independent 128-bit loads in flight per thread
      for (; i + 4 <= p.n; i += 4) {
        uint4 d[4], c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          d[j] = ld_stream_u4(p.depth[i + j] + off);
          c[j] = ld_stream_u4(p.color[i + j] + off);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          zmin(bd.x, bc.x, d[j].x, c[j].x);
          zmin(bd.y, bc.y, d[j].y, c[j].y);
          zmin(bd.z, bc.z, d[j].z, c[j].z);
          zmin(bd.w, bc.w, d[j].w, c[j].w);
        }
      }
      for (; i < p.n; ++i) {
        uint4 d = ld_stream_u4(p.depth[i] + off);
        uint4 c = ld_stream_u4(p.color[i] + off);
        zmin(bd.x, bc.x, d.x, c.x);
        zmin(bd.y, bc.y, d.y, c.y);
        zmin(bd.z, bc.z, d.z, c.z);
        zmin(bd.w, bc.w, d.w, c.w);
      }
      st_stream_u4(p.out_color + ooff, bc);
      if (p.out_depth) st_stream_u4(p.out_depth + ooff, bd);
      if (BBOX) box.add(x, y, rendered4(bd));
    } else {
      const int cnt = min(4, p.w - x);
      for (int k = 0; k < cnt; ++k) {
        uint32_t bd = p.depth[0][off + k], bc = p.color[0][off + k];
        for (int i = 1; i < p.n; ++i) zmin(bd, bc, p.depth[i][off + k], p.color[i][off + k]);
        p.out_color[ooff + k] = bc;
        if (p.out_depth) p.out_depth[ooff + k] = bd;
        if (BBOX) box.add(x + k, y, bd != 0xFFFFFFFFu);
      }
    }
  }
  if (BBOX) box.store_cta(p.cta_box);
}

// Reduce the per-CTA boxes into {x, y, w, h} ({0, 0, 0, 0} if nothing is rendered).
__global__ void bbox_finalize_kernel(const int4 *cta, int ncta, int32_t *out) {
  BBox b;
  for (int i = threadIdx.x; i < ncta; i += blockDim.x) {
    const int4 v = cta[i];
    b.x0 = min(b.x0, v.x);
    b.y0 = min(b.y0, v.y);
    b.x1 = max(b.x1, v.z);
    b.y1 = max(b.y1, v.w);
  }
  __shared__ int4 s_b[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int a = __reduce_min_sync(EQC_FULL, b.x0), c = __reduce_min_sync(EQC_FULL, b.y0);
  int d = __reduce_max_sync(EQC_FULL, b.x1), e = __reduce_max_sync(EQC_FULL, b.y1);
  if (lane == 0) s_b[warp] = make_int4(a, c, d, e);
  __syncthreads();
  if (threadIdx.x == 0) {
    int4 r = s_b[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      r.x = min(r.x, s_b[w].x);
      r.y = min(r.y, s_b[w].y);
      r.z = max(r.z, s_b[w].z);
      r.w = max(r.w, s_b[w].w);
    }
    *reinterpret_cast<int4 *>(out) = r.z < 0 ? make_int4(0, 0, 0, 0) : make_int4(r.x, r.y, r.z - r.x + 1, r.w - r.y + 1);
  }
}

struct BlendParams {
  const uint32_t *color[EQC_MAX_SOURCES];  // already in draw order, back first
  uint32_t *out_color;
  int64_t pitch, out_pitch;
  int n, w, h, groups_per_row;
  float bg[4];
};

// Exact float of byte k of v: build the bit pattern 0x4B0000bb (= 2^23 + bb)
// with one byte permute, then remove the 2^23 bias (both steps exact).
template <int K>
__device__ __forceinline__ float byte_f(uint32_t v) {
  return __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7440 + K)) - 8388608.0f;
}

struct Acc4 {
  float r, g, b, a;
};

// x = s + x * (1 - a_s/255) per channel, all in units of 1/255 (fp32 FMAs).
// Byte -> float conversions are split between the integer-convert pipe
// (I2F.U8 with byte select, R and G) and the ALU/FMA pipes (PRMT + FADD,
// B and A) so neither pipe limits the issue rate; the alpha float is shared
// by the transparency factor and the alpha channel.
__device__ __forceinline__ void over(Acc4 &x, uint32_t s) {
  const float a = byte_f<3>(s);
  const float f = fmaf(a, -1.0f / 255.0f, 1.0f);  // 1 - a/255 (a = 255 -> |f| < 1e-8)
  x.r = fmaf(x.r, f, __uint2float_rn(s & 0xFFu));
  x.g = fmaf(x.g, f, __uint2float_rn((s >> 8) & 0xFFu));
  x.b = fmaf(x.b, f, byte_f<2>(s));
  x.a = fmaf(x.a, f, a);
}

__device__ __forceinline__ uint32_t pack_round(const Acc4 &x) {
  // one rounding to RGBA8 (round-to-nearest), clamped to [0, 255]
  uint32_t r = min(__float2uint_rn(fmaxf(x.r, 0.0f)), 255u);
  uint32_t g = min(__float2uint_rn(fmaxf(x.g, 0.0f)), 255u);
  uint32_t b = min(__float2uint_rn(fmaxf(x.b, 0.0f)), 255u);
  uint32_t a = min(__float2uint_rn(fmaxf(x.a, 0.0f)), 255u);
  return r | (g << 8) | (b << 16) | (a << 24);
}

template <bool VEC>
__global__ void __launch_bounds__(256, 4) blend_ordered_kernel(const __grid_constant__ BlendParams p) {
  // 32-bit group index (the host guarantees groups_per_row * h < 2^31)
  const uint32_t total = (uint32_t)p.groups_per_row * (uint32_t)p.h;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int y = (int)(g / (uint32_t)p.groups_per_row);
    const int x = (int)(g - (uint32_t)y * (uint32_t)p.groups_per_row) * 4;
    const int64_t off = (int64_t)y * p.pitch + x;
    const int64_t ooff = (int64_t)y * p.out_pitch + x;
    if (VEC && x + 4 <= p.w) {
      Acc4 acc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = Acc4{p.bg[0], p.bg[1], p.bg[2], p.bg[3]};
      int k = 0;
      for (; k + 4 <= p.n; k += 4) {
        uint4 s[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) s[j] = ld_stream_u4(p.color[k + j] + off);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          over(acc[0], s[j].x);
          over(acc[1], s[j].y);
          over(acc[2], s[j].z);
          over(acc[3], s[j].w);
        }
      }
      for (; k < p.n; ++k) {
        uint4 s = ld_stream_u4(p.color[k] + off);
        over(acc[0], s.x);
        over(acc[1], s.y);
        over(acc[2], s.z);
        over(acc[3], s.w);
      }
      uint4 o = make_uint4(pack_round(acc[0]), pack_round(acc[1]), pack_round(acc[2]), pack_round(acc[3]));
      st_stream_u4(p.out_color + ooff, o);
    } else {
      const int cnt = min(4, p.w - x);
      for (int q = 0; q < cnt; ++q) {
        Acc4 acc{p.bg[0], p.bg[1], p.bg[2], p.bg[3]};
        for (int k = 0; k < p.n; ++k) over(acc, p.color[k][off + q]);
        p.out_color[ooff + q] = pack_round(acc);
      }
    }
  }
}

// ---- region of interest --------------------------------
// Source i holds pixel data only inside its rectangle d_roi[i] = {x, y, w, h}
// (full-frame coordinates; the buffer is indexed like a full frame and is
// dereferenced only inside the rectangle); elsewhere it is background
// (depth 0xFFFFFFFF, colour 0; for blending: transparent) -- P:2268-2271.
// Rectangles are read on the device (e.g. straight from image_roi), clipped
// to the frame (R-C19), and staged in shared memory as {x0, y0, x1, y1}.
struct Rect {
  int x0, y0, x1, y1;
};

__device__ __forceinline__ Rect load_rect(const int32_t *r, int w, int h) {
  const int4 v = *reinterpret_cast<const int4 *>(r);
  Rect q;
  q.x0 = max(v.x, 0);
  q.y0 = max(v.y, 0);
  q.x1 = (v.z > 0 && v.x < w) ? (int)min((int64_t)v.x + v.z, (int64_t)w) : 0;
  q.y1 = (v.w > 0 && v.y < h) ? (int)min((int64_t)v.y + v.w, (int64_t)h) : 0;
  if (q.x1 <= q.x0 || q.y1 <= q.y0) q = Rect{0, 0, 0, 0};
  return q;
}

// Union over the warp's active lanes of the sources (or draw positions)
// whose rectangle covers one of the lanes' 4-pixel groups, as two 32-bit
// masks.  When the warp's groups lie in one row (the common case: a row of
// 4K is 30 full warps) lane i tests rectangle i against the warp's span --
// one test per source instead of one per source per lane; otherwise every
// lane tests every rectangle and the masks are OR-reduced.
__device__ __forceinline__ void warp_cover_union(const Rect *rs, int n, int y, int x, int cnt, bool live,
                                                 uint32_t wm[2]) {
  const unsigned act = __activemask();
  const unsigned lv = __ballot_sync(act, live);  // lanes whose group is to be composited
  wm[0] = wm[1] = 0;
  if (!lv) return;
  const int lane = threadIdx.x & 31;
  const int l0 = __ffs(lv) - 1, l1 = 31 - __clz(lv);
  const int ya = __shfl_sync(act, y, l0), yb = __shfl_sync(act, y, l1);
  const int xa = __shfl_sync(act, x, l0), xb = __shfl_sync(act, x + cnt, l1);
  // fast path: every live lane lies on row ya inside the span [xa, xb) of the
  // first and last live lanes; the union tested against the span is a
  // superset of the lanes' union (extra sources are then masked per lane)
  const bool one = ya == yb && __all_sync(act, !live || (y == ya && x >= xa && x + cnt <= xb));
  if (one) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      bool c = false;
      const int i = 32 * h + lane;
      if (i < n) {
        const Rect r = rs[i];
        c = (unsigned)(ya - r.y0) < (unsigned)(r.y1 - r.y0) && xa < r.x1 && xb > r.x0;
      }
      wm[h] = __ballot_sync(act, c);
    }
  } else {
    uint32_t m[2] = {0, 0};
    if (live) {
      for (int i = 0; i < n; ++i) {
        const Rect r = rs[i];
        const bool c = (unsigned)(y - r.y0) < (unsigned)(r.y1 - r.y0) && x < r.x1 && x + cnt > r.x0;
        if (i < 32) m[0] |= (uint32_t)c << i; else m[1] |= (uint32_t)c << (i - 32);
      }
    }
    wm[0] = __reduce_or_sync(act, m[0]);
    wm[1] = __reduce_or_sync(act, m[1]);
  }
}

struct DepthRoiParams {
  const uint32_t *color[EQC_MAX_SOURCES];
  const uint32_t *depth[EQC_MAX_SOURCES];
  const int32_t *roi[EQC_MAX_SOURCES];  // device {x, y, w, h} of each source (may live on a peer GPU)
  const int32_t *out_roi;               // nullable device {x, y, w, h}: only groups touching it are written
  int roi_dy;                           // rectangles are in frame rows; this launch covers rows roi_dy..
  uint32_t *out_color;
  uint32_t *out_depth;
  int64_t pitch, out_pitch;
  int n, w, h, groups_per_row;
  int vec;
};

// One thread per 4 consecutive pixels of a row, as depth_composite_kernel;
// a source is read only where its rectangle covers the pixels.  Source 0 is
// taken unconditionally where it is inside (argmin of (depth, index)).
__device__ __forceinline__ Rect load_rect_dy(const int32_t *r, int dy, int w, int h) {
  const int4 v = *reinterpret_cast<const int4 *>(r);
  const int32_t q[4] = {v.x, v.y - dy, v.z, v.w};  // same clipping as load_rect, band-relative rows
  return load_rect(q, w, h);
}

__global__ void __launch_bounds__(256, EQC_ROI_MINB) depth_composite_roi_kernel(const __grid_constant__ DepthRoiParams p) {
  __shared__ Rect s_r[EQC_MAX_SOURCES];
  __shared__ Rect s_out;
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) s_r[i] = load_rect_dy(p.roi[i], p.roi_dy, p.w, p.h);
  if (threadIdx.x == 0) s_out = p.out_roi ? load_rect_dy(p.out_roi, p.roi_dy, p.w, p.h) : Rect{0, 0, p.w, p.h};
  __syncthreads();
  const Rect orr = s_out;
  // 32-bit group index (the host guarantees groups_per_row * h < 2^31)
  const uint32_t total = (uint32_t)p.groups_per_row * (uint32_t)p.h;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int y = (int)(g / (uint32_t)p.groups_per_row);
    const int x = (int)(g - (uint32_t)y * (uint32_t)p.groups_per_row) * 4;
    const int64_t off = (int64_t)y * p.pitch + x;
    const int cnt = min(4, p.w - x);
    // outside the output rectangle nothing is read or written (the lane still
    // takes part in the warp's collectives)
    const bool live = (unsigned)(y - orr.y0) < (unsigned)(orr.y1 - orr.y0) && x < orr.x1 && x + cnt > orr.x0;
    uint32_t bd[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, bc[4] = {0, 0, 0, 0};
    uint32_t wmask[2];
    warp_cover_union(s_r, p.n, y, x, cnt, live, wmask);  // warp-uniform source set
    for (int h = 0; h < 2; ++h) {
      uint32_t wm = wmask[h];
      while (wm) {
        // up to 4 sources of the union per batch (ascending index), loads
        // predicated per lane on full coverage of its 4 pixels
        int src[4];
        uint32_t fb = 0, cb = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          src[b] = -1;
          if (wm) {
            src[b] = 32 * h + __ffs(wm) - 1;
            wm &= wm - 1;
            const Rect r = s_r[src[b]];
            const bool c = live && (unsigned)(y - r.y0) < (unsigned)(r.y1 - r.y0) && x < r.x1 && x + cnt > r.x0;
            const bool f = c && p.vec && x >= r.x0 && x + 4 <= r.x1;
            cb |= (uint32_t)c << b;
            fb |= (uint32_t)f << b;
          }
        }
        uint4 dv[4], cv[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = max(src[b], 0);
          dv[b] = ld_stream_u4_if(p.depth[i] + off, (fb >> b) & 1u);
          cv[b] = ld_stream_u4_if(p.color[i] + off, (fb >> b) & 1u);
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = src[b];
          if (i < 0) break;
          if ((fb >> b) & 1u) {
            const uint32_t d[4] = {dv[b].x, dv[b].y, dv[b].z, dv[b].w};
            const uint32_t c[4] = {cv[b].x, cv[b].y, cv[b].z, cv[b].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const bool t = i == 0 || d[j] < bd[j];  // ties keep the lower index
              bd[j] = t ? d[j] : bd[j];
              bc[j] = t ? c[j] : bc[j];
            }
          } else if ((cb >> b) & 1u) {  // rectangle edge: per pixel
            const Rect r = s_r[i];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (j < cnt && x + j >= r.x0 && x + j < r.x1) {
                const uint32_t dj = ld_stream_u32(p.depth[i] + off + j), cj = ld_stream_u32(p.color[i] + off + j);
                const bool t = i == 0 || dj < bd[j];
                bd[j] = t ? dj : bd[j];
                bc[j] = t ? cj : bc[j];
              }
            }
          }
        }
      }
    }
    if (!live) continue;
    const int64_t ooff = (int64_t)y * p.out_pitch + x;
    if (p.vec && cnt == 4) {
      st_stream_u4(p.out_color + ooff, make_uint4(bc[0], bc[1], bc[2], bc[3]));
      if (p.out_depth) st_stream_u4(p.out_depth + ooff, make_uint4(bd[0], bd[1], bd[2], bd[3]));
    } else {
      for (int j = 0; j < cnt; ++j) {
        p.out_color[ooff + j] = bc[j];
        if (p.out_depth) p.out_depth[ooff + j] = bd[j];
      }
    }
  }
}

struct BlendRoiParams {
  const uint32_t *color[EQC_MAX_SOURCES];  // already in draw order, back first
  const int32_t *roi;                       // device, indexed by SOURCE
  int src_of[EQC_MAX_SOURCES];              // draw position -> source index
  uint32_t *out_color;
  int64_t pitch, out_pitch;
  int n, w, h, groups_per_row;
  int vec;
  float bg[4];
};

// Ordered blend over ROI-restricted layers: outside its rectangle a layer is
// transparent and is skipped (over() with s = 0 is the identity).
__global__ void __launch_bounds__(256, EQC_ROI_MINB) blend_ordered_roi_kernel(const __grid_constant__ BlendRoiParams p) {
  __shared__ Rect s_r[EQC_MAX_SOURCES];
  for (int k = threadIdx.x; k < p.n; k += blockDim.x) s_r[k] = load_rect(p.roi + 4 * p.src_of[k], p.w, p.h);
  __syncthreads();
  // 32-bit group index (the host guarantees groups_per_row * h < 2^31)
  const uint32_t total = (uint32_t)p.groups_per_row * (uint32_t)p.h;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int y = (int)(g / (uint32_t)p.groups_per_row);
    const int x = (int)(g - (uint32_t)y * (uint32_t)p.groups_per_row) * 4;
    const int64_t off = (int64_t)y * p.pitch + x;
    const int cnt = min(4, p.w - x);
    Acc4 acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = Acc4{p.bg[0], p.bg[1], p.bg[2], p.bg[3]};
    uint32_t wmask[2];
    warp_cover_union(s_r, p.n, y, x, cnt, true, wmask);  // draw positions, warp-uniform
    for (int h = 0; h < 2; ++h) {
      uint32_t wm = wmask[h];  // ascending k = draw order
      while (wm) {
        int kk[4];
        uint32_t fb = 0, cb = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          kk[b] = -1;
          if (wm) {
            kk[b] = 32 * h + __ffs(wm) - 1;
            wm &= wm - 1;
            const Rect r = s_r[kk[b]];
            const bool c = (unsigned)(y - r.y0) < (unsigned)(r.y1 - r.y0) && x < r.x1 && x + cnt > r.x0;
            const bool f = c && p.vec && x >= r.x0 && x + 4 <= r.x1;
            cb |= (uint32_t)c << b;
            fb |= (uint32_t)f << b;
          }
        }
        uint4 sv[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) sv[b] = ld_stream_u4_if(p.color[max(kk[b], 0)] + off, (fb >> b) & 1u);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int k = kk[b];
          if (k < 0) break;
          if ((fb >> b) & 1u) {
            over(acc[0], sv[b].x);
            over(acc[1], sv[b].y);
            over(acc[2], sv[b].z);
            over(acc[3], sv[b].w);
          } else if ((cb >> b) & 1u) {
            const Rect r = s_r[k];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < cnt && x + j >= r.x0 && x + j < r.x1) over(acc[j], ld_stream_u32(p.color[k] + off + j));
          }
        }
      }
    }
    const int64_t ooff = (int64_t)y * p.out_pitch + x;
    if (p.vec && cnt == 4) {
      st_stream_u4(p.out_color + ooff,
                   make_uint4(pack_round(acc[0]), pack_round(acc[1]), pack_round(acc[2]), pack_round(acc[3])));
    } else {
      for (int j = 0; j < cnt; ++j) p.out_color[ooff + j] = pack_round(acc[j]);
    }
  }
}

// ---- blend partials for multi-GPU ordered compositing -----
// A rank's partial image is its layers "over"-composited onto a transparent
// background (premultiplied "over" is associative), carried in
// unorm16 per channel (R-C6: an 8-bit intermediate would add up to 1/2 LSB per
// partial) as two uint32 planes: rg = R16 | G16 << 16, ba = B16 | A16 << 16
// (value16 = round(255-scale value * 257)).  The two planes travel through
// the same band/RLE transport as colour and depth.

__device__ __forceinline__ uint32_t u16_round(float v) {  // v in [0, 65535] (clamped)
  return min(__float2uint_rn(fmaxf(v, 0.0f)), 65535u);
}

struct Part16 {
  float r, g, b, a;  // 0..65535
};

__device__ __forceinline__ Part16 unpack16(uint32_t rg, uint32_t ba) {
  return Part16{(float)(rg & 0xFFFFu), (float)(rg >> 16), (float)(ba & 0xFFFFu), (float)(ba >> 16)};
}

// x = s + x * (1 - a_s / 65535), all in unorm16 units
__device__ __forceinline__ void over16(Part16 &x, const Part16 &s) {
  const float f = fmaf(s.a, -1.0f / 65535.0f, 1.0f);
  x.r = fmaf(x.r, f, s.r);
  x.g = fmaf(x.g, f, s.g);
  x.b = fmaf(x.b, f, s.b);
  x.a = fmaf(x.a, f, s.a);
}

struct BlendPartialParams {
  const uint32_t *color[EQC_MAX_SOURCES];  // RGBA8 layers in draw order (back first)
  uint32_t *out_rg, *out_ba;
  int64_t pitch, out_pitch;
  int n, w, h, groups_per_row;
};

// n RGBA8 layers -> one unorm16 partial (transparent background).  VEC: one
// 128-bit load per layer per thread, batches of 4 layers in flight.
template <bool VEC>
__global__ void __launch_bounds__(256, 4) blend_partial_kernel(const __grid_constant__ BlendPartialParams p) {
  const uint32_t total = (uint32_t)p.groups_per_row * (uint32_t)p.h;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int y = (int)(g / (uint32_t)p.groups_per_row);
    const int x = (int)(g - (uint32_t)y * (uint32_t)p.groups_per_row) * 4;
    const int64_t off = (int64_t)y * p.pitch + x;
    const int cnt = min(4, p.w - x);
    Acc4 acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = Acc4{0.0f, 0.0f, 0.0f, 0.0f};
    if (VEC && cnt == 4) {
      int k = 0;
      for (; k + 4 <= p.n; k += 4) {
        uint4 v[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) v[b] = ld_stream_u4(p.color[k + b] + off);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          over(acc[0], v[b].x);
          over(acc[1], v[b].y);
          over(acc[2], v[b].z);
          over(acc[3], v[b].w);
        }
      }
      for (; k < p.n; ++k) {
        const uint4 v = ld_stream_u4(p.color[k] + off);
        over(acc[0], v.x);
        over(acc[1], v.y);
        over(acc[2], v.z);
        over(acc[3], v.w);
      }
    } else {
      for (int k = 0; k < p.n; ++k) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < cnt) over(acc[j], ld_stream_u32(p.color[k] + off + j));
      }
    }
    const int64_t ooff = (int64_t)y * p.out_pitch + x;
    uint32_t rg[4], ba[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      rg[j] = u16_round(acc[j].r * 257.0f) | (u16_round(acc[j].g * 257.0f) << 16);
      ba[j] = u16_round(acc[j].b * 257.0f) | (u16_round(acc[j].a * 257.0f) << 16);
    }
    if (VEC && cnt == 4) {
      st_stream_u4(p.out_rg + ooff, make_uint4(rg[0], rg[1], rg[2], rg[3]));
      st_stream_u4(p.out_ba + ooff, make_uint4(ba[0], ba[1], ba[2], ba[3]));
    } else {
      for (int j = 0; j < cnt; ++j) {
        p.out_rg[ooff + j] = rg[j];
        p.out_ba[ooff + j] = ba[j];
      }
    }
  }
}

struct BlendPartialsParams {
  const uint32_t *rg[EQC_MAX_SOURCES], *ba[EQC_MAX_SOURCES];  // partials, back first
  uint32_t *out_c;           // FINAL: RGBA8 output
  uint32_t *out_rg, *out_ba; // !FINAL: unorm16 partial output
  int64_t pitch, out_pitch;
  int n, w, h, groups_per_row;
  float bg[4];               // FINAL: background in unorm16 units
};

// n unorm16 partials, back to front -> RGBA8 over `bg` (FINAL, one rounding
// to 8 bits) or -> a unorm16 partial over transparent (binary-swap rounds).
// VEC: two 128-bit loads (rg, ba) per partial, batches of 2 partials.
template <bool FINAL, bool VEC>
__global__ void __launch_bounds__(256, 4) blend_partials_kernel(const __grid_constant__ BlendPartialsParams p) {
  const uint32_t total = (uint32_t)p.groups_per_row * (uint32_t)p.h;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int y = (int)(g / (uint32_t)p.groups_per_row);
    const int x = (int)(g - (uint32_t)y * (uint32_t)p.groups_per_row) * 4;
    const int64_t off = (int64_t)y * p.pitch + x;
    const int cnt = min(4, p.w - x);
    Part16 acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      acc[q] = FINAL ? Part16{p.bg[0], p.bg[1], p.bg[2], p.bg[3]} : Part16{0.0f, 0.0f, 0.0f, 0.0f};
    if (VEC && cnt == 4) {
      int k = 0;
      for (; k + 2 <= p.n; k += 2) {
        uint4 a[2], b[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          a[u] = ld_stream_u4(p.rg[k + u] + off);
          b[u] = ld_stream_u4(p.ba[k + u] + off);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          over16(acc[0], unpack16(a[u].x, b[u].x));
          over16(acc[1], unpack16(a[u].y, b[u].y));
          over16(acc[2], unpack16(a[u].z, b[u].z));
          over16(acc[3], unpack16(a[u].w, b[u].w));
        }
      }
      for (; k < p.n; ++k) {
        const uint4 a = ld_stream_u4(p.rg[k] + off), b = ld_stream_u4(p.ba[k] + off);
        over16(acc[0], unpack16(a.x, b.x));
        over16(acc[1], unpack16(a.y, b.y));
        over16(acc[2], unpack16(a.z, b.z));
        over16(acc[3], unpack16(a.w, b.w));
      }
    } else {
      for (int k = 0; k < p.n; ++k) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < cnt) over16(acc[j], unpack16(ld_stream_u32(p.rg[k] + off + j), ld_stream_u32(p.ba[k] + off + j)));
      }
    }
    const int64_t ooff = (int64_t)y * p.out_pitch + x;
    uint32_t o0[4], o1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (FINAL) {
        const float s = 1.0f / 257.0f;
        const uint32_t r = min(__float2uint_rn(fmaxf(acc[j].r * s, 0.0f)), 255u);
        const uint32_t gg = min(__float2uint_rn(fmaxf(acc[j].g * s, 0.0f)), 255u);
        const uint32_t b = min(__float2uint_rn(fmaxf(acc[j].b * s, 0.0f)), 255u);
        const uint32_t a = min(__float2uint_rn(fmaxf(acc[j].a * s, 0.0f)), 255u);
        o0[j] = r | (gg << 8) | (b << 16) | (a << 24);
      } else {
        o0[j] = u16_round(acc[j].r) | (u16_round(acc[j].g) << 16);
        o1[j] = u16_round(acc[j].b) | (u16_round(acc[j].a) << 16);
      }
    }
    if (VEC && cnt == 4) {
      st_stream_u4((FINAL ? p.out_c : p.out_rg) + ooff, make_uint4(o0[0], o0[1], o0[2], o0[3]));
      if (!FINAL) st_stream_u4(p.out_ba + ooff, make_uint4(o1[0], o1[1], o1[2], o1[3]));
    } else {
      for (int j = 0; j < cnt; ++j) {
        (FINAL ? p.out_c : p.out_rg)[ooff + j] = o0[j];
        if (!FINAL) p.out_ba[ooff + j] = o1[j];
      }
    }
  }
}

// ---- subpixel accumulation + averaging --------
// Channel sums of RGBA8 sources held as two packed planes rg = R16 | G16 << 16,
// ba = B16 | A16 << 16 (a sum of <= 64 bytes is <= 16320, so 32-bit adds of
// packed planes never carry between halves: merging partial sums is a plain
// add).  Final: per channel floor((2 sum + N) / (2 N)) (mean rounded half up,
// R-C22), N = the total number of sources.
struct AvgParams {
  const uint32_t *src[EQC_MAX_SOURCES];  // RGBA8 layers (LOCAL) or rg planes (partials)
  const uint32_t *src_ba[EQC_MAX_SOURCES];
  uint32_t *out_c;            // FINAL
  uint32_t *out_rg, *out_ba;  // !FINAL
  int64_t pitch, out_pitch;
  int n, w, h, groups_per_row;
  uint32_t total;             // FINAL: N
  float inv2n;                // 1 / (2 N)
};

// floor((2 sum + N) / (2 N)) without an integer divide: a = 2 sum + N < 2^24
// is exact in fp32, a / 2N is either an integer k (the product may land a few
// ulp below k) or at least 1/(2N) >= 1/512 below the next integer, so adding
// 1e-4 before truncation is exact (fp32 error at <= 255 is ~1.5e-5).
__device__ __forceinline__ uint32_t avg_round(uint32_t sum, uint32_t n, float inv2n) {
  return (uint32_t)fmaf((float)(2 * sum + n), inv2n, 1e-4f);
}

// LOCAL: inputs are RGBA8 layers; else packed partial-sum planes.
template <bool LOCAL, bool FINAL>
__global__ void __launch_bounds__(256) average_kernel(const __grid_constant__ AvgParams p) {
  const uint32_t total = (uint32_t)p.groups_per_row * (uint32_t)p.h;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int y = (int)(g / (uint32_t)p.groups_per_row);
    const int x = (int)(g - (uint32_t)y * (uint32_t)p.groups_per_row) * 4;
    const int64_t off = (int64_t)y * p.pitch + x;
    const int cnt = min(4, p.w - x);
    uint32_t rg[4] = {0, 0, 0, 0}, ba[4] = {0, 0, 0, 0};
    for (int k = 0; k < p.n; ++k) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= cnt) continue;
        if (LOCAL) {
          const uint32_t v = ld_stream_u32(p.src[k] + off + j);
          rg[j] += __byte_perm(v, 0u, 0x4140);  // [R, 0, G, 0]
          ba[j] += __byte_perm(v, 0u, 0x4342);  // [B, 0, A, 0]
        } else {
          rg[j] += ld_stream_u32(p.src[k] + off + j);
          ba[j] += ld_stream_u32(p.src_ba[k] + off + j);
        }
      }
    }
    const int64_t ooff = (int64_t)y * p.out_pitch + x;
    for (int j = 0; j < cnt; ++j) {
      if (FINAL) {
        p.out_c[ooff + j] = avg_round(rg[j] & 0xFFFFu, p.total, p.inv2n) |
                            (avg_round(rg[j] >> 16, p.total, p.inv2n) << 8) |
                            (avg_round(ba[j] & 0xFFFFu, p.total, p.inv2n) << 16) |
                            (avg_round(ba[j] >> 16, p.total, p.inv2n) << 24);
      } else {
        p.out_rg[ooff + j] = rg[j];
        p.out_ba[ooff + j] = ba[j];
      }
    }
  }
}

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

// Grid of a grid-stride kernel over `items` 4-pixel groups: one group per
// thread, at most `cap` CTAs (16 per SM measured best for the streaming
// kernels: several waves even out the per-thread iteration counts).
}  // namespace
// Internal (compose.cu): CTA cap of the streaming kernels launched by the
// calling host thread (0 = default); set around a pipelined peer pull.
thread_local int eqc_grid_cap = 0;
namespace {
inline int grid_for(int64_t items, int cap = 16 * eqc_num_sms()) {
  if (eqc_grid_cap > 0 && cap > eqc_grid_cap) cap = eqc_grid_cap;
  int64_t blocks = (items + 255) / 256;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace

extern "C" int compositor_depth(int n, const uint32_t *const *color, const uint32_t *const *depth,
                                int w, int h, int64_t pitch, uint32_t *out_color,
                                uint32_t *out_depth, int64_t out_pitch, void *stream) {
  if (n < 1 || n > EQC_MAX_SOURCES || !color || !depth || !out_color) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || out_pitch < w) return EQC_E_INVALID;
  DepthParams p;
  bool vec = (pitch % 4 == 0) && (out_pitch % 4 == 0) && aligned16(out_color) &&
             (!out_depth || aligned16(out_depth));
  for (int i = 0; i < n; ++i) {
    if (!color[i] || !depth[i]) return EQC_E_INVALID;
    p.color[i] = color[i];
    p.depth[i] = depth[i];
    vec = vec && aligned16(color[i]) && aligned16(depth[i]);
  }
  p.out_color = out_color;
  p.out_depth = out_depth;
  p.pitch = pitch;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.groups_per_row = (w + 3) / 4;
  const int64_t groups = (int64_t)p.groups_per_row * h;
  if (groups > 0x7FFFFFFFll) return EQC_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (vec)
    depth_composite_kernel<true><<<grid_for(groups), 256, 0, s>>>(p);
  else
    depth_composite_kernel<false><<<grid_for(groups), 256, 0, s>>>(p);
  return eqc_launch_status();
}

// Internal (compose.cu, EQC_FLAG_ROI): compositor_depth that also writes the
// ROI {x, y, w, h} of its output (pixels with depth != 0xFFFFFFFF) to the
// device int32[4] `out_roi`, reduced from per-CTA boxes in `scratch`
// (>= eqc_depth_bbox_scratch_bytes()).
size_t eqc_depth_bbox_scratch_bytes() { return (size_t)16 * eqc_num_sms() * sizeof(int4); }

int eqc_depth_composite_bbox(int n, const uint32_t *const *color, const uint32_t *const *depth, int w, int h,
                             int64_t pitch, uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch,
                             void *scratch, int32_t *out_roi, cudaStream_t s) {
  if (n < 1 || n > EQC_MAX_SOURCES || !color || !depth || !out_color || !out_depth || !scratch || !out_roi)
    return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || out_pitch < w) return EQC_E_INVALID;
  DepthParams p;
  bool vec = (pitch % 4 == 0) && (out_pitch % 4 == 0) && aligned16(out_color) && aligned16(out_depth);
  for (int i = 0; i < n; ++i) {
    if (!color[i] || !depth[i]) return EQC_E_INVALID;
    p.color[i] = color[i];
    p.depth[i] = depth[i];
    vec = vec && aligned16(color[i]) && aligned16(depth[i]);
  }
  p.out_color = out_color;
  p.out_depth = out_depth;
  p.cta_box = reinterpret_cast<int4 *>(scratch);
  p.pitch = pitch;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.groups_per_row = (w + 3) / 4;
  const int64_t groups = (int64_t)p.groups_per_row * h;
  if (groups > 0x7FFFFFFFll) return EQC_E_INVALID;
  const int grid = grid_for(groups);
  if (vec)
    depth_composite_kernel<true, true><<<grid, 256, 0, s>>>(p);
  else
    depth_composite_kernel<false, true><<<grid, 256, 0, s>>>(p);
  bbox_finalize_kernel<<<1, 256, 0, s>>>(p.cta_box, grid, out_roi);
  return eqc_launch_status();
}

// Internal (compose.cu, EQC_OP_BLEND): n RGBA8 layers -> unorm16 partial planes.
int eqc_blend_to_partial(int n, const uint32_t *const *color, int w, int h, int64_t pitch, uint32_t *out_rg,
                         uint32_t *out_ba, int64_t out_pitch, cudaStream_t s) {
  if (n < 1 || n > EQC_MAX_SOURCES || !color || !out_rg || !out_ba) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || out_pitch < w) return EQC_E_INVALID;
  BlendPartialParams p;
  bool vec = (pitch % 4 == 0) && (out_pitch % 4 == 0) && aligned16(out_rg) && aligned16(out_ba);
  for (int k = 0; k < n; ++k) {
    if (!color[k]) return EQC_E_INVALID;
    p.color[k] = color[k];
    vec = vec && aligned16(color[k]);
  }
  p.out_rg = out_rg;
  p.out_ba = out_ba;
  p.pitch = pitch;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.groups_per_row = (w + 3) / 4;
  const int64_t groups = (int64_t)p.groups_per_row * h;
  if (groups > 0x7FFFFFFFll) return EQC_E_INVALID;
  if (vec)
    blend_partial_kernel<true><<<grid_for(groups), 256, 0, s>>>(p);
  else
    blend_partial_kernel<false><<<grid_for(groups), 256, 0, s>>>(p);
  return eqc_launch_status();
}

// Internal: n unorm16 partials (back first) -> RGBA8 over `background`
// (out_c != NULL) or -> one unorm16 partial (out_rg/out_ba).
int eqc_blend_partials(int n, const uint32_t *const *rg, const uint32_t *const *ba, int w, int h, int64_t pitch,
                       uint32_t background, uint32_t *out_c, uint32_t *out_rg, uint32_t *out_ba, int64_t out_pitch,
                       cudaStream_t s) {
  if (n < 1 || n > EQC_MAX_SOURCES || !rg || !ba || (!out_c && (!out_rg || !out_ba))) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || out_pitch < w) return EQC_E_INVALID;
  BlendPartialsParams p;
  bool vec = (pitch % 4 == 0) && (out_pitch % 4 == 0) &&
             (out_c ? aligned16(out_c) : (aligned16(out_rg) && aligned16(out_ba)));
  for (int k = 0; k < n; ++k) {
    if (!rg[k] || !ba[k]) return EQC_E_INVALID;
    p.rg[k] = rg[k];
    p.ba[k] = ba[k];
    vec = vec && aligned16(rg[k]) && aligned16(ba[k]);
  }
  p.out_c = out_c;
  p.out_rg = out_rg;
  p.out_ba = out_ba;
  p.pitch = pitch;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.groups_per_row = (w + 3) / 4;
  for (int c = 0; c < 4; ++c) p.bg[c] = (float)((background >> (8 * c)) & 0xFFu) * 257.0f;
  const int64_t groups = (int64_t)p.groups_per_row * h;
  if (groups > 0x7FFFFFFFll) return EQC_E_INVALID;
  if (out_c) {
    if (vec)
      blend_partials_kernel<true, true><<<grid_for(groups), 256, 0, s>>>(p);
    else
      blend_partials_kernel<true, false><<<grid_for(groups), 256, 0, s>>>(p);
  } else {
    if (vec)
      blend_partials_kernel<false, true><<<grid_for(groups), 256, 0, s>>>(p);
    else
      blend_partials_kernel<false, false><<<grid_for(groups), 256, 0, s>>>(p);
  }
  return eqc_launch_status();
}

// Internal (compose.cu, EQC_OP_AVERAGE) and compositor_average: `local`:
// src = n RGBA8 layers, else n partial-sum plane pairs (src, src_ba).  FINAL
// (out_c != NULL): mean over `total` sources, else partial-sum planes out.
int eqc_average(bool local, int n, const uint32_t *const *src, const uint32_t *const *src_ba, int w, int h,
                int64_t pitch, int total, uint32_t *out_c, uint32_t *out_rg, uint32_t *out_ba, int64_t out_pitch,
                cudaStream_t s) {
  if (n < 1 || n > EQC_MAX_SOURCES || !src || (!local && !src_ba) || (!out_c && (!out_rg || !out_ba)))
    return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || out_pitch < w || total < 1 || total > 256) return EQC_E_INVALID;
  AvgParams p;
  for (int k = 0; k < n; ++k) {
    if (!src[k] || (!local && !src_ba[k])) return EQC_E_INVALID;
    p.src[k] = src[k];
    p.src_ba[k] = local ? nullptr : src_ba[k];
  }
  p.out_c = out_c;
  p.out_rg = out_rg;
  p.out_ba = out_ba;
  p.pitch = pitch;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.groups_per_row = (w + 3) / 4;
  p.total = (uint32_t)total;
  p.inv2n = 1.0f / (2.0f * (float)total);
  const int64_t groups = (int64_t)p.groups_per_row * h;
  if (groups > 0x7FFFFFFFll) return EQC_E_INVALID;
  const int grid = grid_for(groups);
  if (local && out_c)
    average_kernel<true, true><<<grid, 256, 0, s>>>(p);
  else if (local)
    average_kernel<true, false><<<grid, 256, 0, s>>>(p);
  else if (out_c)
    average_kernel<false, true><<<grid, 256, 0, s>>>(p);
  else
    average_kernel<false, false><<<grid, 256, 0, s>>>(p);
  return eqc_launch_status();
}

extern "C" int compositor_average(int n, const uint32_t *const *color, int w, int h, int64_t pitch,
                                  uint32_t *out_color, int64_t out_pitch, void *stream) {
  if (!out_color) return EQC_E_INVALID;
  return eqc_average(true, n, color, nullptr, w, h, pitch, n, out_color, nullptr, nullptr, out_pitch,
                     (cudaStream_t)stream);
}

extern "C" int compositor_blend_ordered(int n, const uint32_t *const *color, const int32_t *order,
                                        int w, int h, int64_t pitch, uint32_t background,
                                        uint32_t *out_color, int64_t out_pitch, void *stream) {
  if (n < 1 || n > EQC_MAX_SOURCES || !color || !out_color) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || out_pitch < w) return EQC_E_INVALID;
  BlendParams p;
  bool seen[EQC_MAX_SOURCES] = {false};
  bool vec = (pitch % 4 == 0) && (out_pitch % 4 == 0) && aligned16(out_color);
  for (int k = 0; k < n; ++k) {
    int src = order ? order[k] : k;
    if (src < 0 || src >= n || seen[src]) return EQC_E_INVALID;  // not a permutation
    seen[src] = true;
    if (!color[src]) return EQC_E_INVALID;
    p.color[k] = color[src];
    vec = vec && aligned16(color[src]);
  }
  p.out_color = out_color;
  p.pitch = pitch;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.groups_per_row = (w + 3) / 4;
  for (int c = 0; c < 4; ++c) p.bg[c] = (float)((background >> (8 * c)) & 0xFFu);
  const int64_t groups = (int64_t)p.groups_per_row * h;
  if (groups > 0x7FFFFFFFll) return EQC_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (vec)
    blend_ordered_kernel<true><<<grid_for(groups), 256, 0, s>>>(p);
  else
    blend_ordered_kernel<false><<<grid_for(groups), 256, 0, s>>>(p);
  return eqc_launch_status();
}

// Internal launcher shared by compositor_depth_roi and the ROI direct send
// (compose.cu): per-source ROI pointers (peer memory allowed), rectangles in
// frame rows offset by roi_dy (a band starting at frame row roi_dy), and an
// optional output rectangle outside which nothing is written.
int eqc_depth_roi_launch(int n, const uint32_t *const *color, const uint32_t *const *depth,
                         const int32_t *const *roi, int roi_dy, const int32_t *out_roi, int w, int h,
                         int64_t pitch, uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch,
                         cudaStream_t stream) {
  if (n < 1 || n > EQC_MAX_SOURCES || !color || !depth || !roi || !out_color) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || out_pitch < w) return EQC_E_INVALID;
  if (out_roi && ((uintptr_t)out_roi & 15) != 0) return EQC_E_INVALID;
  DepthRoiParams p;
  bool vec = (pitch % 4 == 0) && (out_pitch % 4 == 0) && aligned16(out_color) &&
             (!out_depth || aligned16(out_depth));
  for (int i = 0; i < n; ++i) {
    if (!color[i] || !depth[i] || !roi[i] || ((uintptr_t)roi[i] & 15) != 0) return EQC_E_INVALID;
    p.color[i] = color[i];
    p.depth[i] = depth[i];
    p.roi[i] = roi[i];
    vec = vec && aligned16(color[i]) && aligned16(depth[i]);
  }
  p.out_roi = out_roi;
  p.roi_dy = roi_dy;
  p.out_color = out_color;
  p.out_depth = out_depth;
  p.pitch = pitch;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.groups_per_row = (w + 3) / 4;
  p.vec = vec ? 1 : 0;
  const int64_t groups = (int64_t)p.groups_per_row * h;
  if (groups > 0x7FFFFFFFll) return EQC_E_INVALID;
  depth_composite_roi_kernel<<<grid_for(groups, EQC_ROI_GRID(depth_composite_roi_kernel)), 256, 0, stream>>>(p);
  return eqc_launch_status();
}

extern "C" int compositor_depth_roi(int n, const uint32_t *const *color, const uint32_t *const *depth,
                                    const int32_t *d_roi, int w, int h, int64_t pitch, uint32_t *out_color,
                                    uint32_t *out_depth, int64_t out_pitch, void *stream) {
  if (n < 1 || n > EQC_MAX_SOURCES || !d_roi || ((uintptr_t)d_roi & 15) != 0) return EQC_E_INVALID;
  const int32_t *roi[EQC_MAX_SOURCES];
  for (int i = 0; i < n; ++i) roi[i] = d_roi + 4 * i;
  return eqc_depth_roi_launch(n, color, depth, roi, 0, nullptr, w, h, pitch, out_color, out_depth, out_pitch,
                              (cudaStream_t)stream);
}

extern "C" int compositor_blend_ordered_roi(int n, const uint32_t *const *color, const int32_t *order,
                                            const int32_t *d_roi, int w, int h, int64_t pitch,
                                            uint32_t background, uint32_t *out_color, int64_t out_pitch,
                                            void *stream) {
  if (n < 1 || n > EQC_MAX_SOURCES || !color || !d_roi || !out_color) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || out_pitch < w) return EQC_E_INVALID;
  if (((uintptr_t)d_roi & 15) != 0) return EQC_E_INVALID;
  BlendRoiParams p;
  bool seen[EQC_MAX_SOURCES] = {false};
  bool vec = (pitch % 4 == 0) && (out_pitch % 4 == 0) && aligned16(out_color);
  for (int k = 0; k < n; ++k) {
    int src = order ? order[k] : k;
    if (src < 0 || src >= n || seen[src]) return EQC_E_INVALID;  // not a permutation
    seen[src] = true;
    if (!color[src]) return EQC_E_INVALID;
    p.color[k] = color[src];
    p.src_of[k] = src;
    vec = vec && aligned16(color[src]);
  }
  p.roi = d_roi;
  p.out_color = out_color;
  p.pitch = pitch;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.groups_per_row = (w + 3) / 4;
  p.vec = vec ? 1 : 0;
  for (int c = 0; c < 4; ++c) p.bg[c] = (float)((background >> (8 * c)) & 0xFFu);
  const int64_t groups = (int64_t)p.groups_per_row * h;
  if (groups > 0x7FFFFFFFll) return EQC_E_INVALID;
  blend_ordered_roi_kernel<<<grid_for(groups, EQC_ROI_GRID(blend_ordered_roi_kernel)), 256, 0, (cudaStream_t)stream>>>(p);
  return eqc_launch_status();
}

// Load every kernel of this file now (CUDA lazy loading would otherwise load
// one at its first launch, which waits for the device: fatal while another
// virtual rank's flag barrier spins, see compose.cu VirtualP2P).
int eqc_preload_composite() {
  cudaFuncAttributes a;
  bool ok = true;
  ok = ok && cudaFuncGetAttributes(&a, depth_composite_kernel<true, false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, depth_composite_kernel<false, false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, depth_composite_kernel<true, true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, depth_composite_kernel<false, true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, bbox_finalize_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_ordered_kernel<true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_ordered_kernel<false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, depth_composite_roi_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_ordered_roi_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_partial_kernel<true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_partial_kernel<false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_partials_kernel<true, true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_partials_kernel<true, false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_partials_kernel<false, true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, blend_partials_kernel<false, false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, average_kernel<true, true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, average_kernel<true, false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, average_kernel<false, true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, average_kernel<false, false>) == cudaSuccess;
  return ok ? EQC_OK : EQC_E_CUDA;
}
