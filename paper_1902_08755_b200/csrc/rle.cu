// rle.cu -- RLE-BP v1 encode / decode kernels and the fused
// decode + depth-assemble kernel (sm_100a).
//
//  image_compress_rle(_batch)   stage (2) "compression" of the asynchronous
//                               compositing pipeline using the
//                               per-component RLE of P:2402-2405 and the
//                               swizzle of P:2407-2425
//  image_decompress_rle(_batch) stage (5), exact inverse + validation
//  compositor_depth_rle         stages (5) + (7) fused: decode in registers,
//                               depth-composite, one HBM write
//
// Encoder: single pass.  Warp w of a CTA codes chunk 8*tile + w into shared
// memory; the chunk sizes are prefix-summed across the CTA and across CTAs by
// a decoupled look-back (CTA order from an atomic ticket), then each warp
// stores its record at its final offset.  The look-back state lives in a
// caller-owned workspace that the kernel leaves reusable: status words carry
// a 16-bit epoch tag and the last CTA to finish bumps the epoch and resets
// the ticket/done counters, so no memset is needed between calls.
#include "rle.cuh"

using namespace eqc_rle;

namespace {

constexpr int kWarps = 8;     // chunks per CTA (one warp each)
constexpr int kMaxBatch = 64;

// workspace layout (uint64): [0] ticket, [1] done, [2] epoch, [3] pad,
// [4 + t] look-back status of tile t.
constexpr int kWsHeader = 4;
constexpr uint64_t kFlagAgg = 1ull << 46;
constexpr uint64_t kFlagIncl = 2ull << 46;
constexpr uint64_t kFlagMask = 3ull << 46;
constexpr uint64_t kValMask = (1ull << 46) - 1;

__device__ __forceinline__ uint64_t status_word(uint64_t epoch, uint64_t flag, uint64_t v) {
  return ((epoch & 0xFFFFull) << 48) | flag | (v & kValMask);
}
__device__ __forceinline__ void publish(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t poll(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct EncImage {
  const uint32_t *src;
  uint8_t *dst;
  int64_t *d_size;
  int kind, flags;
};

struct EncParams {
  EncImage img[kMaxBatch];
  uint64_t *ws;
  int64_t pitch;
  int64_t nchunks;       // per image
  int count, w, h, S;    // S = chunks per row
  int tiles_per_image;
  int vec;               // 128-bit loads allowed
};

// Warp-cooperative decoupled look-back; returns the exclusive prefix of tile
// `lt` of the image whose tile 0 has status index `t0`.  Called by one warp.
__device__ int64_t lookback(uint64_t *status, int64_t t0, int64_t lt, int64_t agg, uint64_t epoch,
                            int lane) {
  const uint64_t tag = (epoch & 0xFFFFull) << 48;
  if (lt == 0) {
    if (lane == 0) publish(status + t0, status_word(epoch, kFlagIncl, (uint64_t)agg));
    return 0;
  }
  if (lane == 0) publish(status + t0 + lt, status_word(epoch, kFlagAgg, (uint64_t)agg));
  int64_t excl = 0;
  int64_t pred = lt - 1;
  while (true) {
    const int64_t idx = pred - lane;
    uint64_t s;
    if (idx >= 0) {
      do {
        s = poll(status + t0 + idx);
      } while ((s & 0xFFFF000000000000ull) != tag || (s & kFlagMask) == 0);
    } else {
      s = kFlagIncl;  // before tile 0: nothing
    }
    const unsigned incl = __ballot_sync(EQC_FULL, (s & kFlagMask) == kFlagIncl);
    int64_t v = (int64_t)(s & kValMask);
    if (incl) {
      const int k = __ffs(incl) - 1;
      if (lane > k) v = 0;
      for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(EQC_FULL, v, d);
      excl += v;
      break;
    }
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(EQC_FULL, v, d);
    excl += v;
    pred -= 32;
  }
  if (lane == 0) publish(status + t0 + lt, status_word(epoch, kFlagIncl, (uint64_t)(excl + agg)));
  return excl;
}

__device__ __forceinline__ void load_chunk(const uint32_t *row, int L, int lane, bool vec, uint32_t px[4]) {
  const int i0 = 4 * lane;
  if (vec && i0 + 4 <= L) {
    const uint4 v = ld_stream_u4(row + i0);
    px[0] = v.x;
    px[1] = v.y;
    px[2] = v.z;
    px[3] = v.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) px[j] = (i0 + j < L) ? ld_stream_u32(row + i0 + j) : 0u;
  }
}

__global__ void __launch_bounds__(kWarps * 32) rle_encode_kernel(const __grid_constant__ EncParams p) {
  __shared__ __align__(16) uint8_t stage[kWarps][kStageBytes];
  __shared__ __align__(16) uint8_t toks[kWarps][kTokBytes];
  __shared__ int wsize[kWarps];
  __shared__ int64_t woff[kWarps];
  __shared__ int64_t s_tile;
  __shared__ uint64_t s_epoch;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t *ws = p.ws;
  if (tid == 0) {
    s_tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(ws), 1ull);
    s_epoch = poll(ws + 2);
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const uint64_t epoch = s_epoch;
  const int m = (int)(tile / p.tiles_per_image);
  const int64_t lt = tile - (int64_t)m * p.tiles_per_image;
  const EncImage im = p.img[m];
  const int64_t c = lt * kWarps + warp;
  const bool active = c < p.nchunks;
  int y = 0, L = 0;
  EncodeOut eo{0, 0};
  if (active) {
    y = (int)(c / p.S);
    const int k = (int)(c - (int64_t)y * p.S);
    const int x0 = k * kC;
    L = min(kC, p.w - x0);
    uint32_t px[4];
    load_chunk(im.src + (int64_t)y * p.pitch + x0, L, lane, p.vec != 0, px);
    if (im.flags & EQC_FLAG_SWIZZLE) {
#pragma unroll
      for (int j = 0; j < 4; ++j) px[j] = swizzle(px[j]);
    }
    eo = encode_chunk(px, L, lane, stage[warp], toks[warp]);
  }
  if (lane == 0) wsize[warp] = eo.size;
  __syncthreads();
  if (warp == 0) {
    const int v = lane < kWarps ? wsize[lane] : 0;
    const int inc = (int)warp_incl_scan_add((uint32_t)v, lane);
    const int agg = __shfl_sync(EQC_FULL, inc, 31);
    const int64_t excl = lookback(ws + kWsHeader, (int64_t)m * p.tiles_per_image, lt, agg, epoch, lane);
    if (lane < kWarps) woff[lane] = excl + inc - v;
    if (lt == p.tiles_per_image - 1 && lane == 0) {
      // last tile of the image: total payload known -> header + size
      const int64_t payload = excl + agg;
      const int64_t payload0 = 32 + 8 * p.nchunks;
      uint32_t *h32 = reinterpret_cast<uint32_t *>(im.dst);
      h32[0] = kMagic;
      h32[1] = (uint32_t)kVersion | ((uint32_t)im.kind << 8) | ((uint32_t)im.flags << 16) |
               ((uint32_t)kLog2C << 24);
      h32[2] = (uint32_t)p.w;
      h32[3] = (uint32_t)p.h;
      h32[4] = (uint32_t)p.nchunks;
      h32[5] = 0u;
      h32[6] = (uint32_t)(uint64_t)payload;
      h32[7] = (uint32_t)((uint64_t)payload >> 32);
      *im.d_size = payload0 + payload;
    }
  }
  __syncthreads();
  if (tid == 0) {
    // this CTA no longer touches the look-back state
    __threadfence();
    const unsigned long long total = (unsigned long long)p.count * p.tiles_per_image;
    const unsigned long long d = atomicAdd(reinterpret_cast<unsigned long long *>(ws + 1), 1ull);
    if (d == total - 1) {
      atomicExch(reinterpret_cast<unsigned long long *>(ws + 0), 0ull);
      atomicExch(reinterpret_cast<unsigned long long *>(ws + 1), 0ull);
      atomicExch(reinterpret_cast<unsigned long long *>(ws + 2), (unsigned long long)(epoch + 1));
    }
  }
  if (active) {
    const int64_t off = woff[warp];
    if (lane == 0) {
      uint32_t *te = reinterpret_cast<uint32_t *>(im.dst + 32 + 8 * c);
      te[0] = (uint32_t)off;
      te[1] = eo.psizes;
    }
    store_record(im.dst + 32 + 8 * p.nchunks + off, stage[warp], eo.size, lane);
  }
}

// ---------------------------------------------------------------------------
// decoder
// ---------------------------------------------------------------------------

struct StreamHdr {
  int ok, kind, flags, log2c;
  int64_t payload0, payload_bytes, nchunks;
  int S;
};

// Validate a stream header against the expected w x h.
__device__ StreamHdr read_header(const uint8_t *src, int64_t src_bytes, int w, int h) {
  StreamHdr hd{};
  hd.ok = 0;
  if (src_bytes < 32) return hd;
  const uint32_t *h32 = reinterpret_cast<const uint32_t *>(src);
  const uint32_t w0 = h32[0], w1 = h32[1];
  const int ver = w1 & 0xFF, kind = (w1 >> 8) & 0xFF, flags = (w1 >> 16) & 0xFF, log2c = w1 >> 24;
  if (w0 != kMagic || ver != kVersion || kind > 1 || (flags & ~1) || (kind == 1 && flags) || log2c < 5 ||
      log2c > 7)
    return hd;
  if ((int64_t)h32[2] != w || (int64_t)h32[3] != h || h32[5] != 0u) return hd;
  const int C = 1 << log2c;
  const int S = (w + C - 1) / C;
  const int64_t nchunks = (int64_t)S * h;
  if ((int64_t)h32[4] != nchunks) return hd;
  const uint64_t pb = (uint64_t)h32[6] | ((uint64_t)h32[7] << 32);
  const int64_t payload0 = 32 + 8 * nchunks;
  if (src_bytes < payload0 || (uint64_t)(src_bytes - payload0) < pb) return hd;
  hd.ok = 1;
  hd.kind = kind;
  hd.flags = flags;
  hd.log2c = log2c;
  hd.payload0 = payload0;
  hd.payload_bytes = (int64_t)pb;
  hd.nchunks = nchunks;
  hd.S = S;
  return hd;
}

// Decode chunk (y, k) of a validated stream into px[0..3] (lane positions
// 4*lane + j of the chunk).  Returns false (warp-uniform) on corruption.
__device__ bool decode_chunk(const uint8_t *src, int64_t src_bytes, const StreamHdr &hd, int w, int y,
                             int k, int lane, uint8_t *stage, uint16_t *info, uint32_t px[4], int &L) {
  const int C = 1 << hd.log2c;
  const int x0 = k * C;
  L = min(C, w - x0);
  const int64_t c = (int64_t)y * hd.S + k;
  const uint2 te = *reinterpret_cast<const uint2 *>(src + 32 + 8 * c);
  const int64_t off = te.x;
  const uint32_t ps = te.y;
  const int s0 = ps & 0xFF, s1 = (ps >> 8) & 0xFF, s2 = (ps >> 16) & 0xFF, s3 = ps >> 24;
  const int total = s0 + s1 + s2 + s3;
  // offsets monotone and contiguous: chunk c starts where chunk c-1 ends,
  // and the last chunk ends at payload_bytes
  int64_t expect = 0;
  if (c > 0) {
    const uint2 tp = *reinterpret_cast<const uint2 *>(src + 32 + 8 * (c - 1));
    expect = (int64_t)tp.x + (tp.y & 0xFF) + ((tp.y >> 8) & 0xFF) + ((tp.y >> 16) & 0xFF) + (tp.y >> 24);
  }
  bool ok = off == expect && off + total <= hd.payload_bytes && s0 <= L + 2 && s1 <= L + 2 &&
            s2 <= L + 2 && s3 <= L + 2;
  if (c == hd.nchunks - 1) ok = ok && off + total == hd.payload_bytes;
  if (!ok) return false;
  // stage the record (aligned 4-byte words; byte loads at the stream end)
  const uint8_t *rec = src + hd.payload0 + off;
  const uintptr_t a0 = (uintptr_t)rec & ~(uintptr_t)3;
  const int sh = (int)((uintptr_t)rec & 3);
  const int nwords = (sh + total + 3) >> 2;
  const uintptr_t lim = (uintptr_t)src + (uintptr_t)src_bytes;
  uint32_t *st32 = reinterpret_cast<uint32_t *>(stage);
  for (int q = lane; q < nwords; q += 32) {
    const uintptr_t a = a0 + 4 * (uintptr_t)q;
    uint32_t v;
    if (a + 4 <= lim) {
      v = __ldg(reinterpret_cast<const uint32_t *>(a));
    } else {
      v = 0;
      for (int b = 0; b < 4; ++b)
        if (a + b < lim) v |= (uint32_t)__ldg(reinterpret_cast<const uint8_t *>(a + b)) << (8 * b);
    }
    st32[q] = v;
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) px[j] = 0;
  const uint8_t *r = stage + sh;
  ok = decode_plane(r, s0, L, lane, 0, px, info);
  ok = ok && decode_plane(r + s0, s1, L, lane, 1, px, info);
  ok = ok && decode_plane(r + s0 + s1, s2, L, lane, 2, px, info);
  ok = ok && decode_plane(r + s0 + s1 + s2, s3, L, lane, 3, px, info);
  __syncwarp();  // stage/info are reused by the next chunk
  if (ok && (hd.flags & EQC_FLAG_SWIZZLE)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) px[j] = unswizzle(px[j]);
  }
  return ok;
}

__device__ __forceinline__ void store_px(uint32_t *row, int L, int lane, bool vec, const uint32_t px[4]) {
  const int i0 = 4 * lane;
  if (vec && i0 + 4 <= L) {
    st_stream_u4(row + i0, make_uint4(px[0], px[1], px[2], px[3]));
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i0 + j < L) row[i0 + j] = px[j];
  }
}

__device__ __forceinline__ void set_corrupt(int32_t *status) {
  if (status) *reinterpret_cast<volatile int32_t *>(status) = EQC_E_CORRUPT;
}

struct DecImage {
  const uint8_t *src;
  uint32_t *dst;
};

struct DecParams {
  DecImage img[kMaxBatch];
  int32_t *status;
  int64_t pitch, src_bytes;
  int count, w, h;
  int segs_per_row;      // 128-pixel segments per row
  int64_t tiles_per_image;
  int vec;
};

// One warp per 128-pixel row segment (1, 2 or 4 chunks for log2c 7, 6, 5).
__global__ void __launch_bounds__(kWarps * 32) rle_decode_kernel(const __grid_constant__ DecParams p) {
  __shared__ __align__(16) uint8_t stage[kWarps][kStageBytes];
  __shared__ __align__(16) uint16_t info[kWarps][kC];
  __shared__ StreamHdr s_hd;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = (int)(blockIdx.x / p.tiles_per_image);
  const int64_t lt = blockIdx.x - (int64_t)m * p.tiles_per_image;
  const DecImage im = p.img[m];
  if (tid == 0) {
    s_hd = read_header(im.src, p.src_bytes, p.w, p.h);
    if (!s_hd.ok) set_corrupt(p.status);
  }
  __syncthreads();
  const StreamHdr hd = s_hd;
  if (!hd.ok) return;
  const int64_t seg = lt * kWarps + warp;
  if (seg >= (int64_t)p.segs_per_row * p.h) return;
  const int y = (int)(seg / p.segs_per_row);
  const int xs = (int)(seg - (int64_t)y * p.segs_per_row) * kC;
  const int C = 1 << hd.log2c;
  for (int k = xs / C; k * C < min(xs + kC, p.w); ++k) {
    uint32_t px[4];
    int L;
    const bool ok = decode_chunk(im.src, p.src_bytes, hd, p.w, y, k, lane, stage[warp], info[warp], px, L);
    if (!ok) {
      if (lane == 0) set_corrupt(p.status);
      continue;
    }
    store_px(im.dst + (int64_t)y * p.pitch + k * C, L, lane, p.vec != 0 && C == kC, px);
  }
}

// ---------------------------------------------------------------------------
// fused decode + depth composite
// ---------------------------------------------------------------------------

struct FusedParams {
  const uint8_t *color[EQC_MAX_SOURCES];
  const uint8_t *depth[EQC_MAX_SOURCES];
  uint32_t *out_color, *out_depth;
  int32_t *status;
  int64_t out_pitch, src_bytes;
  int n, w, h, segs_per_row;
  int vec;
};

__global__ void __launch_bounds__(kWarps * 32) depth_rle_kernel(const __grid_constant__ FusedParams p) {
  __shared__ __align__(16) uint8_t stage[kWarps][kStageBytes];
  __shared__ __align__(16) uint16_t info[kWarps][kC];
  __shared__ StreamHdr s_hd[2 * EQC_MAX_SOURCES];
  __shared__ int s_bad;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int q = tid; q < 2 * p.n; q += blockDim.x) {
    const bool is_depth = q >= p.n;
    const int i = is_depth ? q - p.n : q;
    StreamHdr hd = read_header(is_depth ? p.depth[i] : p.color[i], p.src_bytes, p.w, p.h);
    if (hd.ok && hd.kind != (is_depth ? 1 : 0)) hd.ok = 0;
    if (hd.ok && hd.log2c != kLog2C) hd.ok = 0;  // fused path: 128-pixel chunks only
    s_hd[q] = hd;
    if (!hd.ok) s_bad = 1;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) set_corrupt(p.status);
    return;
  }
  const int64_t seg = (int64_t)blockIdx.x * kWarps + warp;
  if (seg >= (int64_t)p.segs_per_row * p.h) return;
  const int y = (int)(seg / p.segs_per_row);
  const int k = (int)(seg - (int64_t)y * p.segs_per_row);
  uint32_t bc[4], bd[4];
  int L = 0;
  bool ok = true;
  for (int i = 0; i < p.n && ok; ++i) {
    uint32_t c[4], d[4];
    ok = decode_chunk(p.color[i], p.src_bytes, s_hd[i], p.w, y, k, lane, stage[warp], info[warp], c, L);
    ok = ok && decode_chunk(p.depth[i], p.src_bytes, s_hd[p.n + i], p.w, y, k, lane, stage[warp],
                            info[warp], d, L);
    if (i == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bc[j] = c[j];
        bd[j] = d[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool t = d[j] < bd[j];  // strictly nearer replaces: ties keep the lower index
        bd[j] = t ? d[j] : bd[j];
        bc[j] = t ? c[j] : bc[j];
      }
    }
  }
  if (!ok) {
    if (lane == 0) set_corrupt(p.status);
    return;
  }
  const int64_t row = (int64_t)y * p.out_pitch + (int64_t)k * kC;
  store_px(p.out_color + row, L, lane, p.vec != 0, bc);
  if (p.out_depth) store_px(p.out_depth + row, L, lane, p.vec != 0, bd);
}

inline bool aligned(const void *q, uintptr_t a) { return ((uintptr_t)q & (a - 1)) == 0; }

inline int64_t rle_max_size(int w, int h) {
  const int64_t S = (w + kC - 1) / kC;
  return 32 + 16 * S * (int64_t)h + 4 * (int64_t)w * h;
}

inline int64_t tiles_per_image(int w, int h) {
  const int64_t S = (w + kC - 1) / kC;
  return (S * h + kWarps - 1) / kWarps;
}

}  // namespace

extern "C" int64_t image_rle_max_size(int w, int h) {
  if (w <= 0 || h <= 0) return EQC_E_INVALID;
  return rle_max_size(w, h);
}

extern "C" size_t image_rle_workspace_size_batch(int count, int w, int h) {
  if (count <= 0 || w <= 0 || h <= 0) return 0;
  return (size_t)(kWsHeader + (int64_t)count * tiles_per_image(w, h)) * sizeof(uint64_t);
}

extern "C" size_t image_rle_workspace_size(int w, int h) { return image_rle_workspace_size_batch(1, w, h); }

extern "C" int image_compress_rle_batch(int count, const uint32_t *const *src, int w, int h,
                                        int64_t pitch, const int *kind, const int *flags,
                                        uint8_t *const *dst, int64_t dst_capacity, int64_t *d_sizes,
                                        void *workspace, size_t workspace_bytes, void *stream) {
  if (count < 1 || count > kMaxBatch || !src || !kind || !flags || !dst || !d_sizes || !workspace)
    return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w) return EQC_E_INVALID;
  const int64_t maxsz = rle_max_size(w, h);
  if (maxsz - 32 - 8 * ((int64_t)((w + kC - 1) / kC) * h) > (int64_t)0xFFFFFFFFll) return EQC_E_INVALID;
  if (dst_capacity < maxsz) return EQC_E_CAPACITY;
  if (workspace_bytes < image_rle_workspace_size_batch(count, w, h)) return EQC_E_CAPACITY;
  if (!aligned(workspace, 8)) return EQC_E_INVALID;
  EncParams p;
  bool vec = (pitch % 4) == 0;
  for (int i = 0; i < count; ++i) {
    if (!src[i] || !dst[i]) return EQC_E_INVALID;
    if (kind[i] != EQC_KIND_RGBA8 && kind[i] != EQC_KIND_DEPTH32) return EQC_E_INVALID;
    if (flags[i] & ~EQC_FLAG_SWIZZLE) return EQC_E_INVALID;
    if (kind[i] == EQC_KIND_DEPTH32 && flags[i]) return EQC_E_UNSUPPORTED;
    if (!aligned(dst[i], 8) || !aligned(src[i], 4)) return EQC_E_INVALID;
    vec = vec && aligned(src[i], 16);
    p.img[i] = EncImage{src[i], dst[i], d_sizes + i, kind[i], flags[i]};
  }
  p.ws = reinterpret_cast<uint64_t *>(workspace);
  p.pitch = pitch;
  p.S = (w + kC - 1) / kC;
  p.nchunks = (int64_t)p.S * h;
  p.count = count;
  p.w = w;
  p.h = h;
  p.tiles_per_image = (int)tiles_per_image(w, h);
  p.vec = vec ? 1 : 0;
  const int64_t grid = (int64_t)count * p.tiles_per_image;
  if (grid > 0x7FFFFFFFll) return EQC_E_INVALID;
  rle_encode_kernel<<<(unsigned)grid, kWarps * 32, 0, (cudaStream_t)stream>>>(p);
  return eqc_launch_status();
}

extern "C" int image_compress_rle(const uint32_t *src, int w, int h, int64_t pitch, int kind, int flags,
                                  uint8_t *dst, int64_t dst_capacity, int64_t *d_size, void *workspace,
                                  size_t workspace_bytes, void *stream) {
  const uint32_t *s[1] = {src};
  uint8_t *d[1] = {dst};
  return image_compress_rle_batch(1, s, w, h, pitch, &kind, &flags, d, dst_capacity, d_size, workspace,
                                  workspace_bytes, stream);
}

extern "C" int image_decompress_rle_batch(int count, const uint8_t *const *src, int64_t src_bytes,
                                          uint32_t *const *dst, int64_t pitch, int w, int h,
                                          int32_t *d_status, void *stream) {
  if (count < 1 || count > kMaxBatch || !src || !dst || !d_status) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w || src_bytes < 32) return EQC_E_INVALID;
  DecParams p;
  bool vec = (pitch % 4) == 0;
  for (int i = 0; i < count; ++i) {
    if (!src[i] || !dst[i]) return EQC_E_INVALID;
    if (!aligned(src[i], 8) || !aligned(dst[i], 4)) return EQC_E_INVALID;
    vec = vec && aligned(dst[i], 16);
    p.img[i] = DecImage{src[i], dst[i]};
  }
  p.status = d_status;
  p.pitch = pitch;
  p.src_bytes = src_bytes;
  p.count = count;
  p.w = w;
  p.h = h;
  p.segs_per_row = (w + kC - 1) / kC;
  p.tiles_per_image = ((int64_t)p.segs_per_row * h + kWarps - 1) / kWarps;
  p.vec = vec ? 1 : 0;
  const int64_t grid = (int64_t)count * p.tiles_per_image;
  if (grid > 0x7FFFFFFFll) return EQC_E_INVALID;
  rle_decode_kernel<<<(unsigned)grid, kWarps * 32, 0, (cudaStream_t)stream>>>(p);
  return eqc_launch_status();
}

extern "C" int image_decompress_rle(const uint8_t *src, int64_t src_bytes, uint32_t *dst, int64_t pitch,
                                    int w, int h, int32_t *d_status, void *stream) {
  const uint8_t *s[1] = {src};
  uint32_t *d[1] = {dst};
  return image_decompress_rle_batch(1, s, src_bytes, d, pitch, w, h, d_status, stream);
}

extern "C" int compositor_depth_rle(int n, const uint8_t *const *color_rle, const uint8_t *const *depth_rle,
                                    int64_t src_bytes, int w, int h, uint32_t *out_color,
                                    uint32_t *out_depth, int64_t out_pitch, int32_t *d_status,
                                    void *stream) {
  if (n < 1 || n > EQC_MAX_SOURCES || !color_rle || !depth_rle || !out_color || !d_status)
    return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || out_pitch < w || src_bytes < 32) return EQC_E_INVALID;
  FusedParams p;
  for (int i = 0; i < n; ++i) {
    if (!color_rle[i] || !depth_rle[i]) return EQC_E_INVALID;
    if (!aligned(color_rle[i], 8) || !aligned(depth_rle[i], 8)) return EQC_E_INVALID;
    p.color[i] = color_rle[i];
    p.depth[i] = depth_rle[i];
  }
  if (!aligned(out_color, 4) || (out_depth && !aligned(out_depth, 4))) return EQC_E_INVALID;
  p.out_color = out_color;
  p.out_depth = out_depth;
  p.status = d_status;
  p.out_pitch = out_pitch;
  p.src_bytes = src_bytes;
  p.n = n;
  p.w = w;
  p.h = h;
  p.segs_per_row = (w + kC - 1) / kC;
  p.vec = ((out_pitch % 4) == 0 && aligned(out_color, 16) && (!out_depth || aligned(out_depth, 16))) ? 1 : 0;
  const int64_t grid = ((int64_t)p.segs_per_row * h + kWarps - 1) / kWarps;
  if (grid > 0x7FFFFFFFll) return EQC_E_INVALID;
  depth_rle_kernel<<<(unsigned)grid, kWarps * 32, 0, (cudaStream_t)stream>>>(p);
  return eqc_launch_status();
}
