/*
 * eqc.h -- C ABI of libeqc: B200-native sort-last image compositing and RLE
 * frame transport, after S. Eilemann, "Parallel Rendering and Large Data
 * Visualization" (PhD thesis, UZH 2019; arxiv 1902.08755).
 *
 * Citation keys: P:n = line n of the thesis text; R-Cn = reading n of the
 * ambiguity register in DESIGN.md section 3.
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - A FRAME is a colour buffer plus an optional depth buffer (P:1556-1558,
 *    "transfer buffers (colour, depth)").  Colour = RGBA8 packed in a
 *    little-endian uint32 (R = byte 0 ... A = byte 3, R-C7).  Depth = uint32,
 *    smaller is nearer, background 0xFFFFFFFF (R-C1).
 *  - Buffers are row-major [h][pitch] with pitch (in PIXELS, >= w) shared by
 *    all sources of one call.  A tile/band is a sub-rectangle addressed by
 *    pointer offset + pitch (pixel viewport).
 *  - Pixel-buffer pointers are DEVICE pointers owned by the caller
 *    (e.g. torch.Tensor.data_ptr()).  Arrays OF pointers (const T* const*)
 *    are HOST arrays of device pointers, read during the call only.  The
 *    library never frees caller memory.
 *  - Every call is asynchronous on the caller's CUDA stream (`stream`, a
 *    cudaStream_t passed as void*; NULL = legacy default stream).  It returns
 *    after enqueueing.  Host-side validation failures return before any
 *    work is enqueued.
 *  - Return value: EQC_OK (0) or a negative EQC_E_* code.  Device-side
 *    failures (a corrupt RLE stream) are reported through a caller-provided
 *    device int32 `d_status`: kernels only ever store EQC_E_CORRUPT into it
 *    (sticky); the caller zeroes it.
 *  - The 128-bit vector fast path is taken when pointers are 16-byte aligned
 *    and pitch % 4 == 0; every other shape runs a scalar path with identical
 *    results.
 */
#ifndef EQC_H
#define EQC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define EQC_API __attribute__((visibility("default")))
#else
#define EQC_API
#endif

#define EQC_OK 0
#define EQC_E_INVALID (-1)     /* bad argument: null pointer, n out of range, w/h <= 0, pitch < w, ... */
#define EQC_E_CAPACITY (-2)    /* destination or workspace too small */
#define EQC_E_CORRUPT (-3)     /* RLE stream failed validation (device status word) */
#define EQC_E_UNSUPPORTED (-4) /* valid but unsupported combination (swizzle on depth, non-pow2 binary swap) */
#define EQC_E_CUDA (-5)        /* a CUDA runtime call failed (launch error, bad pointer, ...) */
#define EQC_E_NCCL (-6)        /* an NCCL call failed */

#define EQC_MAX_SOURCES 64     /* N per call (compositing) */

#define EQC_KIND_RGBA8 0       /* RLE kind: colour */
#define EQC_KIND_DEPTH32 1     /* RLE kind: depth */
#define EQC_FLAG_SWIZZLE 1     /* RLE flag: bit-swizzle preconditioner (colour only, R-C11) */
#define EQC_FLAG_RLE64 2       /* RLE flag: the basic 64-bit token codec (pixel pairs, R-C17);
                                  exclusive with EQC_FLAG_SWIZZLE; one codec per encode batch */

/* Human-readable name of an EQC_* code (static string, never NULL). */
EQC_API const char *eqc_strerror(int code);

/* Library ABI version: (major << 16) | (minor << 8) | patch. */
EQC_API int eqc_version(void);

/*
 * compositor_depth -- depth-sorted sort-last compositing ("assigns
 * the final pixel to the colour of the source with the front-most depth buffer
 * values"), one pass over N sources.
 *   out_color[p] = color[k][p], out_depth[p] = depth[k][p] with
 *   k = argmin_i (depth[i][p], i)  (lexicographic; ties -> lower index, R-C2).
 *   n          number of sources, 1 <= n <= EQC_MAX_SOURCES.
 *   color,depth  host arrays of n device pointers, each [h][pitch] uint32.
 *   out_color  device [h][out_pitch] uint32; out_depth nullable (colour only).
 *   Output may not alias inputs.  Errors: EQC_E_INVALID, EQC_E_CUDA.
 */
EQC_API int compositor_depth(int n, const uint32_t *const *color, const uint32_t *const *depth,
                     int w, int h, int64_t pitch, uint32_t *out_color, uint32_t *out_depth,
                     int64_t out_pitch, void *stream);

/*
 * compositor_blend_ordered -- spatial (DB / volume) sort-last compositing:
 * partial images "composited in order, typically with alpha-blending"
 * (P:2139-2146), order supplied by the application.
 * Premultiplied "over", back to front (R-C3), evaluated in fp32 and rounded
 * ONCE to RGBA8 (R-C4; within 1/255 of the exact value):
 *   x = bg/255;  for k = 0..n-1: x = s_{order[k]}/255 + x * (1 - a_{order[k]}/255)
 *   n          1 <= n <= EQC_MAX_SOURCES.
 *   color      host array of n device pointers to premultiplied RGBA8 [h][pitch].
 *   order      HOST int32[n], a permutation of [0, n): order[k] = source drawn
 *              k-th, back first; NULL = identity.  Non-permutation -> EQC_E_INVALID.
 *   background premultiplied RGBA8 drawn behind everything (usually 0).
 */
EQC_API int compositor_blend_ordered(int n, const uint32_t *const *color, const int32_t *order,
                             int w, int h, int64_t pitch, uint32_t background,
                             uint32_t *out_color, int64_t out_pitch, void *stream);

/*
 * compositor_average -- subpixel compositing: "accumulation and averaging of
 * all computed fragments for a pixel".  Per channel
 *   out_c = floor((2 * sum_i s_ic + n) / (2 n))   (mean rounded half up, R-C22)
 *   n          1 <= n <= EQC_MAX_SOURCES; color: host array of n device
 *              pointers to RGBA8 [h][pitch].  Bit-exact.
 */
EQC_API int compositor_average(int n, const uint32_t *const *color, int w, int h, int64_t pitch,
                               uint32_t *out_color, int64_t out_pitch, void *stream);

/*
 * Region of interest.  "The ROI is the screen-space 2D
 * bounding box fully enclosing the data rendered by a single resource"
 * (P:2259-2263); it "is transmitted to all input frames together with the
 * pixel data.  On the input frame, the compositing code respects this
 * parameter to place the pixel data in the right position".
 * A ROI is an int32 {x, y, w, h} in full-frame pixel coordinates; an empty
 * ROI is {0, 0, 0, 0}.  Rectangles are clipped to the frame (R-C19).
 *
 * image_roi -- ROI of each of n frames computed on the GPU "by analysing the
 *   framebuffer": the smallest rectangle containing every pixel
 *   whose value differs from `background` (depth buffers: 0xFFFFFFFF; colour
 *   of a blend layer: 0).
 *   frames     host array of n device pointers, each [h][pitch] uint32.
 *   d_roi      device int32[4 n], 16-byte aligned: receives the n ROIs.
 *   Three launches on `stream` (init, scan, finalise); no host sync.
 *
 * compositor_depth_roi / compositor_blend_ordered_roi -- compositor_depth /
 *   compositor_blend_ordered over sources that hold pixel data only inside
 *   their ROI: outside d_roi[4i..4i+3] source i is background (depth
 *   0xFFFFFFFF, colour 0) for depth compositing and transparent for blending,
 *   and its buffers are never read there.  Buffers are indexed like full
 *   frames ([h][pitch] from color[i]); a cropped buffer holding only the ROI
 *   may be passed as `crop - (y * pitch + x)` (only in-ROI addresses are
 *   dereferenced).  d_roi: DEVICE int32[4 n] (16-byte aligned), e.g. the
 *   output of image_roi, indexed by source (not by draw position).
 *   Results equal the full-frame calls on frames masked outside their ROIs.
 */
EQC_API int image_roi(int n, const uint32_t *const *frames, int w, int h, int64_t pitch, uint32_t background,
                      int32_t *d_roi, void *stream);
EQC_API int compositor_depth_roi(int n, const uint32_t *const *color, const uint32_t *const *depth,
                                 const int32_t *d_roi, int w, int h, int64_t pitch, uint32_t *out_color,
                                 uint32_t *out_depth, int64_t out_pitch, void *stream);
EQC_API int compositor_blend_ordered_roi(int n, const uint32_t *const *color, const int32_t *order,
                                         const int32_t *d_roi, int w, int h, int64_t pitch,
                                         uint32_t background, uint32_t *out_color, int64_t out_pitch,
                                         void *stream);

/*
 * RLE-BP v1 codec: per-component (byte-plane) run-length encoding
 * with the optional bit-swizzle preconditioner, decomposed into
 * 128-pixel row chunks.  Wire format: DESIGN.md section 5 (R-C8).
 *
 * image_rle_max_size -- upper bound of a stream: 32 + 16*ceil(w/128)*h + 4*w*h.
 *   Returns EQC_E_INVALID for w <= 0 or h <= 0.
 * image_rle_workspace_size -- bytes of device scratch image_compress_rle needs
 *   for ONE w x h image (per-run sizes + an L2-resident record scratch).  No
 *   state survives between calls, so no zero fill is needed.  A workspace
 *   must not be shared by calls that may run concurrently.
 */
EQC_API int64_t image_rle_max_size(int w, int h);
EQC_API size_t image_rle_workspace_size(int w, int h);

/*
 * image_compress_rle -- encode one w x h image of uint32 words (colour or depth).
 *   src        device [h][pitch] uint32.
 *   kind       EQC_KIND_RGBA8 or EQC_KIND_DEPTH32.
 *   flags      0 or EQC_FLAG_SWIZZLE (kind RGBA8 only, else EQC_E_UNSUPPORTED).
 *   dst        device buffer of dst_capacity bytes; must hold
 *              image_rle_max_size(w, h) bytes (else EQC_E_CAPACITY), so the
 *              encoder never needs a host round trip.
 *   d_size     device int64: receives the stream size in bytes.
 *   workspace  device scratch of >= image_rle_workspace_size(w, h) bytes,
 *              8-byte aligned.
 *   The stream is byte-identical to the CPU oracle's (deterministic).
 *   Enqueues (all asynchronous on `stream`, CUDA-graph capturable): a
 *   cudaMemsetAsync of the workspace's counters, the persistent encoder
 *   kernel (records into the workspace's record scratch) and the compaction
 *   kernel (records to their payload offsets, table, header, size); RLE-64
 *   batches use the encoder, run-scan and compaction kernels of the round-1
 *   design.
 */
EQC_API int image_compress_rle(const uint32_t *src, int w, int h, int64_t pitch, int kind, int flags,
                       uint8_t *dst, int64_t dst_capacity, int64_t *d_size, void *workspace,
                       size_t workspace_bytes, void *stream);

/*
 * image_decompress_rle -- decode a stream produced by image_compress_rle (or
 * the oracle) into a w x h image.
 *   src        device stream; src_bytes = bytes readable at src (>= the
 *              stream size; the true size is taken from the header).
 *   dst        device [h][pitch] uint32.
 *   d_status   device int32, sticky: set to EQC_E_CORRUPT if the stream fails
 *              validation (header fields vs w/h, offsets monotone and
 *              contiguous, token lengths, payload sizes); the caller zeroes it.
 *              Pixels of chunks that failed validation are unspecified.
 */
EQC_API int image_decompress_rle(const uint8_t *src, int64_t src_bytes, uint32_t *dst, int64_t pitch,
                         int w, int h, int32_t *d_status, void *stream);

/*
 * Batched codec calls: `count` (<= 64) images of identical w x h in ONE launch
 * (the chunked data decomposition of P:2427-2430 applied across images).
 *   Per image i: src[i]/dst[i] device pointers (host arrays), kind[i] and
 *   flags[i] (host arrays), d_sizes[i] (device int64 array); one shared
 *   d_status.  Encoder: each dst[i] holds dst_capacity >=
 *   image_rle_max_size(w, h) bytes; the workspace holds
 *   image_rle_workspace_size_batch(count, w, h) bytes.  Decoder:
 *   src_bytes[i] (host array) = bytes readable at src[i].
 */
EQC_API size_t image_rle_workspace_size_batch(int count, int w, int h);
EQC_API int image_compress_rle_batch(int count, const uint32_t *const *src, int w, int h, int64_t pitch,
                                     const int *kind, const int *flags, uint8_t *const *dst,
                                     int64_t dst_capacity, int64_t *d_sizes, void *workspace,
                                     size_t workspace_bytes, void *stream);
EQC_API int image_decompress_rle_batch(int count, const uint8_t *const *src, const int64_t *src_bytes,
                                       uint32_t *const *dst, int64_t pitch, int w, int h,
                                       int32_t *d_status, void *stream);

/*
 * compositor_depth_rle -- decode (stage 5) fused with depth assembly (stage 7)
 * of the asynchronous compositing pipeline: the n sources arrive
 * as RLE streams (colour and depth), are decoded chunk by chunk into registers
 * and z-composited without materialising the decoded frames in HBM.  Same
 * result as image_decompress_rle on every stream followed by compositor_depth.
 * Depth is decoded first; a source's colour chunk is decoded only where the
 * source wins at least one pixel of the 128-pixel chunk (a hidden source's
 * colour is never read).  Every stream's header and chunk table are
 * validated; record-level validation covers the records that are decoded.
 *   color_rle, depth_rle  host arrays of n device stream pointers (8-byte
 *              aligned); color_bytes[i] / depth_bytes[i] (host) = bytes
 *              readable at each.  Colour streams kind RGBA8 (any flags), depth
 *              streams kind DEPTH32, all w x h with 128-pixel chunks.
 *   out_color  device [h][out_pitch]; out_depth nullable.
 *   d_status   as in image_decompress_rle.
 */
EQC_API int compositor_depth_rle(int n, const uint8_t *const *color_rle, const uint8_t *const *depth_rle,
                                 const int64_t *color_bytes, const int64_t *depth_bytes, int w, int h,
                                 uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch,
                                 int32_t *d_status, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* EQC_H */
