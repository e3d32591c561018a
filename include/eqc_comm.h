/*
 * eqc_comm.h -- multi-GPU parallel compositing schedules of libeqc.
 *
 * Thesis: "Two commonly used parallel compositing algorithms are direct send
 * and binary swap.  Both distribute the compositing task equally over all
 * available resources, then collect the composited tiles on the destination
 * channel".  Direct send: each resource "fully composite[s] a
 * single tile" after every channel "exchanges ... colour+depth tiles with its
 * neighbours" (fDirectSend); binary swap "exchanges pixels
 * between pairs of nodes using a binary compositing tree" (fBS);
 * a "final colour-only output image" is assembled on the destination
 * (P:1582-1584).  Readings: R-C5 (tie rule across schedules), R-C13 (balanced
 * row bands), R-C14 (the destination is also a source), R-C15 (colour-only
 * gather); DESIGN.md section 3.
 *
 * One process per GPU.  The transport is NCCL (NVLink 5 / NVSwitch); the
 * unique id is bootstrapped by the caller (e.g. torch.distributed broadcast).
 * Conventions as in eqc.h: device buffers owned by the caller, host arrays
 * of device pointers, asynchronous on `stream`, negative EQC_E_* on error.
 */
#ifndef EQC_COMM_H
#define EQC_COMM_H

#include "eqc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct eqc_comm eqc_comm;

#define EQC_UNIQUE_ID_BYTES 128
#define EQC_OP_DEPTH 0      /* depth-sorted compositing (compositor_depth semantics) */
#define EQC_OP_BLEND 1      /* ordered back-to-front "over" (compositor_blend_ordered semantics, background 0):
                               global layer order = rank-block order; depth may be NULL; partials cross
                               GPUs as unorm16 RGBA (R-C6) and are rounded once to RGBA8 at the end */
#define EQC_OP_AVERAGE 2    /* subpixel accumulation + averaging (compositor_average semantics):
                               depth may be NULL; partial channel sums cross GPUs exactly as packed 16-bit
                               sums (<= 256 sources in total); bit-exact */
#define EQC_FLAG_RLE 1      /* ship bands as RLE-BP streams (colour swizzled + depth) */
#define EQC_FLAG_NCCL 2     /* direct send: force NCCL grouped send/recv instead of the NVLink peer-memory path */
#define EQC_FLAG_ROI 4      /* region of interest: peer-memory direct send reads and composites
                               only the ROI of every partial frame (computed on the device) */
#define EQC_FLAG_OVERLAP 8  /* the compose runs alongside other GPU work (the asynchronous pipeline,
                               P:2302-2310): the peer-memory pull kernels use at most one CTA per SM,
                               leaving the SMs to the overlapped kernels (higher pipeline throughput,
                               ~10 % longer compose latency when run alone) */

/* NCCL unique id of a new clique (rank 0 calls this and broadcasts the bytes). */
EQC_API int eqc_comm_get_unique_id(uint8_t id[EQC_UNIQUE_ID_BYTES]);

/*
 * eqc_comm_init -- join the clique as `rank` of `nranks` on the CURRENT CUDA
 * device (collective: every rank must call it).  *comm receives an opaque
 * handle that owns the NCCL communicator and the schedule's scratch buffers
 * (allocated lazily by the first compose call, reused afterwards).
 */
EQC_API int eqc_comm_init(eqc_comm **comm, int nranks, int rank, const uint8_t id[EQC_UNIQUE_ID_BYTES]);
EQC_API int eqc_comm_destroy(eqc_comm *comm);

/*
 * Traffic counters of the last compose call on this rank:
 * out[0] band messages sent (one per colour+depth band/region),
 * out[1] gather messages sent (colour bands to the destination),
 * out[2] payload bytes sent, out[3] payload bytes received.
 */
EQC_API int eqc_comm_stats(const eqc_comm *comm, int64_t out[4]);

/*
 * eqc_comm_frame_buffers -- zero-copy partial frames for the peer-memory
 * direct send (collective: every rank calls it with the same w, h; the first
 * call for a size allocates and maps, later calls are host-only lookups).
 * The asynchronous pipeline renders / decodes frame k into a buffer while
 * frame k-1 is composited; when that buffer is one the peers
 * have mapped, the pre-composite copy of step (1) disappears: the band
 * composite reads it in place over NVLink.
 *   slot        0 or 1 (two slots: one being composited, one being filled).
 *   *color, *depth  receive slot `slot`'s device buffers, [h][w] u32 each
 *               (pitch w).  Pass them (n_local = 1, pitch = w, EQC_OP_DEPTH,
 *               no ROI) to compose_direct_send and it skips the local copy;
 *               EVERY rank must then pass its own slot-`slot` buffers (like
 *               the matching calls of a collective; a mismatch is detected
 *               and reported by eqc_comm_check).
 *   *final_color  receives the comm's gather buffer [h][w]: passed as
 *               out_color (out_pitch = w) on dest_rank, the peers' bands land
 *               in it directly and the final band copy is skipped.
 *   stream      orders the collective setup (the call synchronises it on the
 *               first use of a size).
 * Ownership: the buffers belong to `comm` and stay valid until
 * eqc_comm_destroy, a larger eqc_comm_frame_buffers call, or (final_color
 * only) a compose call on a larger frame.  Reuse of a slot must wait for the
 * compose that read it (stream order / an event): peers read it until that
 * compose's closing barrier.
 * Errors: EQC_E_INVALID (arguments), EQC_E_UNSUPPORTED (one rank, or the
 * ranks cannot map each other's memory: use your own buffers, the NCCL
 * transport takes them), EQC_E_CUDA, EQC_E_NCCL.
 */
EQC_API int eqc_comm_frame_buffers(eqc_comm *comm, int w, int h, int slot, uint32_t **color, uint32_t **depth,
                                   uint32_t **final_color, void *stream);

/*
 * eqc_comm_stream_buffers -- peer-mapped RLE stream slots for
 * compose_direct_send_rle_pull (collective, same arguments on every rank;
 * the first call for a (n_streams, cap) allocates and maps both slots).
 *   n_streams   2 * n_local: streams 0..n_local-1 = the rank's colour
 *               streams, n_local..2*n_local-1 = its depth streams (the order
 *               image_compress_rle_batch fills them in).
 *   cap_bytes   capacity of one stream (>= image_rle_max_size(w, h)).
 *   ptrs[0..n_streams-1]  receive slot `slot`'s stream buffers (device).
 * Ownership and reuse as for eqc_comm_frame_buffers.  Errors: EQC_E_INVALID,
 * EQC_E_UNSUPPORTED (one rank, or no peer mapping), EQC_E_CUDA, EQC_E_NCCL.
 */
EQC_API int eqc_comm_stream_buffers(eqc_comm *comm, int n_streams, int64_t cap_bytes, int slot, uint8_t **ptrs,
                                    void *stream);

/*
 * compose_direct_send_rle_pull -- direct send of COMPRESSED sources: the
 * thesis pipeline "compress, transmit, decompress, assemble"
 * with the transmit step done by the decoder itself.  Every rank has encoded
 * its n_local sources into stream slot `slot` (eqc_comm_stream_buffers);
 * after a peer-memory barrier rank j runs the fused decode + depth composite
 * (compositor_depth_rle) over rows of band j (R-C13) of ALL n * n_local
 * sources -- the peers' streams read in place over NVLink, so only the
 * compressed records of band j cross the links (≈ r of the raw bytes) and no
 * partial frame is ever written -- and stores its band straight into the
 * destination's frame; colour gathered as in compose_direct_send.
 * Global source order is rank-major (R-C5): bit-identical to compositor_depth
 * over all sources.  out_color: [h][out_pitch] on dest_rank (the comm's gather
 * buffer from eqc_comm_frame_buffers avoids the final band copy).  d_status:
 * device int32, set non-zero if a stream is corrupt (as compositor_depth_rle).
 * Errors: EQC_E_INVALID (arguments, no stream slots of 2 * n_local streams,
 * n * n_local > 64), EQC_E_UNSUPPORTED (no peer mapping), EQC_E_CUDA.
 */
EQC_API int compose_direct_send_rle_pull(eqc_comm *comm, int n_local, int w, int h, int slot, int dest_rank,
                                         uint32_t *out_color, int64_t out_pitch, int32_t *d_status, void *stream);

/*
 * compositor_depth_rle_scatter + compose_direct_send_scattered -- direct send
 * with the exchange riding the decoder (the thesis's asynchronous pipeline,
 * P:2302-2310, with "transmit" fused into "decompress").  Rank r runs the
 * fused decode + depth composite of its n_local sources (as
 * compositor_depth_rle) band by band (bands R-C13), and stores band j
 * straight into frame slot `slot` of rank j over NVLink, as copy r of that
 * band: rows [r * maxband, r * maxband + rows_j) of the slot (pitch w,
 * maxband = the largest band).  compose_direct_send_scattered then, on every
 * rank after a peer-memory barrier, composites the n copies of its band from
 * its own slot (HBM reads only; global source order rank-major, R-C5) and
 * stores the result into the destination's frame (colour only), as
 * compose_direct_send.  Both are collective in the sense that every rank
 * calls them with the same w, h, slot; the scatter of frame k into slot i
 * must be ordered after every rank's compose of the previous frame that used
 * slot i (the compose ends with a barrier: order the scatter after it on the
 * caller's streams).  Slots come from eqc_comm_frame_buffers (they hold the
 * scattered layout).  d_status as compositor_depth_rle.  flags:
 * EQC_FLAG_OVERLAP caps the band composite at one CTA per SM.
 * Errors: EQC_E_INVALID (arguments, slots smaller than the layout),
 * EQC_E_UNSUPPORTED (one rank, no peer mapping or frame slots), EQC_E_CUDA.
 */
EQC_API int compositor_depth_rle_scatter(eqc_comm *comm, int n_local, const uint8_t *const *color_rle,
                                         const uint8_t *const *depth_rle, const int64_t *color_bytes,
                                         const int64_t *depth_bytes, int w, int h, int slot, int32_t *d_status,
                                         void *stream);
EQC_API int compose_direct_send_scattered(eqc_comm *comm, int w, int h, int slot, int dest_rank,
                                          uint32_t *out_color, int64_t out_pitch, int flags, void *stream);

/*
 * Host-side schedule plans (no GPU needed; used by the executors below and
 * by the tests).
 * eqc_plan_bands: row0[j] = floor(j*h/n), j = 0..n (band j = rows
 *   [row0[j], row0[j+1]), R-C13).
 * eqc_plan_bands_gather: the bands of the peer-memory direct send with a
 *   colour gather to `dest` (R-C13, n >= 3): the destination gets
 *   round(h/(2n-1)) rows, the other ranks equal shares of the rest (so every
 *   rank's NVLink inbound is about 8(n-1)/(2n-1) bytes per frame pixel);
 *   n <= 2 (or EQC_P2P_EQUAL_BANDS=1): eqc_plan_bands.
 * eqc_plan_binary_swap: for rank `rank` of n = 2^k ranks, fills k rounds of
 *   6 ints {partner, low (1 if rank's bit r is 0), keep_y0, keep_y1, send_y0,
 *   send_y1} (rows) and returns k; the region after the last round is the
 *   rank's final band.  EQC_E_UNSUPPORTED if n is not a power of two.
 */
EQC_API int eqc_plan_bands(int h, int n, int *row0);
EQC_API int eqc_plan_bands_gather(int h, int n, int dest, int *row0);
EQC_API int eqc_plan_binary_swap(int h, int n, int rank, int *rounds, int max_rounds);

/*
 * compose_direct_send -- sort-last compositing of all ranks' sources with the
 * direct-send schedule.  Rank g holds the n_local sources with global indices
 * [g*n_local, (g+1)*n_local) (contiguous blocks, R-C5).
 *   comm       this rank's communicator (collective call: every rank calls it
 *              with the same w, h, op, flags, dest_rank).
 *   color, depth  host arrays of n_local device pointers [h][pitch]; depth is
 *              ignored (may be NULL) for EQC_OP_BLEND / EQC_OP_AVERAGE.
 *   op         EQC_OP_DEPTH (below), EQC_OP_BLEND or EQC_OP_AVERAGE (the
 *              same schedule with the operator's partial format, see above).
 *   out_color  device [h][out_pitch] on dest_rank (NULL elsewhere).
 *   Scratch lives in `comm` (allocated at the first call, reused).
 *   Errors: EQC_E_INVALID (arguments), EQC_E_UNSUPPORTED (unknown op, more
 *   than 256 sources for EQC_OP_AVERAGE), EQC_E_CUDA, EQC_E_NCCL.
 *   (1) local pre-composite of the rank's sources (compositor_depth);
 *   (2) [EQC_FLAG_RLE: encode each outgoing band, exchange sizes];
 *   (3) every rank sends band j (colour + depth) to rank j (NCCL grouped
 *       send/recv over NVLink);
 *   (4) [decode]; rank j composites the n partial bands in rank order;
 *   (5) ranks send their composited colour band to dest_rank, which writes
 *       the final image to out_color [h][out_pitch] (ignored on other ranks).
 * Result: bit-identical to compositor_depth over all nranks*n_local sources.
 * Transport: without EQC_FLAG_RLE (raw bands) and when every rank can map
 * every peer's memory (CUDA IPC over NVLink, agreed collectively at the first
 * call), steps (2)-(4) are ONE kernel per rank: the band composite reads band
 * j of every peer's partial frame directly over NVLink and stores its result
 * directly into the destination's frame (two peer-memory flag barriers order
 * the steps; no staging, no NCCL on the data path).  Otherwise, or with
 * EQC_FLAG_NCCL, the bands move with NCCL grouped send/recv.  With
 * EQC_FLAG_RLE the call synchronises `stream` once (the message sizes are
 * read back to the host), so it returns only after the encodes finished and
 * cannot be captured in a CUDA graph; the same holds for the EQC_FLAG_RLE
 * variants of compose_binary_swap, compose_swap23 and compose_stream.
 * EQC_FLAG_ROI (peer-memory path; other transports ignore it): the local
 * pre-composite also reduces the bounding box of its rendered pixels (the
 * ROI computed "by analysing the framebuffer", fused: no extra
 * pass), publishes it in peer memory, and the band composite pulls only the
 * peers' pixels inside their boxes (the ROI travels with the
 * pixel data and places it).  Same result; fewer NVLink bytes when the
 * partial frames cover compact regions.
 */
EQC_API int compose_direct_send(eqc_comm *comm, int n_local, const uint32_t *const *color,
                                const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                int dest_rank, uint32_t *out_color, int64_t out_pitch, void *stream);

/*
 * compose_binary_swap -- same contract with the binary-swap schedule:
 * log2(n) rounds; in round r the partner is rank ^ 2^r, the current row
 * region [y0, y1) splits at m = y0 + floor((y1 - y0)/2), the rank whose bit
 * r is 0 keeps [y0, m) and sends [m, y1), the partner the reverse; the kept
 * half is composited with ties going to the bit-0 group (R-C5).  Finally
 * every rank's region (colour) is gathered on dest_rank.
 * EQC_E_UNSUPPORTED unless nranks is a power of two.
 * Transport: as compose_direct_send -- without EQC_FLAG_RLE / EQC_FLAG_NCCL
 * and when every rank maps every peer, each round's merge reads the
 * partner's half in place over NVLink (flag barriers between rounds) and the
 * last round writes straight into the destination's frame; otherwise NCCL
 * grouped send/recv per round.
 */
EQC_API int compose_binary_swap(eqc_comm *comm, int n_local, const uint32_t *const *color,
                                const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                int dest_rank, uint32_t *out_color, int64_t out_pitch, void *stream);

/*
 * Single-GPU "virtual rank" executors (the thesis's own testing trick of
 * running a sort-last compound on several channels of one GPU):
 * run the identical schedule for nranks virtual ranks in one process, with
 * device-to-device copies standing in for NCCL.  color/depth hold
 * nranks*n_local device pointers (rank-major).  Traffic counters are summed
 * over all virtual ranks into out_stats[4] (nullable).
 */
EQC_API int compose_direct_send_local(int nranks, int n_local, const uint32_t *const *color,
                                      const uint32_t *const *depth, int w, int h, int64_t pitch, int op,
                                      int flags, int dest_rank, uint32_t *out_color, int64_t out_pitch,
                                      int64_t *out_stats, void *stream);
EQC_API int compose_binary_swap_local(int nranks, int n_local, const uint32_t *const *color,
                                      const uint32_t *const *depth, int w, int h, int64_t pitch, int op,
                                      int flags, int dest_rank, uint32_t *out_color, int64_t out_pitch,
                                      int64_t *out_stats, void *stream);

/*
 * compose_swap23 -- the same contract with the 2-3 swap schedule (P:2193-2195:
 * binary swap extended to any number of ranks "by exchanging compositions
 * between groups of two or three nodes"), reading R-C21: with m the largest
 * 2^a 3^b <= nranks, ranks (2i, 2i+1), i < nranks - m, first fold (2i+1's
 * whole partial to 2i); the m remaining ranks then run mixed-radix swap
 * rounds, radix 2 rounds first then radix 3: a group = the ranks whose active
 * index differs only in the round's digit; the current row region splits into
 * k parts at y0 + floor(u (y1 - y0) / k); digit t keeps part t, receives it
 * from the k - 1 other members and composites the k partials in rank order.
 * For a power of two this is binary swap.  Final regions are gathered on
 * dest_rank.  All ops and flags of compose_direct_send; transport: peer
 * memory (in-place merges reading the members over NVLink, as
 * compose_binary_swap) when every rank maps every peer and neither
 * EQC_FLAG_RLE nor EQC_FLAG_NCCL is set, else NCCL.
 * eqc_plan_swap23 -- the plan of `rank` as ints: {fold_role (0 none, 1
 *   receiver, 2 sender), fold_partner, k rounds, final_y0, final_y1}, then per
 *   round {radix, digit, member[3] (-1 padded), bound[4]}; returns k.
 */
EQC_API int compose_swap23(eqc_comm *comm, int n_local, const uint32_t *const *color,
                           const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                           int dest_rank, uint32_t *out_color, int64_t out_pitch, void *stream);
EQC_API int compose_swap23_local(int nranks, int n_local, const uint32_t *const *color,
                                 const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                 int dest_rank, uint32_t *out_color, int64_t out_pitch, int64_t *out_stats,
                                 void *stream);
EQC_API int eqc_plan_swap23(int h, int n, int rank, int *out, int max_ints);

/*
 * compose_stream -- the streaming sort-last chain: rank k
 * receives the whole partial frame of ranks 0..k-1 from rank k-1 (raw or
 * EQC_FLAG_RLE streams), composites it under / before its own partial and
 * passes it to rank k+1; rank n-1 completes the frame and sends the colour to
 * dest_rank.  Latency t_local + (n - 1) (t_transfer + t_merge).
 * All ops; NCCL transport.  compose_stream_local: virtual ranks on one GPU.
 */
EQC_API int compose_stream(eqc_comm *comm, int n_local, const uint32_t *const *color,
                           const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                           int dest_rank, uint32_t *out_color, int64_t out_pitch, void *stream);
EQC_API int compose_stream_local(int nranks, int n_local, const uint32_t *const *color,
                                 const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                 int dest_rank, uint32_t *out_color, int64_t out_pitch, int64_t *out_stats,
                                 void *stream);

/*
 * compose_direct_send_roi -- compose_direct_send (EQC_OP_DEPTH) with
 * application-provided regions of interest: "Equalizer provides an API for
 * the programmer to provide the ROI ... the screen-space 2D bounding box fully
 * enclosing the data rendered by a single resource".
 *   d_src_roi  DEVICE int32[4 n_local] (16-byte aligned): {x, y, w, h} of each
 *              local source (full-frame coordinates, clipped to the frame,
 *              R-C19); outside it a source is background and never read.
 * The pre-composite reads only inside these ROIs; on the peer-memory path the
 * partial frame is written only inside their union box, which is published
 * and bounds the peers' pulls (as EQC_FLAG_ROI, without analysing the
 * frame).  Same result as compose_direct_send when every ROI encloses its
 * source's rendered pixels.  compose_direct_send_roi_local: virtual ranks
 * (d_src_roi holds nranks * n_local ROIs, rank-major).
 */
EQC_API int compose_direct_send_roi(eqc_comm *comm, int n_local, const uint32_t *const *color,
                                    const uint32_t *const *depth, const int32_t *d_src_roi, int w, int h,
                                    int64_t pitch, int flags, int dest_rank, uint32_t *out_color,
                                    int64_t out_pitch, void *stream);
EQC_API int compose_direct_send_roi_local(int nranks, int n_local, const uint32_t *const *color,
                                          const uint32_t *const *depth, const int32_t *d_src_roi, int w, int h,
                                          int64_t pitch, int flags, int dest_rank, uint32_t *out_color,
                                          int64_t out_pitch, int64_t *out_stats, void *stream);

/*
 * compose_tiles -- the display wall: direct send over the
 * wall's tiles, no gather.  The w x h frame is a tiles_x x tiles_y grid of
 * display tiles (segments/channels of a tiled wall):
 * tile t = (t % tiles_x, t / tiles_x) covers x in [floor(c w / tiles_x),
 * floor((c+1) w / tiles_x)), y likewise, and is owned by rank
 * floor(t * nranks / (tiles_x * tiles_y)) -- the channel driving it.
 * Every rank pre-composites its n_local sources (global indices as
 * compose_direct_send), ships each tile of its partial wall to the tile's
 * owner -- with EQC_FLAG_RLE as RLE-BP streams (colour swizzled + depth; the
 * owner runs the fused decode + depth composite over the n streams), else as
 * raw rectangles -- and the owner writes its composited tiles into out_color
 * [h][out_pitch] (its display frame; other tiles untouched).  Result: on
 * every tile, bit-identical to compositor_depth over all sources.  NCCL
 * transport; EQC_FLAG_RLE synchronises `stream` once (stream sizes).
 * EQC_OP_DEPTH only.  flags: 0 or EQC_FLAG_RLE.
 * compose_tiles_local: virtual ranks on one GPU, every rank writing its tiles
 *   into the one out_color; EQC_E_CORRUPT if a stream failed to decode.
 * eqc_plan_tiles: rect = {x0, y0, w, h, owner} of tile `tile`.
 */
EQC_API int compose_tiles(eqc_comm *comm, int n_local, const uint32_t *const *color, const uint32_t *const *depth,
                          int w, int h, int64_t pitch, int tiles_x, int tiles_y, int flags, uint32_t *out_color,
                          int64_t out_pitch, void *stream);
EQC_API int compose_tiles_local(int nranks, int n_local, const uint32_t *const *color, const uint32_t *const *depth,
                                int w, int h, int64_t pitch, int tiles_x, int tiles_y, int flags,
                                uint32_t *out_color, int64_t out_pitch, int64_t *out_stats, void *stream);
EQC_API int eqc_plan_tiles(int w, int h, int tiles_x, int tiles_y, int nranks, int tile, int *rect);

/*
 * Peer-memory transport on ONE GPU: compose_direct_send's NVLink peer-memory
 * path (P:2302-2310 stages (2)-(5) with no staging copy) run
 * for nranks virtual ranks of this process.  Every virtual rank gets its own
 * partial frame, gather buffer and flags page; the "peer mappings" are the
 * other virtual ranks' plain device pointers, and each virtual rank's part of
 * the call runs on its own stream (its flag barriers must run concurrently
 * with the others'), forked from and joined back to `stream`.  The host code
 * and kernels are those of the multi-process path.  The call synchronises
 * `stream` (its scratch is freed before it returns).
 *   mode  EQC_P2P_PLAIN      one pre-composite, barrier, pull + band
 *                            composite, barrier, band copy-out;
 *         EQC_P2P_PIPELINED  bands cut into pieces, pre-composite of piece
 *                            k+1 overlapped with the pull of piece k (progress
 *                            counters in peer memory; no EQC_FLAG_ROI);
 *         EQC_P2P_SLOTS      the partial frames are frame slots read in place
 *                            (n_local = 1, EQC_OP_DEPTH, no ROI; the caller's
 *                            frames are copied into the slots first).
 *   color/depth: nranks * n_local device pointers (rank-major), as
 *   compose_direct_send_local.  Result bit-identical to compositor_depth (or
 *   the op's single-GPU result) over all sources.
 * Errors: as compose_direct_send; EQC_E_NCCL if a flag wait timed out
 * (EQC_P2P_TIMEOUT_MS); EQC_E_INVALID if the ranks disagreed on frame slots.
 */
#define EQC_P2P_PLAIN 0
#define EQC_P2P_PIPELINED 1
#define EQC_P2P_SLOTS 2
EQC_API int compose_direct_send_p2p_local(int nranks, int n_local, const uint32_t *const *color,
                                          const uint32_t *const *depth, int w, int h, int64_t pitch, int op,
                                          int flags, int mode, int dest_rank, uint32_t *out_color,
                                          int64_t out_pitch, int64_t *out_stats, void *stream);

/*
 * compose_binary_swap_p2p_local -- the peer-memory binary swap (the default
 * transport of compose_binary_swap when every rank maps every peer, no
 * EQC_FLAG_RLE / EQC_FLAG_NCCL) for virtual ranks on one GPU, as above:
 * round r merges the kept half in place, reading the partner's rows of it
 * over NVLink; the last round writes the final colour into the destination's
 * frame.  nranks must be a power of two (else EQC_E_UNSUPPORTED).
 */
EQC_API int compose_binary_swap_p2p_local(int nranks, int n_local, const uint32_t *const *color,
                                          const uint32_t *const *depth, int w, int h, int64_t pitch, int op,
                                          int flags, int dest_rank, uint32_t *out_color, int64_t out_pitch,
                                          int64_t *out_stats, void *stream);

/*
 * compose_swap23_p2p_local -- the peer-memory 2-3 swap (the default transport
 * of compose_swap23 when every rank maps every peer, no EQC_FLAG_RLE /
 * EQC_FLAG_NCCL): the fold and each mixed-radix round merge in place, reading
 * the other members' rows over NVLink; the last round writes into the
 * destination's frame.  Virtual ranks on one GPU, any nranks >= 2.
 */
EQC_API int compose_swap23_p2p_local(int nranks, int n_local, const uint32_t *const *color,
                                     const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                     int dest_rank, uint32_t *out_color, int64_t out_pitch, int64_t *out_stats,
                                     void *stream);

/*
 * compose_direct_send_rle_pull on ONE GPU (virtual ranks as above): rank q's
 * 2 * n_local streams (colour 0..n_local-1, then depth) lie contiguously at
 * rank_streams[q], cap_bytes apart; the fused decode + composite of band j
 * (rows [floor(jh/n), floor((j+1)h/n)), R-C13) reads every rank's records in
 * place.  d_status as compositor_depth_rle.  Synchronises `stream`.
 */
EQC_API int compose_direct_send_rle_pull_local(int nranks, int n_local, const uint8_t *const *rank_streams,
                                               int64_t cap_bytes, int w, int h, int dest_rank,
                                               uint32_t *out_color, int64_t out_pitch, int32_t *d_status,
                                               int64_t *out_stats, void *stream);

/*
 * compositor_depth_rle_scatter + compose_direct_send_scattered on ONE GPU
 * (virtual ranks as above, each with its own frame slot): rank q's n_local
 * colour / depth streams are color_rle / depth_rle[q * n_local + i] (bytes in
 * color_bytes / depth_bytes).  Every rank decodes its bands into the ranks'
 * slots, then composites the copies of its own band; colour lands in
 * out_color on dest_rank.  d_status as compositor_depth_rle.  Synchronises
 * `stream`.
 */
EQC_API int compose_direct_send_scatter_local(int nranks, int n_local, const uint8_t *const *color_rle,
                                              const uint8_t *const *depth_rle, const int64_t *color_bytes,
                                              const int64_t *depth_bytes, int w, int h, int dest_rank,
                                              uint32_t *out_color, int64_t out_pitch, int32_t *d_status,
                                              int64_t *out_stats, void *stream);

/*
 * eqc_comm_check -- synchronise `stream`, then report the comm's health:
 * EQC_E_NCCL if NCCL reports an asynchronous error (ncclCommGetAsyncError)
 * or a peer-memory flag wait gave up (a dead or stalled peer: every wait
 * spins at most EQC_P2P_TIMEOUT_MS, default 60000, read at comm creation, so
 * the GPU never hangs on it); EQC_E_INVALID if the ranks passed different
 * frame slots to a compose call (see eqc_comm_frame_buffers); else EQC_OK.
 * After an error the results of the compose calls since the last check are
 * undefined.  eqc_comm_abort -- ncclCommAbort (unblocks NCCL operations of a
 * failed job); the comm may then only be destroyed.
 */
EQC_API int eqc_comm_check(eqc_comm *comm, void *stream);
EQC_API int eqc_comm_abort(eqc_comm *comm);

#ifdef __cplusplus
}
#endif

#endif /* EQC_COMM_H */
