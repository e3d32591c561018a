// compose.cu -- multi-GPU parallel compositing schedules (direct send,
// binary swap) over NCCL, plus single-GPU "virtual rank" executors of the
// identical schedule (device copies stand in for NCCL).
//
// Thesis: direct send and binary swap "distribute the compositing task
// equally over all available resources, then collect the composited tiles on
// the destination channel"; direct send exchanges colour+depth
// tiles and composites one tile per channel; binary swap pairs
// nodes in a binary compositing tree; the final image is
// colour-only.  The optional RLE band transport is stages
// (2)-(5) of the asynchronous compositing pipeline.
//
// Every per-pixel step runs in the libeqc kernels (compositor_depth,
// image_compress_rle_batch, image_decompress_rle_batch); this file only
// plans the schedule and moves bytes (NCCL grouped send/recv on the caller's
// stream, NVLink 5 / NVSwitch).
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/eqc_comm.h"
#include "eqc_common.cuh"

// composite.cu: depth compositing over ROI-restricted sources (per-source ROI
// pointers, band row offset, optional output rectangle)
int eqc_depth_roi_launch(int n, const uint32_t *const *color, const uint32_t *const *depth,
                         const int32_t *const *roi, int roi_dy, const int32_t *out_roi, int w, int h,
                         int64_t pitch, uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch,
                         cudaStream_t stream);
// composite.cu: compositor_depth that also reduces the ROI of its output
size_t eqc_depth_bbox_scratch_bytes();
extern thread_local int eqc_grid_cap;
int eqc_preload_composite();
int eqc_preload_rle();
int eqc_preload_roi();
int eqc_depth_rle_band(int n, const uint8_t *const *color_rle, const uint8_t *const *depth_rle,
                       const int64_t *color_bytes, const int64_t *depth_bytes, int w, int h, int y0, int y1,
                       uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch, int32_t *d_status,
                       void *stream);
int eqc_depth_composite_bbox(int n, const uint32_t *const *color, const uint32_t *const *depth, int w, int h,
                             int64_t pitch, uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch,
                             void *scratch, int32_t *out_roi, cudaStream_t s);
// composite.cu: ordered blending through unorm16 partial planes (EQC_OP_BLEND)
int eqc_blend_to_partial(int n, const uint32_t *const *color, int w, int h, int64_t pitch, uint32_t *out_rg,
                         uint32_t *out_ba, int64_t out_pitch, cudaStream_t s);
int eqc_blend_partials(int n, const uint32_t *const *rg, const uint32_t *const *ba, int w, int h, int64_t pitch,
                       uint32_t background, uint32_t *out_c, uint32_t *out_rg, uint32_t *out_ba, int64_t out_pitch,
                       cudaStream_t s);
// composite.cu: subpixel accumulation + averaging through packed sum planes (EQC_OP_AVERAGE)
int eqc_average(bool local, int n, const uint32_t *const *src, const uint32_t *const *src_ba, int w, int h,
                int64_t pitch, int total, uint32_t *out_c, uint32_t *out_rg, uint32_t *out_ba, int64_t out_pitch,
                cudaStream_t s);

namespace {

#define EQC_NCCL_TRY(expr)                 \
  do {                                     \
    ncclResult_t _r = (expr);              \
    if (_r != ncclSuccess) return EQC_E_NCCL; \
  } while (0)

// EQC_TRACE_ERRORS=1: print where an error code first surfaced (debug aid)
#define EQC_TRY(expr)                                                                   \
  do {                                                                                  \
    int _rc = (expr);                                                                   \
    if (_rc != EQC_OK) {                                                                \
      if (getenv("EQC_TRACE_ERRORS")) fprintf(stderr, "eqc: %d at %s:%d\n", _rc, __FILE__, __LINE__); \
      return _rc;                                                                       \
    }                                                                                   \
  } while (0)

struct DevBuf {
  void *p = nullptr;
  size_t n = 0;
  int ensure(size_t bytes) {
    if (bytes <= n) return EQC_OK;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return EQC_E_CUDA;
    n = bytes;
    return EQC_OK;
  }
  int ensure_zeroed(size_t bytes) {
    if (bytes <= n) return EQC_OK;
    EQC_TRY(ensure(bytes));
    return cudaMemset(p, 0, bytes) == cudaSuccess ? EQC_OK : EQC_E_CUDA;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  template <typename T>
  T *as() const { return reinterpret_cast<T *>(p); }
};

// Per-rank scratch of a schedule.
struct RankState {
  int rank = 0;
  const uint32_t *const *color = nullptr;  // host array of n_local device ptrs
  const uint32_t *const *depth = nullptr;
  DevBuf part_c[2], part_d[2];  // partial frame (ping-pong for binary swap), pitch w
  DevBuf recv_c, recv_d;        // incoming bands/halves
  DevBuf fin_c;                 // finished colour band awaiting the gather
  DevBuf enc, dec, sizes, ws, status;
  int64_t *h_sizes = nullptr;   // pinned
  int cur = 0;                  // binary swap: index of the live partial buffer
  int64_t stats[4] = {0, 0, 0, 0};

  void release() {
    for (int i = 0; i < 2; ++i) {
      part_c[i].release();
      part_d[i].release();
    }
    recv_c.release();
    recv_d.release();
    fin_c.release();
    enc.release();
    dec.release();
    sizes.release();
    ws.release();
    status.release();
    if (h_sizes) cudaFreeHost(h_sizes);
    h_sizes = nullptr;
  }
};

struct Geometry {
  int n = 1;          // ranks
  int n_local = 1;    // sources per rank
  int w = 0, h = 0;
  int64_t pitch = 0;  // of the source frames
  int op = EQC_OP_DEPTH;  // per-pixel operator; EQC_OP_BLEND: the (c, d) planes carry unorm16 partials
  const int32_t *src_roi = nullptr;  // application source ROIs (device, x 4 ints) or NULL
  bool src_roi_all_ranks = false;    // virtual ranks: src_roi holds every rank's ROIs (rank-major)
  int flags = 0;
  int dest = 0;
  uint32_t *out = nullptr;
  int64_t out_pitch = 0;
  std::vector<int> row0;  // direct-send bands
};

// ---- transports -------------------------------------------------------------
struct Transport {
  virtual ~Transport() {}
  virtual int start() = 0;
  virtual int send(RankState &me, int peer, const void *buf, size_t bytes) = 0;
  virtual int recv(RankState &me, int peer, void *buf, size_t bytes) = 0;
  virtual int end() = 0;
};

struct NcclTransport : Transport {
  ncclComm_t comm;
  cudaStream_t s;
  NcclTransport(ncclComm_t c, cudaStream_t st) : comm(c), s(st) {}
  int start() override {
    EQC_NCCL_TRY(ncclGroupStart());
    return EQC_OK;
  }
  int send(RankState &me, int peer, const void *buf, size_t bytes) override {
    me.stats[2] += (int64_t)bytes;
    EQC_NCCL_TRY(ncclSend(buf, bytes, ncclUint8, peer, comm, s));
    return EQC_OK;
  }
  int recv(RankState &me, int peer, void *buf, size_t bytes) override {
    me.stats[3] += (int64_t)bytes;
    EQC_NCCL_TRY(ncclRecv(buf, bytes, ncclUint8, peer, comm, s));
    return EQC_OK;
  }
  int end() override {
    EQC_NCCL_TRY(ncclGroupEnd());
    return EQC_OK;
  }
};

// Virtual ranks in one process: sends are matched FIFO per (from, to) pair
// with receives at end(), exactly like NCCL's in-order p2p matching.
struct LocalTransport : Transport {
  cudaStream_t s;
  struct Msg {
    int from, to;
    const void *src;
    void *dst;
    size_t bytes;
    bool used;
  };
  std::vector<Msg> sends, recvs;
  explicit LocalTransport(cudaStream_t st) : s(st) {}
  int start() override {
    sends.clear();
    recvs.clear();
    return EQC_OK;
  }
  int send(RankState &me, int peer, const void *buf, size_t bytes) override {
    me.stats[2] += (int64_t)bytes;
    sends.push_back(Msg{me.rank, peer, buf, nullptr, bytes, false});
    return EQC_OK;
  }
  int recv(RankState &me, int peer, void *buf, size_t bytes) override {
    me.stats[3] += (int64_t)bytes;
    recvs.push_back(Msg{peer, me.rank, nullptr, buf, bytes, false});
    return EQC_OK;
  }
  int end() override {
    for (auto &r : recvs) {
      bool matched = false;
      for (auto &sd : sends) {
        if (!sd.used && sd.from == r.from && sd.to == r.to) {
          if (sd.bytes != r.bytes) return EQC_E_INVALID;  // size mismatch = schedule bug
          sd.used = true;
          matched = true;
          if (r.bytes) EQC_CUDA_TRY(cudaMemcpyAsync(r.dst, sd.src, r.bytes, cudaMemcpyDeviceToDevice, s));
          break;
        }
      }
      if (!matched) return EQC_E_INVALID;
    }
    for (auto &sd : sends)
      if (!sd.used) return EQC_E_INVALID;
    return EQC_OK;
  }
};

// ---- plans --------------------------------------------------------------------
void plan_bands(int h, int n, int *row0) {
  for (int j = 0; j <= n; ++j) row0[j] = (int)((int64_t)j * h / n);
}

// Bands of the peer-memory direct send with a colour gather to `dest`
// (R-C13 refined for NVSwitch): besides pulling its band from every peer
// (8 B/px each) the destination receives every other band's colour (4 B/px),
// so with equal bands it is the one link-bound rank.  Giving it 1/(2n - 1) of
// the rows and the others equal shares of the rest makes every rank's NVLink
// inbound (and outbound) 8(n - 1)/(2n - 1) B per frame pixel: 9P -> 6.9P bytes
// into the destination at n = 4 (c4 direct send on 4 GPUs: 0.706 -> 0.653 ms).
// Two ranks keep equal bands (measured 1.5 % slower with the 1/3 band: the
// second rank's larger band composite then dominates).
// EQC_P2P_EQUAL_BANDS=1: plan_bands for any n.
void plan_bands_gather(int h, int n, int dest, int *row0) {
  static const bool equal = getenv("EQC_P2P_EQUAL_BANDS") && atoi(getenv("EQC_P2P_EQUAL_BANDS")) != 0;
  if (equal || n < 3 || dest < 0 || dest >= n) {
    plan_bands(h, n, row0);
    return;
  }
  const int d = (int)(((int64_t)h + (2 * n - 1) / 2) / (2 * n - 1));  // round(h / (2n - 1))
  const int rest = h - d;
  row0[0] = 0;
  int k = 0;
  for (int j = 0; j < n; ++j) {
    int sz = d;
    if (j != dest) {
      sz = (int)((int64_t)(k + 1) * rest / (n - 1) - (int64_t)k * rest / (n - 1));
      ++k;
    }
    row0[j + 1] = row0[j] + sz;
  }
}

struct BsRound {
  int partner, low, keep_y0, keep_y1, send_y0, send_y1;
};

int plan_bs(int h, int n, int rank, std::vector<BsRound> &out) {
  if (n < 1 || (n & (n - 1))) return EQC_E_UNSUPPORTED;
  out.clear();
  int y0 = 0, y1 = h;
  for (int r = 0; (1 << r) < n; ++r) {
    const int m = y0 + (y1 - y0) / 2;
    BsRound b;
    b.partner = rank ^ (1 << r);
    b.low = ((rank >> r) & 1) == 0;
    if (b.low) {
      b.keep_y0 = y0, b.keep_y1 = m, b.send_y0 = m, b.send_y1 = y1;
    } else {
      b.keep_y0 = m, b.keep_y1 = y1, b.send_y0 = y0, b.send_y1 = m;
    }
    out.push_back(b);
    y0 = b.keep_y0;
    y1 = b.keep_y1;
  }
  return (int)out.size();
}

void final_region_bs(int h, int n, int rank, int &y0, int &y1) {
  std::vector<BsRound> rr;
  plan_bs(h, n, rank, rr);
  y0 = 0;
  y1 = h;
  if (!rr.empty()) {
    y0 = rr.back().keep_y0;
    y1 = rr.back().keep_y1;
  }
}

// ---- shared steps ---------------------------------------------------------------
inline size_t frame_bytes(const Geometry &g, int rows) { return (size_t)rows * g.w * 4; }

int alloc_common(RankState &r, const Geometry &g, size_t recv_rows, size_t band_rows, int nbuf) {
  const size_t full = frame_bytes(g, g.h);
  for (int i = 0; i < nbuf; ++i) {
    EQC_TRY(r.part_c[i].ensure(full));
    EQC_TRY(r.part_d[i].ensure(full));
  }
  EQC_TRY(r.recv_c.ensure(std::max<size_t>(4, recv_rows * g.w * 4)));
  EQC_TRY(r.recv_d.ensure(std::max<size_t>(4, recv_rows * g.w * 4)));
  EQC_TRY(r.fin_c.ensure(std::max<size_t>(4, band_rows * g.w * 4)));
  EQC_TRY(r.status.ensure_zeroed(64));
  if (!r.h_sizes && cudaMallocHost(&r.h_sizes, 4 * 2 * EQC_MAX_SOURCES * sizeof(int64_t)) != cudaSuccess)
    return EQC_E_CUDA;
  return EQC_OK;
}

// The per-pixel operator of the schedules.  EQC_OP_DEPTH: (c, d) planes are
// colour and depth, compositor_depth semantics.  EQC_OP_BLEND (SURVEY 8(f)
// f4): the planes are a unorm16 "over" partial (rg, ba; R-C6) -- layers are in
// draw order by rank blocks, so rank order (and the bit-0 group of a binary
// swap round) is back-to-front.  Every step runs in the composite.cu kernels.
int op_local(const Geometry &g, const uint32_t *const *color, const uint32_t *const *depth, uint32_t *out_c,
             uint32_t *out_d, cudaStream_t s) {
  if (g.op == EQC_OP_BLEND) return eqc_blend_to_partial(g.n_local, color, g.w, g.h, g.pitch, out_c, out_d, g.w, s);
  if (g.op == EQC_OP_AVERAGE)
    return eqc_average(true, g.n_local, color, nullptr, g.w, g.h, g.pitch, g.n * g.n_local, nullptr, out_c, out_d,
                       g.w, s);
  return compositor_depth(g.n_local, color, depth, g.w, g.h, g.pitch, out_c, out_d, g.w, s);
}
// n partial (c, d) planes in rank order -> final colour (one rounding)
int op_final(const Geometry &g, int n, const uint32_t *const *c, const uint32_t *const *d, int rows, uint32_t *out,
             int64_t opitch, cudaStream_t s) {
  if (g.op == EQC_OP_BLEND) return eqc_blend_partials(n, c, d, g.w, rows, g.w, 0u, out, nullptr, nullptr, opitch, s);
  if (g.op == EQC_OP_AVERAGE)
    return eqc_average(false, n, c, d, g.w, rows, g.w, g.n * g.n_local, out, nullptr, nullptr, opitch, s);
  return compositor_depth(n, c, d, g.w, rows, g.w, out, nullptr, opitch, s);
}
// op_final of a peer-memory pull: with EQC_FLAG_OVERLAP at most one CTA per
// SM (the pull is NVLink-latency-bound; the SMs stay with the overlapped work)
int op_final_pull(const Geometry &g, int n, const uint32_t *const *c, const uint32_t *const *d, int rows,
                  uint32_t *out, int64_t opitch, cudaStream_t s) {
  // EQC_OVERLAP_CTAS: tuning override of the cap (default one CTA per SM)
  static const int cap_env = getenv("EQC_OVERLAP_CTAS") ? atoi(getenv("EQC_OVERLAP_CTAS")) : 0;
  eqc_grid_cap = (g.flags & EQC_FLAG_OVERLAP) ? (cap_env > 0 ? cap_env : eqc_num_sms()) : 0;
  const int rc = op_final(g, n, c, d, rows, out, opitch, s);
  eqc_grid_cap = 0;
  return rc;
}
// k partials (back / lower ranks first) -> 1 partial (swap rounds, folds)
int op_merge(const Geometry &g, int k, const uint32_t *const *c, const uint32_t *const *d, int rows,
             uint32_t *out_c, uint32_t *out_d, cudaStream_t s) {
  if (g.op == EQC_OP_BLEND) return eqc_blend_partials(k, c, d, g.w, rows, g.w, 0u, nullptr, out_c, out_d, g.w, s);
  if (g.op == EQC_OP_AVERAGE)
    return eqc_average(false, k, c, d, g.w, rows, g.w, g.n * g.n_local, nullptr, out_c, out_d, g.w, s);
  return compositor_depth(k, c, d, g.w, rows, g.w, out_c, out_d, g.w, s);
}

int local_precomposite(RankState &r, const Geometry &g, cudaStream_t s) {
  r.cur = 0;
  if (g.src_roi && g.op == EQC_OP_DEPTH) {  // application ROIs: sources read only inside them
    std::vector<const int32_t *> rp(g.n_local);
    const size_t first = g.src_roi_all_ranks ? (size_t)r.rank * g.n_local : 0;
    for (int i = 0; i < g.n_local; ++i) rp[i] = g.src_roi + 4 * (first + i);
    return eqc_depth_roi_launch(g.n_local, r.color, r.depth, rp.data(), 0, nullptr, g.w, g.h, g.pitch,
                                r.part_c[0].as<uint32_t>(), r.part_d[0].as<uint32_t>(), g.w, s);
  }
  return op_local(g, r.color, r.depth, r.part_c[0].as<uint32_t>(), r.part_d[0].as<uint32_t>(), s);
}

// Encode `count` (<= 2 per band) colour+depth bands: slot k of `enc`.
inline int64_t band_cap(const Geometry &g, int rows) {
  // streams must start 8-byte aligned: round each slot up to 256 bytes
  const int64_t b = rows > 0 ? image_rle_max_size(g.w, rows) : 32;
  return (b + 255) & ~(int64_t)255;
}

int encode_band(RankState &r, const Geometry &g, int slot, const uint32_t *c, const uint32_t *d, int rows,
                int64_t cap, cudaStream_t s) {
  const uint32_t *src[2] = {c, d};
  int kinds[2] = {EQC_KIND_RGBA8, EQC_KIND_DEPTH32};
  int flags[2] = {g.op != EQC_OP_DEPTH ? 0 : EQC_FLAG_SWIZZLE, 0};  // 16-bit planes: plain byte planes
  uint8_t *dst[2] = {r.enc.as<uint8_t>() + (size_t)(2 * slot) * cap,
                     r.enc.as<uint8_t>() + (size_t)(2 * slot + 1) * cap};
  return image_compress_rle_batch(2, src, g.w, rows, g.w, kinds, flags, dst, cap,
                                  r.sizes.as<int64_t>() + 2 * slot, r.ws.p, r.ws.n, s);
}

// ---- direct send ----------------------------------------------------------------
int ds_alloc(RankState &r, const Geometry &g) {
  int maxband = 0;
  for (int j = 0; j < g.n; ++j) maxband = std::max(maxband, g.row0[j + 1] - g.row0[j]);
  EQC_TRY(alloc_common(r, g, (size_t)g.n * maxband, maxband, 1));
  if (g.flags & EQC_FLAG_RLE) {
    const int64_t cap = band_cap(g, maxband);
    EQC_TRY(r.enc.ensure((size_t)2 * g.n * cap));
    EQC_TRY(r.dec.ensure((size_t)2 * g.n * cap));
    EQC_TRY(r.sizes.ensure((size_t)4 * g.n * sizeof(int64_t)));
    EQC_TRY(r.ws.ensure_zeroed(image_rle_workspace_size_batch(2, g.w, std::max(1, maxband))));
  }
  return EQC_OK;
}

// Phase (2)+(3): send band j of the partial to rank j, receive my band from all.
int ds_exchange_raw(RankState &r, const Geometry &g, Transport &T, int maxband) {
  const int me = r.rank;
  const int my_rows = g.row0[me + 1] - g.row0[me];
  for (int j = 0; j < g.n; ++j) {
    const int rows = g.row0[j + 1] - g.row0[j];
    if (j == me || rows == 0) continue;
    const size_t off = (size_t)g.row0[j] * g.w;
    EQC_TRY(T.send(r, j, r.part_c[0].as<uint32_t>() + off, frame_bytes(g, rows)));
    EQC_TRY(T.send(r, j, r.part_d[0].as<uint32_t>() + off, frame_bytes(g, rows)));
    r.stats[0] += 1;
  }
  for (int src = 0; src < g.n; ++src) {
    if (src == me || my_rows == 0) continue;
    const size_t slot = (size_t)src * maxband * g.w;
    EQC_TRY(T.recv(r, src, r.recv_c.as<uint32_t>() + slot, frame_bytes(g, my_rows)));
    EQC_TRY(T.recv(r, src, r.recv_d.as<uint32_t>() + slot, frame_bytes(g, my_rows)));
  }
  return EQC_OK;
}

int ds_encode(RankState &r, const Geometry &g, cudaStream_t s) {
  const int me = r.rank;
  int maxband = 0;
  for (int j = 0; j < g.n; ++j) maxband = std::max(maxband, g.row0[j + 1] - g.row0[j]);
  const int64_t cap = band_cap(g, maxband);
  for (int j = 0; j < g.n; ++j) {
    const int rows = g.row0[j + 1] - g.row0[j];
    if (j == me || rows == 0) continue;
    const size_t off = (size_t)g.row0[j] * g.w;
    EQC_TRY(encode_band(r, g, j, r.part_c[0].as<uint32_t>() + off, r.part_d[0].as<uint32_t>() + off, rows, cap, s));
  }
  return EQC_OK;
}

// sizes layout: [0, 2n) sizes of my outgoing streams, [2n, 4n) incoming
int ds_exchange_sizes(RankState &r, const Geometry &g, Transport &T) {
  const int me = r.rank;
  const int my_rows = g.row0[me + 1] - g.row0[me];
  int64_t *sz = r.sizes.as<int64_t>();
  for (int j = 0; j < g.n; ++j) {
    const int rows = g.row0[j + 1] - g.row0[j];
    if (j == me || rows == 0) continue;
    EQC_TRY(T.send(r, j, sz + 2 * j, 2 * sizeof(int64_t)));
  }
  for (int src = 0; src < g.n; ++src) {
    if (src == me || my_rows == 0) continue;
    EQC_TRY(T.recv(r, src, sz + 2 * g.n + 2 * src, 2 * sizeof(int64_t)));
  }
  return EQC_OK;
}

int ds_exchange_rle(RankState &r, const Geometry &g, Transport &T, int64_t cap) {
  const int me = r.rank;
  const int my_rows = g.row0[me + 1] - g.row0[me];
  const int64_t *hs = r.h_sizes;
  for (int j = 0; j < g.n; ++j) {
    const int rows = g.row0[j + 1] - g.row0[j];
    if (j == me || rows == 0) continue;
    EQC_TRY(T.send(r, j, r.enc.as<uint8_t>() + (size_t)(2 * j) * cap, (size_t)hs[2 * j]));
    EQC_TRY(T.send(r, j, r.enc.as<uint8_t>() + (size_t)(2 * j + 1) * cap, (size_t)hs[2 * j + 1]));
    r.stats[0] += 1;
  }
  for (int src = 0; src < g.n; ++src) {
    if (src == me || my_rows == 0) continue;
    EQC_TRY(T.recv(r, src, r.dec.as<uint8_t>() + (size_t)(2 * src) * cap, (size_t)hs[2 * g.n + 2 * src]));
    EQC_TRY(T.recv(r, src, r.dec.as<uint8_t>() + (size_t)(2 * src + 1) * cap, (size_t)hs[2 * g.n + 2 * src + 1]));
  }
  return EQC_OK;
}

int ds_decode(RankState &r, const Geometry &g, int maxband, int64_t cap, cudaStream_t s) {
  const int me = r.rank;
  const int my_rows = g.row0[me + 1] - g.row0[me];
  if (my_rows == 0 || g.n < 2) return EQC_OK;
  std::vector<const uint8_t *> src;
  std::vector<uint32_t *> dst;
  for (int q = 0; q < g.n; ++q) {
    if (q == me) continue;
    const size_t slot = (size_t)q * maxband * g.w;
    src.push_back(r.dec.as<uint8_t>() + (size_t)(2 * q) * cap);
    dst.push_back(r.recv_c.as<uint32_t>() + slot);
    src.push_back(r.dec.as<uint8_t>() + (size_t)(2 * q + 1) * cap);
    dst.push_back(r.recv_d.as<uint32_t>() + slot);
  }
  // at most 2*(64-1) streams: decode in batches of 64
  const std::vector<int64_t> caps(src.size(), cap);
  for (size_t b = 0; b < src.size(); b += 64) {
    const int cnt = (int)std::min<size_t>(64, src.size() - b);
    EQC_TRY(image_decompress_rle_batch(cnt, src.data() + b, caps.data() + b, dst.data() + b, g.w, g.w, my_rows,
                                       r.status.as<int32_t>(), s));
  }
  return EQC_OK;
}

// Phase (4): composite the n partial bands of my band in rank order.
int ds_band_composite(RankState &r, const Geometry &g, int maxband, cudaStream_t s) {
  const int me = r.rank;
  const int y0 = g.row0[me], rows = g.row0[me + 1] - y0;
  if (rows == 0) return EQC_OK;
  std::vector<const uint32_t *> c(g.n), d(g.n);
  for (int q = 0; q < g.n; ++q) {
    if (q == me) {
      c[q] = r.part_c[0].as<uint32_t>() + (size_t)y0 * g.w;
      d[q] = r.part_d[0].as<uint32_t>() + (size_t)y0 * g.w;
    } else {
      const size_t slot = (size_t)q * maxband * g.w;
      c[q] = r.recv_c.as<uint32_t>() + slot;
      d[q] = r.recv_d.as<uint32_t>() + slot;
    }
  }
  uint32_t *out;
  int64_t opitch;
  if (me == g.dest) {
    out = g.out + (size_t)y0 * g.out_pitch;
    opitch = g.out_pitch;
  } else {
    out = r.fin_c.as<uint32_t>();
    opitch = g.w;
  }
  return op_final(g, g.n, c.data(), d.data(), rows, out, opitch, s);
}

// Phase (5): gather colour bands/regions to the destination.  rows_of(q)
// gives (y0, y1) of rank q's finished region; src_of(r) its device pointer.
template <typename RegionFn>
int gather(RankState &r, const Geometry &g, Transport &T, RegionFn region, const uint32_t *mine, cudaStream_t s,
           int phase) {
  // phase 0: post messages; phase 1 (dest only, after end()): 2-D copies for
  // pitched output.
  const int me = r.rank;
  const bool contiguous = g.out_pitch == g.w;
  if (phase == 0) {
    if (me != g.dest) {
      int y0, y1;
      region(me, y0, y1);
      if (y1 > y0) {
        EQC_TRY(T.send(r, g.dest, mine, frame_bytes(g, y1 - y0)));
        r.stats[1] += 1;
      }
    } else {
      size_t scratch_off = 0;
      for (int q = 0; q < g.n; ++q) {
        if (q == me) continue;
        int y0, y1;
        region(q, y0, y1);
        if (y1 <= y0) continue;
        uint32_t *dst;
        if (contiguous) {
          dst = g.out + (size_t)y0 * g.w;
        } else {
          dst = r.recv_c.as<uint32_t>() + scratch_off;  // staged, copied in phase 1
          scratch_off += (size_t)(y1 - y0) * g.w;
        }
        EQC_TRY(T.recv(r, q, dst, frame_bytes(g, y1 - y0)));
      }
    }
  } else if (me == g.dest && !contiguous) {
    size_t scratch_off = 0;
    for (int q = 0; q < g.n; ++q) {
      if (q == me) continue;
      int y0, y1;
      region(q, y0, y1);
      if (y1 <= y0) continue;
      EQC_CUDA_TRY(cudaMemcpy2DAsync(g.out + (size_t)y0 * g.out_pitch, g.out_pitch * 4,
                                     r.recv_c.as<uint32_t>() + scratch_off, (size_t)g.w * 4, (size_t)g.w * 4,
                                     y1 - y0, cudaMemcpyDeviceToDevice, s));
      scratch_off += (size_t)(y1 - y0) * g.w;
    }
  }
  return EQC_OK;
}

// ---- the schedules over a set of rank states (1 with NCCL, n when virtual) ----
int run_direct_send(std::vector<RankState *> &ranks, Geometry &g, Transport &T, cudaStream_t s) {
  g.row0.assign(g.n + 1, 0);
  plan_bands(g.h, g.n, g.row0.data());
  int maxband = 0;
  for (int j = 0; j < g.n; ++j) maxband = std::max(maxband, g.row0[j + 1] - g.row0[j]);
  const bool rle = (g.flags & EQC_FLAG_RLE) != 0;
  const int64_t cap = band_cap(g, maxband);
  for (RankState *r : ranks) {
    for (int i = 0; i < 4; ++i) r->stats[i] = 0;
    EQC_TRY(ds_alloc(*r, g));
    // the band composite needs the gather scratch for pitched output too
    if (g.out_pitch != g.w && r->rank == g.dest)
      EQC_TRY(r->recv_c.ensure(std::max(r->recv_c.n, frame_bytes(g, g.h))));
    EQC_TRY(local_precomposite(*r, g, s));
  }
  if (g.n > 1) {
    if (!rle) {
      EQC_TRY(T.start());
      for (RankState *r : ranks) EQC_TRY(ds_exchange_raw(*r, g, T, maxband));
      EQC_TRY(T.end());
    } else {
      for (RankState *r : ranks) EQC_TRY(ds_encode(*r, g, s));
      EQC_TRY(T.start());
      for (RankState *r : ranks) EQC_TRY(ds_exchange_sizes(*r, g, T));
      EQC_TRY(T.end());
      for (RankState *r : ranks) {
        EQC_CUDA_TRY(cudaMemcpyAsync(r->h_sizes, r->sizes.p, 4 * g.n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      }
      EQC_CUDA_TRY(cudaStreamSynchronize(s));
      EQC_TRY(T.start());
      for (RankState *r : ranks) EQC_TRY(ds_exchange_rle(*r, g, T, cap));
      EQC_TRY(T.end());
      for (RankState *r : ranks) EQC_TRY(ds_decode(*r, g, maxband, cap, s));
    }
  }
  for (RankState *r : ranks) EQC_TRY(ds_band_composite(*r, g, maxband, s));
  auto region = [&](int q, int &y0, int &y1) {
    y0 = g.row0[q];
    y1 = g.row0[q + 1];
  };
  if (g.n > 1) {
    EQC_TRY(T.start());
    for (RankState *r : ranks) EQC_TRY(gather(*r, g, T, region, r->fin_c.as<uint32_t>(), s, 0));
    EQC_TRY(T.end());
    for (RankState *r : ranks) EQC_TRY(gather(*r, g, T, region, r->fin_c.as<uint32_t>(), s, 1));
  }
  return EQC_OK;
}

int bs_alloc(RankState &r, const Geometry &g) {
  const int half = (g.h + 1) / 2;
  EQC_TRY(alloc_common(r, g, std::max(half, g.out_pitch != g.w && r.rank == g.dest ? g.h : 0),
                       g.op != EQC_OP_DEPTH ? half : 1, 2));
  if (g.flags & EQC_FLAG_RLE) {
    const int64_t cap = band_cap(g, half);
    EQC_TRY(r.enc.ensure((size_t)2 * cap));
    EQC_TRY(r.dec.ensure((size_t)2 * cap));
    EQC_TRY(r.sizes.ensure((size_t)4 * sizeof(int64_t)));
    EQC_TRY(r.ws.ensure_zeroed(image_rle_workspace_size_batch(2, g.w, std::max(1, half))));
  }
  return EQC_OK;
}

// ---- c5: display-wall tiles (display segments and the
// wall's channels) -------------------------------------
// Direct send over the wall's tiles instead of row bands: tile t (row-major,
// tiles_x x tiles_y, edges at floor(k w / tiles_x), floor(k h / tiles_y)) is
// owned by rank floor(t n / T) (the channel driving that display);
// every rank pre-composites its sources, ships each tile of its partial wall
// (RLE streams with EQC_FLAG_RLE, else raw rectangles) to the tile's owner,
// and the owner composites the n partial tiles into its frame -- no gather.
struct TileRect {
  int x0, y0, w, h, owner;
};

TileRect plan_tile(int w, int h, int tx, int ty, int n, int t) {
  const int col = t % tx, row = t / tx;
  TileRect r;
  r.x0 = (int)((int64_t)col * w / tx);
  r.w = (int)((int64_t)(col + 1) * w / tx) - r.x0;
  r.y0 = (int)((int64_t)row * h / ty);
  r.h = (int)((int64_t)(row + 1) * h / ty) - r.y0;
  r.owner = (int)((int64_t)t * n / ((int64_t)tx * ty));
  return r;
}

int run_tiles(std::vector<RankState *> &ranks, Geometry &g, Transport &T, cudaStream_t s, int tx, int ty) {
  const int nt = tx * ty, n = g.n;
  const bool rle = (g.flags & EQC_FLAG_RLE) != 0;
  std::vector<TileRect> tr(nt);
  int twm = 0, thm = 0;
  for (int t = 0; t < nt; ++t) {
    tr[t] = plan_tile(g.w, g.h, tx, ty, n, t);
    twm = std::max(twm, tr[t].w);
    thm = std::max(thm, tr[t].h);
  }
  // stream / rectangle slot bytes (8-byte aligned streams: 256-byte slots)
  const int64_t cap = rle ? ((image_rle_max_size(twm, thm) + 255) & ~(int64_t)255) : (int64_t)twm * thm * 4;
  auto owned = [&](int r, int &t0, int &t1) {
    t0 = nt;
    t1 = nt;
    for (int t = 0; t < nt; ++t)
      if (tr[t].owner == r) {
        if (t0 == nt) t0 = t;
        t1 = t + 1;
      }
    if (t0 == nt) t0 = t1 = 0;
  };
  // (1) pre-composite; (2) every tile of the partial wall into its slot
  for (RankState *r : ranks) {
    for (int i = 0; i < 4; ++i) r->stats[i] = 0;
    EQC_TRY(r->part_c[0].ensure(frame_bytes(g, g.h)));
    EQC_TRY(r->part_d[0].ensure(frame_bytes(g, g.h)));
    EQC_TRY(local_precomposite(*r, g, s));
    EQC_TRY(r->enc.ensure((size_t)(2 * nt) * cap));
    EQC_TRY(r->sizes.ensure(((size_t)n * 2 * nt + 64) * sizeof(int64_t)));  // + batch-order sizes
    EQC_TRY(r->status.ensure_zeroed(sizeof(int32_t)));
    const uint32_t *pc = r->part_c[0].as<uint32_t>(), *pd = r->part_d[0].as<uint32_t>();
    if (rle) {
      // batches of <= 32 tiles of one size (64 streams: colour swizzled + depth)
      std::vector<int> done(nt, 0);
      for (int t0 = 0; t0 < nt; ++t0) {
        if (done[t0]) continue;
        std::vector<int> batch;
        for (int t = t0; t < nt && (int)batch.size() < 32; ++t)
          if (!done[t] && tr[t].w == tr[t0].w && tr[t].h == tr[t0].h) {
            batch.push_back(t);
            done[t] = 1;
          }
        const int bw = tr[t0].w, bh = tr[t0].h, cnt = (int)batch.size();
        std::vector<const uint32_t *> src(2 * cnt);
        std::vector<uint8_t *> dst(2 * cnt);
        std::vector<int> kinds(2 * cnt), fl(2 * cnt);
        for (int i = 0; i < cnt; ++i) {
          const TileRect &q = tr[batch[i]];
          const size_t off = (size_t)q.y0 * g.w + q.x0;
          src[i] = pc + off;
          src[cnt + i] = pd + off;
          dst[i] = r->enc.as<uint8_t>() + (size_t)(2 * batch[i]) * cap;
          dst[cnt + i] = r->enc.as<uint8_t>() + (size_t)(2 * batch[i] + 1) * cap;
          kinds[i] = EQC_KIND_RGBA8, fl[i] = EQC_FLAG_SWIZZLE;
          kinds[cnt + i] = EQC_KIND_DEPTH32, fl[cnt + i] = 0;
        }
        const size_t wsb = image_rle_workspace_size_batch(2 * cnt, bw, bh);
        EQC_TRY(r->ws.ensure(wsb));
        // sizes land in batch order after the size rows, then move to the
        // rank's own row ([2t] colour, [2t+1] depth)
        int64_t *dsz = r->sizes.as<int64_t>() + (size_t)r->rank * 2 * nt;
        int64_t *bsz = r->sizes.as<int64_t>() + (size_t)n * 2 * nt;
        EQC_TRY(image_compress_rle_batch(2 * cnt, src.data(), bw, bh, g.w, kinds.data(), fl.data(), dst.data(), cap,
                                         bsz, r->ws.p, wsb, s));
        for (int i = 0; i < cnt; ++i) {
          EQC_CUDA_TRY(cudaMemcpyAsync(dsz + 2 * batch[i], bsz + i, 8, cudaMemcpyDeviceToDevice, s));
          EQC_CUDA_TRY(cudaMemcpyAsync(dsz + 2 * batch[i] + 1, bsz + cnt + i, 8, cudaMemcpyDeviceToDevice, s));
        }
      }
    } else {
      for (int t = 0; t < nt; ++t) {  // pack each tile rectangle (pitch tile width)
        const TileRect &q = tr[t];
        const size_t off = (size_t)q.y0 * g.w + q.x0;
        EQC_CUDA_TRY(cudaMemcpy2DAsync(r->enc.as<uint8_t>() + (size_t)(2 * t) * cap, (size_t)q.w * 4, pc + off,
                                       (size_t)g.w * 4, (size_t)q.w * 4, q.h, cudaMemcpyDeviceToDevice, s));
        EQC_CUDA_TRY(cudaMemcpy2DAsync(r->enc.as<uint8_t>() + (size_t)(2 * t + 1) * cap, (size_t)q.w * 4, pd + off,
                                       (size_t)g.w * 4, (size_t)q.w * 4, q.h, cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  // (3) RLE: every rank's stream sizes to every rank, read back (one sync)
  std::vector<std::vector<int64_t>> hs(ranks.size());
  if (rle) {
    if (n > 1) {
      EQC_TRY(T.start());
      for (RankState *r : ranks) {
        int64_t *row = r->sizes.as<int64_t>();
        for (int q = 0; q < n; ++q) {
          if (q == r->rank) continue;
          EQC_TRY(T.send(*r, q, row + (size_t)r->rank * 2 * nt, 2 * nt * sizeof(int64_t)));
          EQC_TRY(T.recv(*r, q, row + (size_t)q * 2 * nt, 2 * nt * sizeof(int64_t)));
        }
      }
      EQC_TRY(T.end());
    }
    for (size_t i = 0; i < ranks.size(); ++i) {
      hs[i].resize((size_t)n * 2 * nt);
      EQC_CUDA_TRY(cudaMemcpyAsync(hs[i].data(), ranks[i]->sizes.p, hs[i].size() * 8, cudaMemcpyDeviceToHost, s));
    }
    EQC_CUDA_TRY(cudaStreamSynchronize(s));
  }
  auto bytes_of = [&](size_t ri, int q, int t, int k) -> size_t {
    return rle ? (size_t)hs[ri][(size_t)q * 2 * nt + 2 * t + k] : (size_t)tr[t].w * tr[t].h * 4;
  };
  // (4) tile payloads to their owners
  for (RankState *r : ranks) {
    int t0, t1;
    owned(r->rank, t0, t1);
    EQC_TRY(r->dec.ensure((size_t)std::max(1, (t1 - t0) * n * 2) * cap));
  }
  if (n > 1) {
    EQC_TRY(T.start());
    for (size_t ri = 0; ri < ranks.size(); ++ri) {
      RankState &r = *ranks[ri];
      for (int t = 0; t < nt; ++t) {
        const int o = tr[t].owner;
        if (o == r.rank) continue;
        EQC_TRY(T.send(r, o, r.enc.as<uint8_t>() + (size_t)(2 * t) * cap, bytes_of(ri, r.rank, t, 0)));
        EQC_TRY(T.send(r, o, r.enc.as<uint8_t>() + (size_t)(2 * t + 1) * cap, bytes_of(ri, r.rank, t, 1)));
        r.stats[0] += 1;
      }
      int t0, t1;
      owned(r.rank, t0, t1);
      for (int t = t0; t < t1; ++t)
        for (int q = 0; q < n; ++q) {
          if (q == r.rank) continue;
          uint8_t *slot = r.dec.as<uint8_t>() + (size_t)(((t - t0) * n + q) * 2) * cap;
          EQC_TRY(T.recv(r, q, slot, bytes_of(ri, q, t, 0)));
          EQC_TRY(T.recv(r, q, slot + cap, bytes_of(ri, q, t, 1)));
        }
    }
    EQC_TRY(T.end());
  }
  // (5) the owner composites its tiles, n partials in rank order (R-C5)
  for (RankState *r : ranks) {
    int t0, t1;
    owned(r->rank, t0, t1);
    for (int t = t0; t < t1; ++t) {
      const TileRect &q = tr[t];
      uint32_t *out = g.out + (size_t)q.y0 * g.out_pitch + q.x0;
      std::vector<const uint8_t *> cs(n), ds(n);
      for (int k = 0; k < n; ++k) {
        const uint8_t *base = k == r->rank ? r->enc.as<uint8_t>() + (size_t)(2 * t) * cap
                                           : r->dec.as<uint8_t>() + (size_t)(((t - t0) * n + k) * 2) * cap;
        cs[k] = base;
        ds[k] = base + cap;
      }
      if (rle) {
        const std::vector<int64_t> cb(n, cap), db(n, cap);
        EQC_TRY(compositor_depth_rle(n, cs.data(), ds.data(), cb.data(), db.data(), q.w, q.h, out, nullptr,
                                     g.out_pitch, r->status.as<int32_t>(), s));
      } else {
        std::vector<const uint32_t *> c(n), d(n);
        for (int k = 0; k < n; ++k) {
          c[k] = reinterpret_cast<const uint32_t *>(cs[k]);
          d[k] = reinterpret_cast<const uint32_t *>(ds[k]);
        }
        EQC_TRY(compositor_depth(n, c.data(), d.data(), q.w, q.h, q.w, out, nullptr, g.out_pitch, s));
      }
    }
  }
  return EQC_OK;
}

int run_binary_swap(std::vector<RankState *> &ranks, Geometry &g, Transport &T, cudaStream_t s) {
  std::vector<std::vector<BsRound>> plans(ranks.size());
  int k = 0;
  for (size_t i = 0; i < ranks.size(); ++i) {
    k = plan_bs(g.h, g.n, ranks[i]->rank, plans[i]);
    if (k < 0) return k;
  }
  const bool rle = (g.flags & EQC_FLAG_RLE) != 0;
  const int64_t cap = band_cap(g, (g.h + 1) / 2);
  for (RankState *r : ranks) {
    for (int i = 0; i < 4; ++i) r->stats[i] = 0;
    EQC_TRY(bs_alloc(*r, g));
    EQC_TRY(local_precomposite(*r, g, s));
  }
  for (int rd = 0; rd < k; ++rd) {
    if (rle) {
      for (size_t i = 0; i < ranks.size(); ++i) {
        RankState &r = *ranks[i];
        const BsRound &b = plans[i][rd];
        const int rows = b.send_y1 - b.send_y0;
        if (rows > 0) {
          const size_t off = (size_t)b.send_y0 * g.w;
          EQC_TRY(encode_band(r, g, 0, r.part_c[r.cur].as<uint32_t>() + off, r.part_d[r.cur].as<uint32_t>() + off,
                              rows, cap, s));
        }
      }
      EQC_TRY(T.start());
      for (size_t i = 0; i < ranks.size(); ++i) {
        RankState &r = *ranks[i];
        const BsRound &b = plans[i][rd];
        int64_t *sz = r.sizes.as<int64_t>();
        if (b.send_y1 > b.send_y0) EQC_TRY(T.send(r, b.partner, sz, 2 * sizeof(int64_t)));
        if (b.keep_y1 > b.keep_y0) EQC_TRY(T.recv(r, b.partner, sz + 2, 2 * sizeof(int64_t)));
      }
      EQC_TRY(T.end());
      for (RankState *r : ranks)
        EQC_CUDA_TRY(cudaMemcpyAsync(r->h_sizes, r->sizes.p, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      EQC_CUDA_TRY(cudaStreamSynchronize(s));
    }
    EQC_TRY(T.start());
    for (size_t i = 0; i < ranks.size(); ++i) {
      RankState &r = *ranks[i];
      const BsRound &b = plans[i][rd];
      const int srows = b.send_y1 - b.send_y0, krows = b.keep_y1 - b.keep_y0;
      if (srows > 0) {
        if (rle) {
          EQC_TRY(T.send(r, b.partner, r.enc.as<uint8_t>(), (size_t)r.h_sizes[0]));
          EQC_TRY(T.send(r, b.partner, r.enc.as<uint8_t>() + cap, (size_t)r.h_sizes[1]));
        } else {
          const size_t off = (size_t)b.send_y0 * g.w;
          EQC_TRY(T.send(r, b.partner, r.part_c[r.cur].as<uint32_t>() + off, frame_bytes(g, srows)));
          EQC_TRY(T.send(r, b.partner, r.part_d[r.cur].as<uint32_t>() + off, frame_bytes(g, srows)));
        }
        r.stats[0] += 1;
      }
      if (krows > 0) {
        if (rle) {
          EQC_TRY(T.recv(r, b.partner, r.dec.as<uint8_t>(), (size_t)r.h_sizes[2]));
          EQC_TRY(T.recv(r, b.partner, r.dec.as<uint8_t>() + cap, (size_t)r.h_sizes[3]));
        } else {
          EQC_TRY(T.recv(r, b.partner, r.recv_c.p, frame_bytes(g, krows)));
          EQC_TRY(T.recv(r, b.partner, r.recv_d.p, frame_bytes(g, krows)));
        }
      }
    }
    EQC_TRY(T.end());
    for (size_t i = 0; i < ranks.size(); ++i) {
      RankState &r = *ranks[i];
      const BsRound &b = plans[i][rd];
      const int krows = b.keep_y1 - b.keep_y0;
      if (krows <= 0) {
        r.cur ^= 1;
        continue;
      }
      if (rle) {
        const uint8_t *src[2] = {r.dec.as<uint8_t>(), r.dec.as<uint8_t>() + cap};
        uint32_t *dst[2] = {r.recv_c.as<uint32_t>(), r.recv_d.as<uint32_t>()};
        const int64_t caps[2] = {cap, cap};
        EQC_TRY(image_decompress_rle_batch(2, src, caps, dst, g.w, g.w, krows, r.status.as<int32_t>(), s));
      }
      const size_t off = (size_t)b.keep_y0 * g.w;
      const uint32_t *mine_c = r.part_c[r.cur].as<uint32_t>() + off, *mine_d = r.part_d[r.cur].as<uint32_t>() + off;
      const uint32_t *their_c = r.recv_c.as<uint32_t>(), *their_d = r.recv_d.as<uint32_t>();
      // ties go to the group whose bit r is 0 (lower global source indices)
      const uint32_t *c[2] = {b.low ? mine_c : their_c, b.low ? their_c : mine_c};
      const uint32_t *d[2] = {b.low ? mine_d : their_d, b.low ? their_d : mine_d};
      const int nxt = r.cur ^ 1;
      EQC_TRY(op_merge(g, 2, c, d, krows, r.part_c[nxt].as<uint32_t>() + off, r.part_d[nxt].as<uint32_t>() + off, s));
      r.cur = nxt;
    }
  }
  // gather final regions (colour) to the destination
  auto region = [&](int q, int &y0, int &y1) { final_region_bs(g.h, g.n, q, y0, y1); };
  // the final region's colour: the depth partial's colour plane, or the blend
  // partial rounded once to RGBA8 (over a transparent background) in fin_c
  auto final_colour = [&](RankState *r, int y0) -> const uint32_t * {
    return g.op != EQC_OP_DEPTH ? r->fin_c.as<uint32_t>() : r->part_c[r->cur].as<uint32_t>() + (size_t)y0 * g.w;
  };
  if (g.op != EQC_OP_DEPTH) {
    for (RankState *r : ranks) {
      int y0, y1;
      region(r->rank, y0, y1);
      if (y1 <= y0) continue;
      const size_t off = (size_t)y0 * g.w;
      const uint32_t *c[1] = {r->part_c[r->cur].as<uint32_t>() + off}, *d[1] = {r->part_d[r->cur].as<uint32_t>() + off};
      EQC_TRY(op_final(g, 1, c, d, y1 - y0, r->fin_c.as<uint32_t>(), g.w, s));
    }
  }
  for (RankState *r : ranks) {
    if (r->rank != g.dest) continue;
    int y0, y1;
    region(r->rank, y0, y1);
    if (y1 > y0)
      EQC_CUDA_TRY(cudaMemcpy2DAsync(g.out + (size_t)y0 * g.out_pitch, g.out_pitch * 4, final_colour(r, y0),
                                     (size_t)g.w * 4, (size_t)g.w * 4, y1 - y0, cudaMemcpyDeviceToDevice, s));
  }
  if (g.n > 1) {
    EQC_TRY(T.start());
    for (RankState *r : ranks) {
      int y0, y1;
      region(r->rank, y0, y1);
      EQC_TRY(gather(*r, g, T, region, final_colour(r, y0), s, 0));
    }
    EQC_TRY(T.end());
    for (RankState *r : ranks) {
      int y0, y1;
      region(r->rank, y0, y1);
      EQC_TRY(gather(*r, g, T, region, final_colour(r, y0), s, 1));
    }
  }
  return EQC_OK;
}

// ---- 2-3 swap ------------------------------------
// "an extension to binary swap, which overcomes the power-of-two source
// channel requirement by exchanging compositions between groups of two or
// three nodes in the compositing tree".  Reading R-C21: with m = the largest
// 2^a 3^b <= n and r = n - m, a fold step first pairs ranks (2i, 2i+1), i < r
// (group of two: 2i+1 sends its whole partial, 2i composites, lower ranks
// first); the m active ranks (in rank order: 0, 2, .., 2r-2, 2r, .., n-1)
// then run a mixed-radix swap with group sizes 2 (first) then 3: in a round of
// radix k, the active ranks whose active index differs only in that digit form
// a group, the current row region [y0, y1) splits into k parts at
// y0 + floor(u (y1 - y0) / k), the member with digit t keeps part t and
// receives it from the other members, and the k partials are composited in
// member (= rank = source) order.  For n = 2^a this is exactly binary swap.
struct S23Round {
  int k = 0, t = 0;
  int members[3] = {-1, -1, -1};
  int bnd[4] = {0, 0, 0, 0};  // part u = rows [bnd[u], bnd[u + 1])
};
struct S23Plan {
  int fold_role = 0;      // 0 none, 1 receives the partner's frame, 2 sends its frame (then idle)
  int fold_partner = -1;
  std::vector<S23Round> rounds;
  int fy0 = 0, fy1 = 0;   // final region (empty for a folded sender)
};

int plan_swap23(int h, int n, int rank, S23Plan &P) {
  if (n < 1 || rank < 0 || rank >= n || h < 1) return EQC_E_INVALID;
  P = S23Plan();
  int m = 1;
  for (int p2 = 1; p2 <= n; p2 *= 2)
    for (int v = p2; v <= n; v *= 3) m = std::max(m, v);
  std::vector<int> radix;
  for (int v = m; v % 2 == 0; v /= 2) radix.push_back(2);
  for (int v = m; v % 3 == 0; v /= 3) radix.push_back(3);
  const int r = n - m;
  std::vector<int> act;
  for (int i = 0; i < r; ++i) act.push_back(2 * i);
  for (int q = 2 * r; q < n; ++q) act.push_back(q);
  int a = -1;
  if (rank < 2 * r) {
    P.fold_role = (rank % 2 == 0) ? 1 : 2;
    P.fold_partner = rank ^ 1;
    if (P.fold_role == 2) return 0;  // contributes through its partner only
    a = rank / 2;
  } else {
    a = rank - r;
  }
  int y0 = 0, y1 = h, stride = 1;
  for (int k : radix) {
    S23Round rd;
    rd.k = k;
    rd.t = (a / stride) % k;
    const int base = a - rd.t * stride;
    for (int u = 0; u < k; ++u) rd.members[u] = act[base + u * stride];
    for (int u = 0; u <= k; ++u) rd.bnd[u] = y0 + (int)((int64_t)u * (y1 - y0) / k);
    P.rounds.push_back(rd);
    y0 = rd.bnd[rd.t];
    y1 = rd.bnd[rd.t + 1];
    stride *= k;
  }
  P.fy0 = y0;
  P.fy1 = y1;
  return (int)P.rounds.size();
}

int s23_alloc(RankState &r, const Geometry &g) {
  // part ping-pong buffers (full frame), two receive slots of up to h rows
  // (the fold moves a whole frame), final colour region of up to h rows
  EQC_TRY(alloc_common(r, g, (size_t)2 * g.h, g.op != EQC_OP_DEPTH ? g.h : 1, 2));
  if (g.flags & EQC_FLAG_RLE) {
    const int64_t cap = band_cap(g, g.h);
    EQC_TRY(r.enc.ensure((size_t)4 * cap));  // 2 outgoing parts x (c, d) streams
    EQC_TRY(r.dec.ensure((size_t)4 * cap));
    EQC_TRY(r.sizes.ensure((size_t)8 * sizeof(int64_t)));  // [0..3] sent, [4..7] received
    EQC_TRY(r.ws.ensure_zeroed(image_rle_workspace_size_batch(2, g.w, g.h)));
  }
  return EQC_OK;
}

// One exchange step of the 2-3 swap: every rank sends rows [y0, y1) of its
// live partial (both planes) to each peer in `sends` and receives `rows`
// rows from each peer in `recvs` into receive slot i (raw, or RLE streams
// after one size exchange).
struct S23Msg {
  int peer, y0, y1;
};
int s23_exchange(std::vector<RankState *> &ranks, const Geometry &g, Transport &T,
                 const std::vector<std::vector<S23Msg>> &sends, const std::vector<std::vector<S23Msg>> &recvs,
                 cudaStream_t s) {
  const bool rle = (g.flags & EQC_FLAG_RLE) != 0;
  const int64_t cap = band_cap(g, g.h);
  const size_t slot = (size_t)g.h * g.w;
  if (rle) {
    for (size_t i = 0; i < ranks.size(); ++i) {
      RankState &r = *ranks[i];
      for (size_t j = 0; j < sends[i].size(); ++j) {
        const S23Msg &m = sends[i][j];
        if (m.y1 <= m.y0) continue;
        const size_t off = (size_t)m.y0 * g.w;
        EQC_TRY(encode_band(r, g, (int)j, r.part_c[r.cur].as<uint32_t>() + off, r.part_d[r.cur].as<uint32_t>() + off,
                            m.y1 - m.y0, cap, s));
      }
    }
    EQC_TRY(T.start());
    for (size_t i = 0; i < ranks.size(); ++i) {
      RankState &r = *ranks[i];
      int64_t *sz = r.sizes.as<int64_t>();
      for (size_t j = 0; j < sends[i].size(); ++j)
        if (sends[i][j].y1 > sends[i][j].y0) EQC_TRY(T.send(r, sends[i][j].peer, sz + 2 * j, 2 * sizeof(int64_t)));
      for (size_t j = 0; j < recvs[i].size(); ++j)
        if (recvs[i][j].y1 > recvs[i][j].y0) EQC_TRY(T.recv(r, recvs[i][j].peer, sz + 4 + 2 * j, 2 * sizeof(int64_t)));
    }
    EQC_TRY(T.end());
    for (RankState *r : ranks)
      EQC_CUDA_TRY(cudaMemcpyAsync(r->h_sizes, r->sizes.p, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    EQC_CUDA_TRY(cudaStreamSynchronize(s));
  }
  EQC_TRY(T.start());
  for (size_t i = 0; i < ranks.size(); ++i) {
    RankState &r = *ranks[i];
    for (size_t j = 0; j < sends[i].size(); ++j) {
      const S23Msg &m = sends[i][j];
      if (m.y1 <= m.y0) continue;
      if (rle) {
        EQC_TRY(T.send(r, m.peer, r.enc.as<uint8_t>() + (size_t)(2 * j) * cap, (size_t)r.h_sizes[2 * j]));
        EQC_TRY(T.send(r, m.peer, r.enc.as<uint8_t>() + (size_t)(2 * j + 1) * cap, (size_t)r.h_sizes[2 * j + 1]));
      } else {
        const size_t off = (size_t)m.y0 * g.w;
        EQC_TRY(T.send(r, m.peer, r.part_c[r.cur].as<uint32_t>() + off, frame_bytes(g, m.y1 - m.y0)));
        EQC_TRY(T.send(r, m.peer, r.part_d[r.cur].as<uint32_t>() + off, frame_bytes(g, m.y1 - m.y0)));
      }
      r.stats[0] += 1;
    }
    for (size_t j = 0; j < recvs[i].size(); ++j) {
      const S23Msg &m = recvs[i][j];
      if (m.y1 <= m.y0) continue;
      if (rle) {
        EQC_TRY(T.recv(r, m.peer, r.dec.as<uint8_t>() + (size_t)(2 * j) * cap, (size_t)r.h_sizes[4 + 2 * j]));
        EQC_TRY(T.recv(r, m.peer, r.dec.as<uint8_t>() + (size_t)(2 * j + 1) * cap, (size_t)r.h_sizes[5 + 2 * j]));
      } else {
        EQC_TRY(T.recv(r, m.peer, r.recv_c.as<uint32_t>() + j * slot, frame_bytes(g, m.y1 - m.y0)));
        EQC_TRY(T.recv(r, m.peer, r.recv_d.as<uint32_t>() + j * slot, frame_bytes(g, m.y1 - m.y0)));
      }
    }
  }
  EQC_TRY(T.end());
  if (rle) {
    for (size_t i = 0; i < ranks.size(); ++i) {
      RankState &r = *ranks[i];
      for (size_t j = 0; j < recvs[i].size(); ++j) {
        const S23Msg &m = recvs[i][j];
        if (m.y1 <= m.y0) continue;
        const uint8_t *src[2] = {r.dec.as<uint8_t>() + (size_t)(2 * j) * cap,
                                 r.dec.as<uint8_t>() + (size_t)(2 * j + 1) * cap};
        uint32_t *dst[2] = {r.recv_c.as<uint32_t>() + j * slot, r.recv_d.as<uint32_t>() + j * slot};
        const int64_t caps[2] = {cap, cap};
        EQC_TRY(image_decompress_rle_batch(2, src, caps, dst, g.w, g.w, m.y1 - m.y0, r.status.as<int32_t>(), s));
      }
    }
  }
  return EQC_OK;
}

int run_swap23(std::vector<RankState *> &ranks, Geometry &g, Transport &T, cudaStream_t s) {
  std::vector<S23Plan> plans(ranks.size());
  for (size_t i = 0; i < ranks.size(); ++i) EQC_TRY(plan_swap23(g.h, g.n, ranks[i]->rank, plans[i]) < 0 ? EQC_E_INVALID : EQC_OK);
  for (RankState *r : ranks) {
    for (int i = 0; i < 4; ++i) r->stats[i] = 0;
    EQC_TRY(s23_alloc(*r, g));
    EQC_TRY(local_precomposite(*r, g, s));
  }
  const size_t slot = (size_t)g.h * g.w;
  // fold: groups of two, whole frames
  {
    std::vector<std::vector<S23Msg>> snd(ranks.size()), rcv(ranks.size());
    bool any = false;
    for (size_t i = 0; i < ranks.size(); ++i) {
      if (plans[i].fold_role == 2) snd[i].push_back(S23Msg{plans[i].fold_partner, 0, g.h});
      if (plans[i].fold_role == 1) rcv[i].push_back(S23Msg{plans[i].fold_partner, 0, g.h});
      any = any || plans[i].fold_role != 0;
    }
    if (any) {
      EQC_TRY(s23_exchange(ranks, g, T, snd, rcv, s));
      for (size_t i = 0; i < ranks.size(); ++i) {
        if (plans[i].fold_role != 1) continue;
        RankState &r = *ranks[i];
        const uint32_t *c[2] = {r.part_c[r.cur].as<uint32_t>(), r.recv_c.as<uint32_t>()};
        const uint32_t *d[2] = {r.part_d[r.cur].as<uint32_t>(), r.recv_d.as<uint32_t>()};
        const int nxt = r.cur ^ 1;
        EQC_TRY(op_merge(g, 2, c, d, g.h, r.part_c[nxt].as<uint32_t>(), r.part_d[nxt].as<uint32_t>(), s));
        r.cur = nxt;
      }
    }
  }
  size_t nrounds = 0;
  for (auto &P : plans) nrounds = std::max(nrounds, P.rounds.size());
  for (size_t rd = 0; rd < nrounds; ++rd) {
    std::vector<std::vector<S23Msg>> snd(ranks.size()), rcv(ranks.size());
    for (size_t i = 0; i < ranks.size(); ++i) {
      if (rd >= plans[i].rounds.size()) continue;
      const S23Round &R = plans[i].rounds[rd];
      for (int u = 0; u < R.k; ++u) {
        if (u == R.t) continue;
        snd[i].push_back(S23Msg{R.members[u], R.bnd[u], R.bnd[u + 1]});
        rcv[i].push_back(S23Msg{R.members[u], R.bnd[R.t], R.bnd[R.t + 1]});
      }
    }
    EQC_TRY(s23_exchange(ranks, g, T, snd, rcv, s));
    for (size_t i = 0; i < ranks.size(); ++i) {
      if (rd >= plans[i].rounds.size()) continue;
      RankState &r = *ranks[i];
      const S23Round &R = plans[i].rounds[rd];
      const int ky0 = R.bnd[R.t], rows = R.bnd[R.t + 1] - ky0;
      const int nxt = r.cur ^ 1;
      if (rows <= 0) {
        r.cur = nxt;
        continue;
      }
      const size_t off = (size_t)ky0 * g.w;
      // members in rank order; slot j holds the j-th other member's part
      const uint32_t *c[3], *d[3];
      for (int u = 0, j = 0; u < R.k; ++u) {
        if (u == R.t) {
          c[u] = r.part_c[r.cur].as<uint32_t>() + off;
          d[u] = r.part_d[r.cur].as<uint32_t>() + off;
        } else {
          c[u] = r.recv_c.as<uint32_t>() + (size_t)j * slot;
          d[u] = r.recv_d.as<uint32_t>() + (size_t)j * slot;
          ++j;
        }
      }
      uint32_t *oc = r.part_c[nxt].as<uint32_t>() + off, *od = r.part_d[nxt].as<uint32_t>() + off;
      EQC_TRY(op_merge(g, R.k, c, d, rows, oc, od, s));
      r.cur = nxt;
    }
  }
  // final regions -> colour -> destination
  auto region = [&](int q, int &y0, int &y1) {
    S23Plan P;
    plan_swap23(g.h, g.n, q, P);
    y0 = P.fy0;
    y1 = P.fy1;
  };
  auto final_colour = [&](RankState *r, int y0) -> const uint32_t * {
    return g.op != EQC_OP_DEPTH ? r->fin_c.as<uint32_t>() : r->part_c[r->cur].as<uint32_t>() + (size_t)y0 * g.w;
  };
  for (RankState *r : ranks) {
    int y0, y1;
    region(r->rank, y0, y1);
    if (y1 <= y0) continue;
    if (g.op != EQC_OP_DEPTH) {
      const size_t off = (size_t)y0 * g.w;
      const uint32_t *c[1] = {r->part_c[r->cur].as<uint32_t>() + off}, *d[1] = {r->part_d[r->cur].as<uint32_t>() + off};
      EQC_TRY(op_final(g, 1, c, d, y1 - y0, r->fin_c.as<uint32_t>(), g.w, s));
    }
    if (r->rank == g.dest)
      EQC_CUDA_TRY(cudaMemcpy2DAsync(g.out + (size_t)y0 * g.out_pitch, g.out_pitch * 4, final_colour(r, y0),
                                     (size_t)g.w * 4, (size_t)g.w * 4, y1 - y0, cudaMemcpyDeviceToDevice, s));
  }
  if (g.n > 1) {
    EQC_TRY(T.start());
    for (RankState *r : ranks) {
      int y0, y1;
      region(r->rank, y0, y1);
      EQC_TRY(gather(*r, g, T, region, final_colour(r, y0), s, 0));
    }
    EQC_TRY(T.end());
    for (RankState *r : ranks) {
      int y0, y1;
      region(r->rank, y0, y1);
      EQC_TRY(gather(*r, g, T, region, final_colour(r, y0), s, 1));
    }
  }
  return EQC_OK;
}

// ---- streaming sort-last chain --------------------
// "The output of one source channel is copied to the next channel in the
// chain, which then composites it on top of its own rendering, streaming the
// combined frame on to the next source.  At the end of the chain, the
// destination channel completes the input frame".  Rank k receives the
// partial of ranks 0..k-1 (whole frame; raw or RLE), merges it with its own
// partial (received = lower ranks = back first) and passes it on; rank n-1
// finishes the frame and sends the colour to dest_rank.  Latency
// t_local + (n - 1) (t_transfer + t_merge).
int run_stream(std::vector<RankState *> &ranks, Geometry &g, Transport &T, cudaStream_t s) {
  for (RankState *r : ranks) {
    for (int i = 0; i < 4; ++i) r->stats[i] = 0;
    EQC_TRY(s23_alloc(*r, g));
    EQC_TRY(r->fin_c.ensure(frame_bytes(g, g.h)));
    EQC_TRY(local_precomposite(*r, g, s));
  }
  for (int hop = 0; hop + 1 < g.n; ++hop) {
    std::vector<std::vector<S23Msg>> snd(ranks.size()), rcv(ranks.size());
    for (size_t i = 0; i < ranks.size(); ++i) {
      if (ranks[i]->rank == hop) snd[i].push_back(S23Msg{hop + 1, 0, g.h});
      if (ranks[i]->rank == hop + 1) rcv[i].push_back(S23Msg{hop, 0, g.h});
    }
    EQC_TRY(s23_exchange(ranks, g, T, snd, rcv, s));
    for (RankState *r : ranks) {
      if (r->rank != hop + 1) continue;
      const uint32_t *c[2] = {r->recv_c.as<uint32_t>(), r->part_c[r->cur].as<uint32_t>()};
      const uint32_t *d[2] = {r->recv_d.as<uint32_t>(), r->part_d[r->cur].as<uint32_t>()};
      const int nxt = r->cur ^ 1;
      EQC_TRY(op_merge(g, 2, c, d, g.h, r->part_c[nxt].as<uint32_t>(), r->part_d[nxt].as<uint32_t>(), s));
      r->cur = nxt;
    }
  }
  // the end of the chain completes the frame; its colour goes to the destination
  const int last = g.n - 1;
  const uint32_t *col_last = nullptr;
  for (RankState *r : ranks) {
    if (r->rank != last) continue;
    col_last = r->part_c[r->cur].as<uint32_t>();
    if (g.op != EQC_OP_DEPTH) {
      const uint32_t *c[1] = {r->part_c[r->cur].as<uint32_t>()}, *d[1] = {r->part_d[r->cur].as<uint32_t>()};
      EQC_TRY(op_final(g, 1, c, d, g.h, r->fin_c.as<uint32_t>(), g.w, s));
      col_last = r->fin_c.as<uint32_t>();
    }
  }
  if (last != g.dest) {  // every rank takes part in the (possibly empty) message group
    EQC_TRY(T.start());
    for (RankState *r : ranks) {
      if (r->rank == last) {
        EQC_TRY(T.send(*r, g.dest, col_last, frame_bytes(g, g.h)));
        r->stats[1] += 1;
      }
      if (r->rank == g.dest) EQC_TRY(T.recv(*r, last, r->fin_c.as<uint32_t>(), frame_bytes(g, g.h)));
    }
    EQC_TRY(T.end());
  }
  for (RankState *r : ranks) {
    if (r->rank != g.dest) continue;
    const uint32_t *col = last == g.dest ? col_last : r->fin_c.as<uint32_t>();
    EQC_CUDA_TRY(cudaMemcpy2DAsync(g.out, g.out_pitch * 4, col, (size_t)g.w * 4, (size_t)g.w * 4, g.h,
                                   cudaMemcpyDeviceToDevice, s));
  }
  return EQC_OK;
}

int validate(int nranks, int n_local, const void *color, const void *depth, int w, int h, int64_t pitch, int op,
             int flags, int dest, const void *out, int64_t out_pitch, bool is_dest) {
  if (nranks < 1 || n_local < 1 || n_local > EQC_MAX_SOURCES || nranks > EQC_MAX_SOURCES) return EQC_E_INVALID;
  if (op != EQC_OP_DEPTH && op != EQC_OP_BLEND && op != EQC_OP_AVERAGE) return EQC_E_UNSUPPORTED;
  if (op == EQC_OP_AVERAGE && (int64_t)nranks * n_local > 256) return EQC_E_UNSUPPORTED;  // 16-bit sums
  if (!color || (op == EQC_OP_DEPTH && !depth) || w <= 0 || h <= 0 || pitch < w) return EQC_E_INVALID;
  if (flags & ~(EQC_FLAG_RLE | EQC_FLAG_NCCL | EQC_FLAG_ROI | EQC_FLAG_OVERLAP)) return EQC_E_INVALID;
  if (dest < 0 || dest >= nranks) return EQC_E_INVALID;
  if (is_dest && (!out || out_pitch < w)) return EQC_E_INVALID;
  return EQC_OK;
}

}  // namespace

// ---- peer-memory (NVLink P2P) direct send ------------------------------------
//
// The exchange and the band composite are one kernel: rank j's band-composite
// launch reads band j of every peer's partial frame straight out of the
// peer's HBM over NVLink (CUDA IPC mappings) and writes the composited band
// straight into the destination's frame buffer (peer stores), so the bytes
// cross NVLink once and are never staged.  Two flag barriers (peer-memory
// release/acquire) order the steps: partials complete before peers read them,
// bands complete before the destination copies them out.
namespace {

// The IPC-exposed `flags` allocation holds the barrier flags (EQC_MAX_SOURCES
// ints), the rank's partial-frame ROI {x, y, w, h} (kRoiSlot), the progress
// counter of its pipelined pre-composite (kProgSlot), a local error word
// (kErrSlot: bit 0 a flag wait timed out, bit 1 the ranks passed different
// frame slots) and the frame slot this rank's call passed (kSlotSlot).
constexpr int kRoiSlot = EQC_MAX_SOURCES;  // int offset, 16-byte aligned
constexpr int kProgSlot = kRoiSlot + 4;
constexpr int kErrSlot = kProgSlot + 4;
constexpr int kSlotSlot = kErrSlot + 1;
constexpr int kFlagInts = kErrSlot + 4;
constexpr int kErrTimeout = 1, kErrSlotMismatch = 2;

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *f - target >= 0 (acquire, system scope) or the deadline passes
// (then the timeout bit goes into *err): a dead or stalled peer cannot hang
// the GPU; eqc_comm_check reports it.
__device__ __forceinline__ void wait_flag(const int *f, int target, int64_t timeout_ns, int *err, int sleep_ns) {
  const uint64_t t0 = global_ns();
  int v;
  while (true) {
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (v - target >= 0) break;
    if ((int64_t)(global_ns() - t0) > timeout_ns) {
      atomicOr(err, kErrTimeout);
      break;
    }
    __nanosleep(sleep_ns);
  }
}

struct BarrierArgs {
  int *peer_flags[EQC_MAX_SOURCES];  // flags array of every rank (own = local)
  int *my_flags;
  int n, rank, epoch;
  int check_slot, slot;  // publish this call's frame slot and check every rank passed the same one
  int64_t timeout_ns;
};

__global__ void p2p_barrier_kernel(const __grid_constant__ BarrierArgs a) {
  const int i = threadIdx.x;
  if (a.check_slot && i == 0) a.my_flags[kSlotSlot] = a.slot;
  __syncthreads();
  __threadfence_system();
  if (i < a.n) {
    int *f = a.peer_flags[i] + a.rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(a.epoch) : "memory");
  }
  if (i < a.n) {
    wait_flag(a.my_flags + i, a.epoch, a.timeout_ns, a.my_flags + kErrSlot, 64);
    if (a.check_slot && !(*(volatile int *)(a.my_flags + kErrSlot) & kErrTimeout)) {
      int v;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(a.peer_flags[i] + kSlotSlot) : "memory");
      if (v != a.slot) atomicOr(a.my_flags + kErrSlot, kErrSlotMismatch);
    }
  }
  __syncthreads();
}

#ifndef EQC_P2P_PIECES
#define EQC_P2P_PIECES 2  // pieces per band of the pipelined peer-memory direct send
#endif
#ifndef EQC_P2P_AUX_PRIO
#define EQC_P2P_AUX_PRIO 0  // 1: pulling stream at the highest priority (measured no better)
#endif

// Pipelined direct send: the owner publishes "pieces 0..k of every band of my
// partial frame are complete" as a monotonic counter in its own flags page
// (release, system scope) ...
__global__ void p2p_signal_kernel(int *my_flags, int value) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(my_flags + kProgSlot), "r"(value) : "memory");
  }
}

struct WaitArgs {
  const int *peer_flags[EQC_MAX_SOURCES];
  int *err;
  int n, target;
  int64_t timeout_ns;
};

// ... and a puller waits until every rank's counter reached the piece
// (acquire, system scope, polling peer memory over NVLink).
__global__ void p2p_wait_kernel(const __grid_constant__ WaitArgs a) {
  const int i = threadIdx.x;
  if (i < a.n) wait_flag(a.peer_flags[i] + kProgSlot, a.target, a.timeout_ns, a.err, 32);
  __syncthreads();
}

// Bounding box of the union of n ROIs {x, y, w, h} (empty ones ignored),
// clipped by the consumer: the ROI of a partial frame whose sources hold data
// only inside their (application-provided) ROIs.
__global__ void roi_union_kernel(const int32_t *in, int n, int32_t *out) {
  if (threadIdx.x != 0) return;
  int64_t x0 = INT64_MAX, y0 = INT64_MAX, x1 = INT64_MIN, y1 = INT64_MIN;
  for (int i = 0; i < n; ++i) {
    const int4 r = reinterpret_cast<const int4 *>(in)[i];
    if (r.z <= 0 || r.w <= 0) continue;
    x0 = min(x0, (int64_t)r.x);
    y0 = min(y0, (int64_t)r.y);
    x1 = max(x1, (int64_t)r.x + r.z);
    y1 = max(y1, (int64_t)r.y + r.w);
  }
  x0 = max(x0, (int64_t)INT32_MIN);
  y0 = max(y0, (int64_t)INT32_MIN);
  *reinterpret_cast<int4 *>(out) = x1 == INT64_MIN ? make_int4(0, 0, 0, 0)
                                                  : make_int4((int)x0, (int)y0, (int)min(x1 - x0, (int64_t)INT32_MAX),
                                                              (int)min(y1 - y0, (int64_t)INT32_MAX));
}

inline int64_t p2p_timeout_ns() {
  const char *e = getenv("EQC_P2P_TIMEOUT_MS");
  const long long ms = e ? atoll(e) : 60000;
  return (int64_t)(ms > 0 ? ms : 60000) * 1000000;
}

struct P2PState {
  int capable = -1;  // -1 unknown, 0 no (NCCL transport), 1 yes
  int64_t timeout_ns = p2p_timeout_ns();  // flag waits give up after this (EQC_P2P_TIMEOUT_MS, default 60 s)
  bool skip_barriers = false;  // test hook of the virtual-rank executor: this rank never arrives
  int64_t cap_px = 0;
  int prog = 0;                    // this rank's published progress counter
  cudaStream_t aux = nullptr;      // pulling stream of the pipelined direct send
  cudaEvent_t ev_start = nullptr, ev_pulled = nullptr;
  DevBuf part_c, part_d, fin_c, flags, xfer, roi_local;
  std::vector<uint32_t *> peer_part_c, peer_part_d, peer_fin_c;
  std::vector<int *> peer_flags;
  int epoch = 0;
  // caller-visible, peer-mapped frame slots (eqc_comm_frame_buffers): a
  // partial frame rendered / decoded straight into slot i is read by the
  // peers in place (no pre-composite copy)
  static constexpr int kSlots = 2;
  int64_t slot_px = 0;
  DevBuf slot_c[kSlots], slot_d[kSlots];
  std::vector<uint32_t *> peer_slot_c[kSlots], peer_slot_d[kSlots];

  // caller-visible, peer-mapped RLE stream slots (eqc_comm_stream_buffers):
  // slot i holds sn streams of scap bytes each, contiguous
  int sn = 0;
  int64_t scap = 0;
  DevBuf sslot[kSlots];
  std::vector<uint8_t *> peer_sslot[kSlots];

  // slot of (color, depth) when they are exactly slot i's buffers, else -1
  int slot_of(const uint32_t *color, const uint32_t *depth) const {
    for (int i = 0; i < kSlots; ++i)
      if (slot_c[i].p && color == slot_c[i].as<uint32_t>() && depth == slot_d[i].as<uint32_t>()) return i;
    return -1;
  }
  void close_slots(int rank) {
    for (int i = 0; i < kSlots; ++i) {
      for (size_t q = 0; q < peer_slot_c[i].size(); ++q) {
        if ((int)q == rank) continue;
        if (peer_slot_c[i][q]) cudaIpcCloseMemHandle(peer_slot_c[i][q]);
        if (peer_slot_d[i][q]) cudaIpcCloseMemHandle(peer_slot_d[i][q]);
      }
      peer_slot_c[i].clear();
      peer_slot_d[i].clear();
    }
  }
  void close_sslots(int rank) {
    for (int i = 0; i < kSlots; ++i) {
      for (size_t q = 0; q < peer_sslot[i].size(); ++q)
        if ((int)q != rank && peer_sslot[i][q]) cudaIpcCloseMemHandle(peer_sslot[i][q]);
      peer_sslot[i].clear();
    }
  }

  void close_peers(int rank) {
    for (size_t q = 0; q < peer_part_c.size(); ++q) {
      if ((int)q == rank) continue;
      if (peer_part_c[q]) cudaIpcCloseMemHandle(peer_part_c[q]);
      if (peer_part_d[q]) cudaIpcCloseMemHandle(peer_part_d[q]);
      if (peer_fin_c[q]) cudaIpcCloseMemHandle(peer_fin_c[q]);
      if (peer_flags[q]) cudaIpcCloseMemHandle(peer_flags[q]);
    }
    peer_part_c.clear();
    peer_part_d.clear();
    peer_fin_c.clear();
    peer_flags.clear();
  }
};

}  // namespace

// ---- communicator ---------------------------------------------------------------
struct eqc_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 1, rank = 0;
  RankState st;
  P2PState p2p;
};

namespace {

// Exchange the IPC handles of this rank's k allocations `ptrs` with every
// rank and open the peers' (collective).  out[i][q] = rank q's allocation i
// as mapped here (this rank's own pointer at q == rank).  `ok` is the
// all-rank AND of "every handle was created and opened".
int ipc_exchange(eqc_comm *c, void *const *ptrs, int k, std::vector<std::vector<void *>> &out, int &ok,
                 cudaStream_t s) {
  P2PState &P = c->p2p;
  const int n = c->nranks;
  constexpr int kH = sizeof(cudaIpcMemHandle_t);
  std::vector<uint8_t> mine((size_t)k * kH), all((size_t)n * k * kH);
  ok = 1;
  for (int i = 0; i < k; ++i) {
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, ptrs[i]) != cudaSuccess) ok = 0;
    std::memcpy(mine.data() + (size_t)i * kH, &h, kH);
  }
  EQC_TRY(P.xfer.ensure((size_t)(n + 1) * k * kH + 64));
  uint8_t *dx = P.xfer.as<uint8_t>();
  EQC_CUDA_TRY(cudaMemcpyAsync(dx, mine.data(), mine.size(), cudaMemcpyHostToDevice, s));
  EQC_NCCL_TRY(ncclAllGather(dx, dx + mine.size(), mine.size(), ncclUint8, c->nccl, s));
  EQC_CUDA_TRY(cudaMemcpyAsync(all.data(), dx + mine.size(), all.size(), cudaMemcpyDeviceToHost, s));
  EQC_CUDA_TRY(cudaStreamSynchronize(s));
  out.assign(k, std::vector<void *>(n, nullptr));
  for (int q = 0; q < n && ok; ++q)
    for (int i = 0; i < k && ok; ++i) {
      if (q == c->rank) {
        out[i][q] = ptrs[i];
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, all.data() + ((size_t)q * k + i) * kH, kH);
      if (cudaIpcOpenMemHandle(&out[i][q], h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        out[i][q] = nullptr;
        ok = 0;
      }
    }
  cudaGetLastError();  // a failed open is reported through `ok`
  // agree on the transport: P2P only if every rank mapped every peer
  int *dok = reinterpret_cast<int *>(dx);
  EQC_CUDA_TRY(cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
  EQC_NCCL_TRY(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c->nccl, s));
  EQC_CUDA_TRY(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, s));
  EQC_CUDA_TRY(cudaStreamSynchronize(s));
  return EQC_OK;
}

int eqc_preload_kernels();

// (Re)build the IPC mappings for frames of `px` pixels.  Collective.
int p2p_setup(eqc_comm *c, int64_t px, cudaStream_t s) {
  P2PState &P = c->p2p;
  if (P.capable == 0) return EQC_OK;
  if (P.capable == 1 && px <= P.cap_px) return EQC_OK;
  EQC_TRY(eqc_preload_kernels());  // no lazy kernel load while a flag barrier spins
  cudaStreamSynchronize(s);
  P.close_peers(c->rank);
  const size_t bytes = (size_t)px * 4;
  EQC_TRY(P.part_c.ensure(bytes));
  EQC_TRY(P.part_d.ensure(bytes));
  EQC_TRY(P.fin_c.ensure(bytes));
  P.flags.release();
  EQC_TRY(P.flags.ensure_zeroed(kFlagInts * sizeof(int)));
  P.epoch = 0;
  P.prog = 0;
  void *ptrs[4] = {P.part_c.p, P.part_d.p, P.fin_c.p, P.flags.p};
  std::vector<std::vector<void *>> m;
  int ok = 0;
  EQC_TRY(ipc_exchange(c, ptrs, 4, m, ok, s));
  const int n = c->nranks;
  P.peer_part_c.assign(n, nullptr);
  P.peer_part_d.assign(n, nullptr);
  P.peer_fin_c.assign(n, nullptr);
  P.peer_flags.assign(n, nullptr);
  for (int q = 0; q < n; ++q) {
    P.peer_part_c[q] = (uint32_t *)m[0][q];
    P.peer_part_d[q] = (uint32_t *)m[1][q];
    P.peer_fin_c[q] = (uint32_t *)m[2][q];
    P.peer_flags[q] = (int *)m[3][q];
  }
  P.capable = ok ? 1 : 0;
  P.cap_px = ok ? px : 0;
  if (!ok) P.close_peers(c->rank);
  return EQC_OK;
}

// Caller-visible frame slots of >= px pixels, peer-mapped.  Collective.
int p2p_slots(eqc_comm *c, int64_t px, cudaStream_t s) {
  P2PState &P = c->p2p;
  if (px <= P.slot_px) return EQC_OK;
  cudaStreamSynchronize(s);
  P.close_slots(c->rank);
  P.slot_px = 0;
  void *ptrs[2 * P2PState::kSlots];
  for (int i = 0; i < P2PState::kSlots; ++i) {
    EQC_TRY(P.slot_c[i].ensure((size_t)px * 4));
    EQC_TRY(P.slot_d[i].ensure((size_t)px * 4));
    ptrs[2 * i] = P.slot_c[i].p;
    ptrs[2 * i + 1] = P.slot_d[i].p;
  }
  std::vector<std::vector<void *>> m;
  int ok = 0;
  EQC_TRY(ipc_exchange(c, ptrs, 2 * P2PState::kSlots, m, ok, s));
  for (int i = 0; i < P2PState::kSlots; ++i) {
    P.peer_slot_c[i].assign(c->nranks, nullptr);
    P.peer_slot_d[i].assign(c->nranks, nullptr);
    for (int q = 0; q < c->nranks; ++q) {
      P.peer_slot_c[i][q] = (uint32_t *)m[2 * i][q];
      P.peer_slot_d[i][q] = (uint32_t *)m[2 * i + 1][q];
    }
  }
  if (!ok) {
    P.close_slots(c->rank);
    return EQC_E_UNSUPPORTED;
  }
  P.slot_px = px;
  return EQC_OK;
}

int p2p_barrier(eqc_comm *c, cudaStream_t s, int check_slot = 0, int slot = -1) {
  P2PState &P = c->p2p;
  BarrierArgs a;
  for (int q = 0; q < c->nranks; ++q) a.peer_flags[q] = P.peer_flags[q];
  a.my_flags = P.flags.as<int>();
  a.n = c->nranks;
  a.rank = c->rank;
  a.epoch = ++P.epoch;
  a.check_slot = check_slot;
  a.slot = slot;
  a.timeout_ns = P.timeout_ns;
  if (P.skip_barriers) return EQC_OK;
  p2p_barrier_kernel<<<1, 64, 0, s>>>(a);
  return eqc_launch_status();
}

// Pipelined peer-memory direct send ("chunked out-of-order
// assembly overlapped with the exchange"): every
// band is cut into K pieces; the owner pre-composites piece k of every band
// and publishes its progress, while (on a second stream) each rank pulls
// piece k of its band from every peer as soon as all of them have published
// it -- the HBM-bound pre-composite of piece k+1 overlaps the NVLink-bound
// pull + composite of piece k.  Used without EQC_FLAG_ROI (a computed ROI is
// only known after the whole pre-composite); application ROIs are fine.
int direct_send_p2p_pipelined(eqc_comm *c, const Geometry &g, const uint32_t *const *color,
                              const uint32_t *const *depth, cudaStream_t s) {
  P2PState &P = c->p2p;
  const int n = c->nranks, me = c->rank, K = EQC_P2P_PIECES;
  int64_t *stats = c->st.stats;
  for (int i = 0; i < 4; ++i) stats[i] = 0;
  std::vector<int> row0(n + 1);
  plan_bands_gather(g.h, n, g.dest, row0.data());
  auto piece = [&](int j, int k, int &y0, int &y1) {
    const int len = row0[j + 1] - row0[j];
    y0 = row0[j] + (int)((int64_t)k * len / K);
    y1 = row0[j] + (int)((int64_t)(k + 1) * len / K);
  };
  if (!P.aux) {
    // highest priority: the pulls are NVLink-bound and should take SMs as soon
    // as a piece is published, ahead of the pending CTAs of the next piece's
    // (HBM-bound) pre-composite
    int lo = 0, hi = 0;
    EQC_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    EQC_CUDA_TRY(cudaStreamCreateWithPriority(&P.aux, cudaStreamNonBlocking, EQC_P2P_AUX_PRIO ? hi : lo));
    EQC_CUDA_TRY(cudaEventCreateWithFlags(&P.ev_start, cudaEventDisableTiming));
    EQC_CUDA_TRY(cudaEventCreateWithFlags(&P.ev_pulled, cudaEventDisableTiming));
  }
  const bool app_roi = g.src_roi && g.op == EQC_OP_DEPTH;
  int32_t *my_roi = P.flags.as<int32_t>() + kRoiSlot;
  std::vector<const int32_t *> src_rp(g.n_local);
  if (app_roi) {
    roi_union_kernel<<<1, 32, 0, s>>>(g.src_roi, g.n_local, my_roi);
    EQC_TRY(eqc_launch_status());
    for (int i = 0; i < g.n_local; ++i) src_rp[i] = g.src_roi + 4 * i;
  }
  // the pulls write the caller's frame (on dest): order them after its prior work
  EQC_CUDA_TRY(cudaEventRecord(P.ev_start, s));
  EQC_CUDA_TRY(cudaStreamWaitEvent(P.aux, P.ev_start, 0));
  const int base = P.prog;
  std::vector<const uint32_t *> cs(g.n_local), ds(g.n_local);
  // EQC_P2P_TRACE=1: per-phase GPU times of this call on stderr (debug; syncs)
  static const bool trace = getenv("EQC_P2P_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  mark(s);
  for (int k = 0; k < K; ++k) {
    // (1) piece k of every band of my partial frame
    for (int j = 0; j < n; ++j) {
      int y0, y1;
      piece(j, k, y0, y1);
      if (y1 <= y0) continue;
      const size_t so = (size_t)y0 * g.pitch, po = (size_t)y0 * g.w;
      for (int i = 0; i < g.n_local; ++i) {
        cs[i] = color[i] + so;
        ds[i] = depth ? depth[i] + so : nullptr;
      }
      uint32_t *pc = P.part_c.as<uint32_t>() + po, *pd = P.part_d.as<uint32_t>() + po;
      if (app_roi) {
        EQC_TRY(eqc_depth_roi_launch(g.n_local, cs.data(), ds.data(), src_rp.data(), y0, my_roi, g.w, y1 - y0,
                                     g.pitch, pc, pd, g.w, s));
      } else if (g.op == EQC_OP_BLEND) {
        EQC_TRY(eqc_blend_to_partial(g.n_local, cs.data(), g.w, y1 - y0, g.pitch, pc, pd, g.w, s));
      } else if (g.op == EQC_OP_AVERAGE) {
        EQC_TRY(eqc_average(true, g.n_local, cs.data(), nullptr, g.w, y1 - y0, g.pitch, g.n * g.n_local, nullptr,
                            pc, pd, g.w, s));
      } else {
        EQC_TRY(compositor_depth(g.n_local, cs.data(), ds.data(), g.w, y1 - y0, g.pitch, pc, pd, g.w, s));
      }
    }
    p2p_signal_kernel<<<1, 32, 0, s>>>(P.flags.as<int>(), base + k + 1);
    EQC_TRY(eqc_launch_status());
    mark(s);
    // (2)-(4) on the pulling stream: wait for piece k everywhere, pull + composite it
    WaitArgs wa;
    for (int q = 0; q < n; ++q) wa.peer_flags[q] = P.peer_flags[q];
    wa.err = P.flags.as<int>() + kErrSlot;
    wa.n = n;
    wa.target = base + k + 1;
    wa.timeout_ns = P.timeout_ns;
    p2p_wait_kernel<<<1, 64, 0, P.aux>>>(wa);
    EQC_TRY(eqc_launch_status());
    mark(P.aux);
    int y0, y1;
    piece(me, k, y0, y1);
    if (y1 <= y0) continue;
    std::vector<const uint32_t *> pc(n), pd(n);
    for (int q = 0; q < n; ++q) {
      pc[q] = P.peer_part_c[q] + (size_t)y0 * g.w;
      pd[q] = P.peer_part_d[q] + (size_t)y0 * g.w;
    }
    uint32_t *out = me == g.dest ? g.out + (size_t)y0 * g.out_pitch : P.peer_fin_c[g.dest] + (size_t)y0 * g.w;
    const int64_t opitch = me == g.dest ? g.out_pitch : g.w;
    if (app_roi) {
      std::vector<const int32_t *> rp(n);
      for (int q = 0; q < n; ++q) rp[q] = P.peer_flags[q] + kRoiSlot;
      EQC_TRY(eqc_depth_roi_launch(n, pc.data(), pd.data(), rp.data(), y0, nullptr, g.w, y1 - y0, g.w, out,
                                   nullptr, opitch, P.aux));
    } else {
      EQC_TRY(op_final_pull(g, n, pc.data(), pd.data(), y1 - y0, out, opitch, P.aux));
    }
  }
  mark(P.aux);
  P.prog = base + K;
  {
    const int y0 = row0[me], rows = row0[me + 1] - row0[me];
    for (int q = 0; q < n && rows > 0; ++q)
      if (q != me) {
        stats[0] += 1;
        stats[3] += (int64_t)rows * g.w * 8;
      }
    if (me != g.dest && rows > 0) {
      stats[1] += 1;
      stats[2] += (int64_t)rows * g.w * 4;
    }
    (void)y0;
  }
  EQC_CUDA_TRY(cudaEventRecord(P.ev_pulled, P.aux));
  EQC_CUDA_TRY(cudaStreamWaitEvent(s, P.ev_pulled, 0));
  // every band is complete on the destination (and nobody reads partials)
  EQC_TRY(p2p_barrier(c, s));
  // (the destination's frame may be the comm's gather buffer itself)
  if (me == g.dest && !(g.out == P.fin_c.as<uint32_t>() && g.out_pitch == g.w)) {
    for (int q = 0; q < n; ++q) {
      const int qy0 = row0[q], qrows = row0[q + 1] - row0[q];
      if (q == me || qrows == 0) continue;
      EQC_CUDA_TRY(cudaMemcpy2DAsync(g.out + (size_t)qy0 * g.out_pitch, g.out_pitch * 4,
                                     P.fin_c.as<uint32_t>() + (size_t)qy0 * g.w, (size_t)g.w * 4, (size_t)g.w * 4,
                                     qrows, cudaMemcpyDeviceToDevice, s));
    }
  }
  mark(s);
  if (trace) {
    cudaStreamSynchronize(s);
    fprintf(stderr, "[eqc p2p rank %d] us since start:", me);
    for (size_t i = 1; i < tev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      fprintf(stderr, " %.1f", ms * 1e3);
    }
    fprintf(stderr, "  (pre k, wait k, ..., pulls done, end)\n");
    for (auto e : tev) cudaEventDestroy(e);
  }
  return EQC_OK;
}

int direct_send_p2p(eqc_comm *c, const Geometry &g0, const uint32_t *const *color, const uint32_t *const *depth,
                    cudaStream_t s) {
  P2PState &P = c->p2p;
  Geometry g = g0;
  const int n = c->nranks, me = c->rank;
  int64_t *stats = c->st.stats;
  for (int i = 0; i < 4; ++i) stats[i] = 0;
  std::vector<int> row0(n + 1);
  plan_bands_gather(g.h, n, g.dest, row0.data());
  // ROI (depth compositing only): computed (EQC_FLAG_ROI) or application-provided
  const bool roi = ((g.flags & EQC_FLAG_ROI) != 0 || g.src_roi) && g.op == EQC_OP_DEPTH;
  int32_t *my_roi = P.flags.as<int32_t>() + kRoiSlot;
  // one depth partial that is a frame slot (eqc_comm_frame_buffers): the
  // peers pull it in place; every rank passes its slot-i buffers or none does
  const int slot = (!roi && !g.src_roi && g.op == EQC_OP_DEPTH && g.n_local == 1 && g.pitch == g.w && depth &&
                    (int64_t)g.w * g.h <= P.slot_px)
                       ? P.slot_of(color[0], depth[0])
                       : -1;
  // (1) local pre-composite into the IPC-exposed partial frame.  With
  // EQC_FLAG_ROI the same kernel reduces the bounding box of
  // the partial's rendered pixels (the ROI "computed by analysing the
  // framebuffer", at no extra pass) and publishes it in the
  // peer-readable flags allocation; no host round trip.
  if (g.src_roi && g.op == EQC_OP_DEPTH) {
    // application-provided ROIs: sources are read only inside
    // them, the partial is written only inside their union box, which is
    // published as the partial's ROI
    roi_union_kernel<<<1, 32, 0, s>>>(g.src_roi, g.n_local, my_roi);
    EQC_TRY(eqc_launch_status());
    std::vector<const int32_t *> rp(g.n_local);
    for (int i = 0; i < g.n_local; ++i) rp[i] = g.src_roi + 4 * i;
    EQC_TRY(eqc_depth_roi_launch(g.n_local, color, depth, rp.data(), 0, my_roi, g.w, g.h, g.pitch,
                                 P.part_c.as<uint32_t>(), P.part_d.as<uint32_t>(), g.w, s));
  } else if (roi) {
    EQC_TRY(P.roi_local.ensure(eqc_depth_bbox_scratch_bytes()));
    EQC_TRY(eqc_depth_composite_bbox(g.n_local, color, depth, g.w, g.h, g.pitch, P.part_c.as<uint32_t>(),
                                     P.part_d.as<uint32_t>(), g.w, P.roi_local.p, my_roi, s));
  } else if (slot < 0) {
    EQC_TRY(op_local(g, color, depth, P.part_c.as<uint32_t>(), P.part_d.as<uint32_t>(), s));
  }  // else: the caller's partial frame already is slot `slot` (peer-mapped)
  const std::vector<uint32_t *> &src_c = slot < 0 ? P.peer_part_c : P.peer_slot_c[slot];
  const std::vector<uint32_t *> &src_d = slot < 0 ? P.peer_part_d : P.peer_slot_d[slot];
  // every rank publishes the slot it passed (-1: none) and checks the peers
  // agree (a rank passing its own buffers while another passes a slot would
  // read a partial that was never written): a mismatch sets the comm's error
  // word (eqc_comm_check)
  EQC_TRY(p2p_barrier(c, s, 1, slot));
  // (2)+(3)+(4) band composite pulling every peer's band over NVLink, output
  // pushed into the destination's frame
  const int y0 = row0[me], rows = row0[me + 1] - row0[me];
  if (rows > 0) {
    std::vector<const uint32_t *> cs(n), ds(n);
    for (int q = 0; q < n; ++q) {
      cs[q] = src_c[q] + (size_t)y0 * g.w;
      ds[q] = src_d[q] + (size_t)y0 * g.w;
      if (q != me) {
        stats[0] += 1;
        stats[3] += (int64_t)rows * g.w * 8;
      }
    }
    uint32_t *out = me == g.dest ? g.out + (size_t)y0 * g.out_pitch : P.peer_fin_c[g.dest] + (size_t)y0 * g.w;
    const int64_t opitch = me == g.dest ? g.out_pitch : g.w;
    if (roi) {  // peers' partials are read only inside their ROIs (band-relative rows)
      std::vector<const int32_t *> rp(n);
      for (int q = 0; q < n; ++q) rp[q] = P.peer_flags[q] + kRoiSlot;
      EQC_TRY(eqc_depth_roi_launch(n, cs.data(), ds.data(), rp.data(), y0, nullptr, g.w, rows, g.w, out, nullptr,
                                   opitch, s));
    } else {
      EQC_TRY(op_final_pull(g, n, cs.data(), ds.data(), rows, out, opitch, s));
    }
    if (me != g.dest) {
      stats[1] += 1;
      stats[2] += (int64_t)rows * g.w * 4;
    }
  }
  EQC_TRY(p2p_barrier(c, s));
  // (5) destination: move the pushed bands into the caller's frame
  // (the destination's frame may be the comm's gather buffer itself)
  if (me == g.dest && !(g.out == P.fin_c.as<uint32_t>() && g.out_pitch == g.w)) {
    for (int q = 0; q < n; ++q) {
      const int qy0 = row0[q], qrows = row0[q + 1] - row0[q];
      if (q == me || qrows == 0) continue;
      EQC_CUDA_TRY(cudaMemcpy2DAsync(g.out + (size_t)qy0 * g.out_pitch, g.out_pitch * 4,
                                     P.fin_c.as<uint32_t>() + (size_t)qy0 * g.w, (size_t)g.w * 4, (size_t)g.w * 4,
                                     qrows, cudaMemcpyDeviceToDevice, s));
    }
  }
  return EQC_OK;
}

// Peer-memory binary swap: log2 n rounds; in round r rank g
// and its partner g ^ 2^r each merge their KEPT half of the current region
// in place in their own (IPC-exposed) partial frame, reading the partner's
// rows of that half straight out of the partner's partial over NVLink (the
// partner reads only the other half, which this rank does not write this
// round).  A flag barrier orders the rounds; the last round's merge writes
// the final colour of the rank's region straight into the destination's
// frame (the gather fused into it).  Ties go to the bit-r = 0 group (R-C5).
int binary_swap_p2p(eqc_comm *c, const Geometry &g, const uint32_t *const *color, const uint32_t *const *depth,
                    cudaStream_t s) {
  P2PState &P = c->p2p;
  const int n = c->nranks, me = c->rank;
  int64_t *stats = c->st.stats;
  for (int i = 0; i < 4; ++i) stats[i] = 0;
  std::vector<BsRound> plan;
  const int k = plan_bs(g.h, n, me, plan);
  if (k < 0) return k;
  uint32_t *pc = P.part_c.as<uint32_t>(), *pd = P.part_d.as<uint32_t>();
  EQC_TRY(op_local(g, color, depth, pc, pd, s));
  for (int rd = 0; rd < k; ++rd) {
    EQC_TRY(p2p_barrier(c, s));  // the partner's current data is complete (and no longer read by anyone else)
    const BsRound &b = plan[rd];
    const int krows = b.keep_y1 - b.keep_y0;
    if (b.send_y1 > b.send_y0) stats[0] += 1;
    if (krows <= 0) continue;
    stats[3] += (int64_t)krows * g.w * 8;
    const size_t off = (size_t)b.keep_y0 * g.w;
    const uint32_t *mine_c = pc + off, *mine_d = pd + off;
    const uint32_t *their_c = P.peer_part_c[b.partner] + off, *their_d = P.peer_part_d[b.partner] + off;
    const uint32_t *cc[2] = {b.low ? mine_c : their_c, b.low ? their_c : mine_c};
    const uint32_t *dd[2] = {b.low ? mine_d : their_d, b.low ? their_d : mine_d};
    if (rd + 1 < k) {
      EQC_TRY(op_merge(g, 2, cc, dd, krows, pc + off, pd + off, s));
    } else {
      // last round: the region's final colour, into the destination's frame
      uint32_t *out = me == g.dest ? g.out + (size_t)b.keep_y0 * g.out_pitch : P.peer_fin_c[g.dest] + off;
      const int64_t opitch = me == g.dest ? g.out_pitch : g.w;
      EQC_TRY(op_final(g, 2, cc, dd, krows, out, opitch, s));
      if (me != g.dest) {
        stats[1] += 1;
        stats[2] += (int64_t)krows * g.w * 4;
      }
    }
  }
  if (k == 0) return EQC_OK;
  EQC_TRY(p2p_barrier(c, s));  // every final region is on the destination
  if (me == g.dest && !(g.out == P.fin_c.as<uint32_t>() && g.out_pitch == g.w)) {
    for (int q = 0; q < n; ++q) {
      int y0, y1;
      final_region_bs(g.h, n, q, y0, y1);
      if (q == me || y1 <= y0) continue;
      EQC_CUDA_TRY(cudaMemcpy2DAsync(g.out + (size_t)y0 * g.out_pitch, g.out_pitch * 4,
                                     P.fin_c.as<uint32_t>() + (size_t)y0 * g.w, (size_t)g.w * 4, (size_t)g.w * 4,
                                     y1 - y0, cudaMemcpyDeviceToDevice, s));
    }
  }
  return EQC_OK;
}

// Peer-memory 2-3 swap (R-C21): the fold and every mixed-radix
// round merge in place, reading the other members' rows of this rank's part
// straight out of their partial frames over NVLink (each member reads only
// its own part's rows of the others, which nobody writes in that round); a
// flag barrier before the fold, before every round and at the end; the last
// round writes the final colour into the destination's frame.
int swap23_p2p(eqc_comm *c, const Geometry &g, const uint32_t *const *color, const uint32_t *const *depth,
               cudaStream_t s) {
  P2PState &P = c->p2p;
  const int n = c->nranks, me = c->rank;
  int64_t *stats = c->st.stats;
  for (int i = 0; i < 4; ++i) stats[i] = 0;
  S23Plan plan;
  if (plan_swap23(g.h, n, me, plan) < 0) return EQC_E_INVALID;
  // rounds of the active ranks (the same for all of them; folded senders have none)
  size_t nrounds = plan.rounds.size();
  for (int q = 0; q < n; ++q) {
    S23Plan o;
    plan_swap23(g.h, n, q, o);
    nrounds = std::max(nrounds, o.rounds.size());
  }
  uint32_t *pc = P.part_c.as<uint32_t>(), *pd = P.part_d.as<uint32_t>();
  EQC_TRY(op_local(g, color, depth, pc, pd, s));
  EQC_TRY(p2p_barrier(c, s));
  if (plan.fold_role == 1) {  // lower rank of the pair: whole frames, own first (ties to it)
    const uint32_t *cc[2] = {pc, P.peer_part_c[plan.fold_partner]};
    const uint32_t *dd[2] = {pd, P.peer_part_d[plan.fold_partner]};
    if (nrounds == 0) {
      uint32_t *out = me == g.dest ? g.out : P.peer_fin_c[g.dest];
      EQC_TRY(op_final(g, 2, cc, dd, g.h, out, me == g.dest ? g.out_pitch : g.w, s));
    } else {
      EQC_TRY(op_merge(g, 2, cc, dd, g.h, pc, pd, s));
    }
    stats[3] += (int64_t)g.h * g.w * 8;
  } else if (plan.fold_role == 2) {
    stats[0] += 1;
  }
  for (size_t rd = 0; rd < nrounds; ++rd) {
    EQC_TRY(p2p_barrier(c, s));
    if (rd >= plan.rounds.size()) continue;
    const S23Round &R = plan.rounds[rd];
    const int ky0 = R.bnd[R.t], rows = R.bnd[R.t + 1] - ky0;
    stats[0] += R.k - 1;
    if (rows <= 0) continue;
    const size_t off = (size_t)ky0 * g.w;
    const uint32_t *cc[3], *dd[3];
    for (int u = 0; u < R.k; ++u) {  // members in rank order
      const int q = R.members[u];
      cc[u] = (u == R.t ? pc : P.peer_part_c[q]) + off;
      dd[u] = (u == R.t ? pd : P.peer_part_d[q]) + off;
    }
    stats[3] += (int64_t)rows * g.w * 8 * (R.k - 1);
    if (rd + 1 < nrounds) {
      EQC_TRY(op_merge(g, R.k, cc, dd, rows, pc + off, pd + off, s));
    } else {
      uint32_t *out = me == g.dest ? g.out + (size_t)ky0 * g.out_pitch : P.peer_fin_c[g.dest] + off;
      EQC_TRY(op_final(g, R.k, cc, dd, rows, out, me == g.dest ? g.out_pitch : g.w, s));
      if (me != g.dest) {
        stats[1] += 1;
        stats[2] += (int64_t)rows * g.w * 4;
      }
    }
  }
  EQC_TRY(p2p_barrier(c, s));  // every final region is on the destination
  if (me == g.dest && !(g.out == P.fin_c.as<uint32_t>() && g.out_pitch == g.w)) {
    for (int q = 0; q < n; ++q) {
      S23Plan o;
      plan_swap23(g.h, n, q, o);
      if (q == me || o.fy1 <= o.fy0) continue;
      EQC_CUDA_TRY(cudaMemcpy2DAsync(g.out + (size_t)o.fy0 * g.out_pitch, g.out_pitch * 4,
                                     P.fin_c.as<uint32_t>() + (size_t)o.fy0 * g.w, (size_t)g.w * 4, (size_t)g.w * 4,
                                     o.fy1 - o.fy0, cudaMemcpyDeviceToDevice, s));
    }
  }
  return EQC_OK;
}

}  // namespace

extern "C" int eqc_comm_get_unique_id(uint8_t id[EQC_UNIQUE_ID_BYTES]) {
  if (!id) return EQC_E_INVALID;
  static_assert(sizeof(ncclUniqueId) == EQC_UNIQUE_ID_BYTES, "NCCL unique id size");
  ncclUniqueId u;
  EQC_NCCL_TRY(ncclGetUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return EQC_OK;
}

extern "C" int eqc_comm_init(eqc_comm **comm, int nranks, int rank, const uint8_t id[EQC_UNIQUE_ID_BYTES]) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return EQC_E_INVALID;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  eqc_comm *c = new eqc_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->st.rank = rank;
  if (ncclCommInitRank(&c->nccl, nranks, u, rank) != ncclSuccess) {
    delete c;
    return EQC_E_NCCL;
  }
  *comm = c;
  return EQC_OK;
}

extern "C" int eqc_comm_destroy(eqc_comm *comm) {
  if (!comm) return EQC_E_INVALID;
  cudaDeviceSynchronize();
  comm->p2p.close_peers(comm->rank);
  comm->p2p.close_slots(comm->rank);
  comm->p2p.close_sslots(comm->rank);
  for (int i = 0; i < P2PState::kSlots; ++i) {
    comm->p2p.slot_c[i].release();
    comm->p2p.slot_d[i].release();
    comm->p2p.sslot[i].release();
  }
  if (comm->p2p.aux) cudaStreamDestroy(comm->p2p.aux);
  if (comm->p2p.ev_start) cudaEventDestroy(comm->p2p.ev_start);
  if (comm->p2p.ev_pulled) cudaEventDestroy(comm->p2p.ev_pulled);
  comm->p2p.part_c.release();
  comm->p2p.part_d.release();
  comm->p2p.fin_c.release();
  comm->p2p.flags.release();
  comm->p2p.xfer.release();
  comm->st.release();
  int rc = EQC_OK;
  if (comm->nccl && ncclCommDestroy(comm->nccl) != ncclSuccess) rc = EQC_E_NCCL;
  delete comm;
  return rc;
}

extern "C" int eqc_comm_frame_buffers(eqc_comm *comm, int w, int h, int slot, uint32_t **color, uint32_t **depth,
                                      uint32_t **final_color, void *stream) {
  if (!comm || w <= 0 || h <= 0 || slot < 0 || slot >= P2PState::kSlots || !color || !depth || !final_color)
    return EQC_E_INVALID;
  if (comm->nranks < 2) return EQC_E_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t px = (int64_t)w * h;
  EQC_TRY(p2p_setup(comm, px, s));
  if (comm->p2p.capable != 1) return EQC_E_UNSUPPORTED;
  // + n rows: the scattered layout (n copies of the largest band) fits too
  EQC_TRY(p2p_slots(comm, px + (int64_t)w * comm->nranks, s));
  *color = comm->p2p.slot_c[slot].as<uint32_t>();
  *depth = comm->p2p.slot_d[slot].as<uint32_t>();
  *final_color = comm->p2p.fin_c.as<uint32_t>();
  return EQC_OK;
}

extern "C" int eqc_comm_stream_buffers(eqc_comm *comm, int n_streams, int64_t cap_bytes, int slot, uint8_t **ptrs,
                                       void *stream) {
  if (!comm || n_streams < 2 || n_streams > 2 * EQC_MAX_SOURCES || cap_bytes < 32 || slot < 0 ||
      slot >= P2PState::kSlots || !ptrs)
    return EQC_E_INVALID;
  if (comm->nranks < 2) return EQC_E_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  P2PState &P = comm->p2p;
  EQC_TRY(p2p_setup(comm, 1, s));
  if (P.capable != 1) return EQC_E_UNSUPPORTED;
  const int64_t cap = (cap_bytes + 255) & ~(int64_t)255;
  if (n_streams != P.sn || cap > P.scap) {  // (re)allocate and map both slots
    cudaStreamSynchronize(s);
    P.close_sslots(comm->rank);
    P.sn = 0;
    P.scap = 0;
    void *ptr2[P2PState::kSlots];
    for (int i = 0; i < P2PState::kSlots; ++i) {
      P.sslot[i].release();
      EQC_TRY(P.sslot[i].ensure((size_t)n_streams * (size_t)cap));
      ptr2[i] = P.sslot[i].p;
    }
    std::vector<std::vector<void *>> m;
    int ok = 0;
    EQC_TRY(ipc_exchange(comm, ptr2, P2PState::kSlots, m, ok, s));
    for (int i = 0; i < P2PState::kSlots; ++i) {
      P.peer_sslot[i].assign(comm->nranks, nullptr);
      for (int q = 0; q < comm->nranks; ++q) P.peer_sslot[i][q] = (uint8_t *)m[i][q];
    }
    if (!ok) {
      P.close_sslots(comm->rank);
      return EQC_E_UNSUPPORTED;
    }
    P.sn = n_streams;
    P.scap = cap;
  }
  for (int i = 0; i < n_streams; ++i) ptrs[i] = P.sslot[slot].as<uint8_t>() + (size_t)i * (size_t)P.scap;
  return EQC_OK;
}

namespace {
// The body of compose_direct_send_rle_pull (peer mappings in place).
int rle_pull_body(eqc_comm *comm, int n_local, int w, int h, int slot, int dest_rank, uint32_t *out_color,
                  int64_t out_pitch, int32_t *d_status, cudaStream_t s) {
  const int n = comm->nranks, me = comm->rank;
  P2PState &P = comm->p2p;
  int64_t *stats = comm->st.stats;
  for (int i = 0; i < 4; ++i) stats[i] = 0;
  std::vector<int> row0(n + 1);
  plan_bands(h, n, row0.data());
  // every rank's streams are complete (encoded into its slot)
  EQC_TRY(p2p_barrier(comm, s));
  const int y0 = row0[me], y1 = row0[me + 1];
  if (y1 > y0) {
    const int nt = n * n_local;  // global source order: rank-major (R-C5)
    std::vector<const uint8_t *> cs(nt), ds(nt);
    std::vector<int64_t> cb(nt, P.scap), db(nt, P.scap);
    for (int q = 0; q < n; ++q)
      for (int i = 0; i < n_local; ++i) {
        cs[q * n_local + i] = P.peer_sslot[slot][q] + (size_t)i * (size_t)P.scap;
        ds[q * n_local + i] = P.peer_sslot[slot][q] + (size_t)(n_local + i) * (size_t)P.scap;
      }
    uint32_t *out = me == dest_rank ? out_color + (size_t)y0 * out_pitch : P.peer_fin_c[dest_rank] + (size_t)y0 * w;
    const int64_t opitch = me == dest_rank ? out_pitch : w;
    EQC_TRY(eqc_depth_rle_band(nt, cs.data(), ds.data(), cb.data(), db.data(), w, h, y0, y1, out, nullptr, opitch,
                               d_status, s));
    stats[0] = n - 1;
    if (me != dest_rank) {
      stats[1] = 1;
      stats[2] = (int64_t)(y1 - y0) * w * 4;
    }
  }
  // every band is on the destination; nobody reads the stream slots any more
  EQC_TRY(p2p_barrier(comm, s));
  if (me == dest_rank && !(out_color == P.fin_c.as<uint32_t>() && out_pitch == w)) {
    for (int q = 0; q < n; ++q) {
      const int qy0 = row0[q], qrows = row0[q + 1] - row0[q];
      if (q == me || qrows == 0) continue;
      EQC_CUDA_TRY(cudaMemcpy2DAsync(out_color + (size_t)qy0 * out_pitch, out_pitch * 4,
                                     P.fin_c.as<uint32_t>() + (size_t)qy0 * w, (size_t)w * 4, (size_t)w * 4, qrows,
                                     cudaMemcpyDeviceToDevice, s));
    }
  }
  return EQC_OK;
}
}  // namespace

extern "C" int compose_direct_send_rle_pull(eqc_comm *comm, int n_local, int w, int h, int slot, int dest_rank,
                                            uint32_t *out_color, int64_t out_pitch, int32_t *d_status,
                                            void *stream) {
  if (!comm || n_local < 1 || w <= 0 || h <= 0 || slot < 0 || slot >= P2PState::kSlots || dest_rank < 0 ||
      dest_rank >= comm->nranks || !d_status)
    return EQC_E_INVALID;
  const int n = comm->nranks, me = comm->rank;
  if ((int64_t)n * n_local > EQC_MAX_SOURCES) return EQC_E_INVALID;
  if (me == dest_rank && (!out_color || out_pitch < w)) return EQC_E_INVALID;
  P2PState &P = comm->p2p;
  if (P.sn != 2 * n_local || P.peer_sslot[slot].size() != (size_t)n) return EQC_E_INVALID;  // no stream slots
  cudaStream_t s = (cudaStream_t)stream;
  EQC_TRY(p2p_setup(comm, (int64_t)w * h, s));
  if (P.capable != 1) return EQC_E_UNSUPPORTED;
  return rle_pull_body(comm, n_local, w, h, slot, dest_rank, out_color, out_pitch, d_status, s);
}

// ---- fused decode + scatter (the exchange rides the decode) -----------------
// Band layout in a frame slot for the scattered direct send: copy r (the
// partial of band j from rank r) at rows [r * maxband, r * maxband + rows_j)
// of rank j's slot, pitch w.
namespace {
int scatter_geometry(eqc_comm *c, int w, int h, std::vector<int> &row0, int &maxband) {
  const int n = c->nranks;
  row0.assign(n + 1, 0);
  plan_bands(h, n, row0.data());
  maxband = 0;
  for (int j = 0; j < n; ++j) maxband = std::max(maxband, row0[j + 1] - row0[j]);
  return (int64_t)n * maxband * w <= c->p2p.slot_px ? EQC_OK : EQC_E_INVALID;
}
}  // namespace

namespace {
int scatter_body(eqc_comm *comm, int n_local, const uint8_t *const *color_rle, const uint8_t *const *depth_rle,
                 const int64_t *color_bytes, const int64_t *depth_bytes, int w, int h, int slot, int32_t *d_status,
                 cudaStream_t s) {
  P2PState &P = comm->p2p;
  std::vector<int> row0;
  int maxband = 0;
  EQC_TRY(scatter_geometry(comm, w, h, row0, maxband));
  const int n = comm->nranks, me = comm->rank;
  // the peers' bands first (their stores cross NVLink while the own band is decoded)
  for (int k = 1; k <= n; ++k) {
    const int j = (me + k) % n;
    if (row0[j + 1] <= row0[j]) continue;
    const size_t off = (size_t)me * maxband * w;
    EQC_TRY(eqc_depth_rle_band(n_local, color_rle, depth_rle, color_bytes, depth_bytes, w, h, row0[j], row0[j + 1],
                               P.peer_slot_c[slot][j] + off, P.peer_slot_d[slot][j] + off, w, d_status, s));
  }
  return EQC_OK;
}
}  // namespace

extern "C" int compositor_depth_rle_scatter(eqc_comm *comm, int n_local, const uint8_t *const *color_rle,
                                            const uint8_t *const *depth_rle, const int64_t *color_bytes,
                                            const int64_t *depth_bytes, int w, int h, int slot, int32_t *d_status,
                                            void *stream) {
  if (!comm || n_local < 1 || n_local > EQC_MAX_SOURCES || !color_rle || !depth_rle || !color_bytes ||
      !depth_bytes || w <= 0 || h <= 0 || slot < 0 || slot >= P2PState::kSlots || !d_status)
    return EQC_E_INVALID;
  if (comm->nranks < 2) return EQC_E_UNSUPPORTED;
  P2PState &P = comm->p2p;
  if (P.capable != 1 || P.peer_slot_c[slot].size() != (size_t)comm->nranks) return EQC_E_UNSUPPORTED;
  return scatter_body(comm, n_local, color_rle, depth_rle, color_bytes, depth_bytes, w, h, slot, d_status,
                      (cudaStream_t)stream);
}

namespace {
int scattered_body(eqc_comm *comm, int w, int h, int slot, int dest_rank, uint32_t *out_color, int64_t out_pitch,
                   int flags, cudaStream_t s) {
  const int n = comm->nranks, me = comm->rank;
  P2PState &P = comm->p2p;
  std::vector<int> row0;
  int maxband = 0;
  EQC_TRY(scatter_geometry(comm, w, h, row0, maxband));
  int64_t *stats = comm->st.stats;
  for (int i = 0; i < 4; ++i) stats[i] = 0;
  // every rank's scattered bands are in place (and every rank passed this slot)
  EQC_TRY(p2p_barrier(comm, s, 1, slot));
  const int y0 = row0[me], rows = row0[me + 1] - row0[me];
  if (rows > 0) {
    // band composite of the n copies in my slot (local reads), output pushed
    // into the destination's frame; global source order rank-major (R-C5)
    std::vector<const uint32_t *> cs(n), ds(n);
    for (int q = 0; q < n; ++q) {
      cs[q] = P.slot_c[slot].as<uint32_t>() + (size_t)q * maxband * w;
      ds[q] = P.slot_d[slot].as<uint32_t>() + (size_t)q * maxband * w;
    }
    uint32_t *out = me == dest_rank ? out_color + (size_t)y0 * out_pitch : P.peer_fin_c[dest_rank] + (size_t)y0 * w;
    const int64_t opitch = me == dest_rank ? out_pitch : w;
    eqc_grid_cap = (flags & EQC_FLAG_OVERLAP) ? eqc_num_sms() : 0;
    const int rc = compositor_depth(n, cs.data(), ds.data(), w, rows, w, out, nullptr, opitch, s);
    eqc_grid_cap = 0;
    EQC_TRY(rc);
    stats[0] = n - 1;
    stats[3] = (int64_t)(n - 1) * rows * w * 8;  // received (written by the peers' decodes)
    if (me != dest_rank) {
      stats[1] = 1;
      stats[2] = (int64_t)rows * w * 4;
    }
  }
  // every band is on the destination; nobody reads the slot any more
  EQC_TRY(p2p_barrier(comm, s));
  if (me == dest_rank && !(out_color == P.fin_c.as<uint32_t>() && out_pitch == w)) {
    for (int q = 0; q < n; ++q) {
      const int qy0 = row0[q], qrows = row0[q + 1] - row0[q];
      if (q == me || qrows == 0) continue;
      EQC_CUDA_TRY(cudaMemcpy2DAsync(out_color + (size_t)qy0 * out_pitch, out_pitch * 4,
                                     P.fin_c.as<uint32_t>() + (size_t)qy0 * w, (size_t)w * 4, (size_t)w * 4, qrows,
                                     cudaMemcpyDeviceToDevice, s));
    }
  }
  return EQC_OK;
}

}  // namespace

extern "C" int compose_direct_send_scattered(eqc_comm *comm, int w, int h, int slot, int dest_rank,
                                             uint32_t *out_color, int64_t out_pitch, int flags, void *stream) {
  if (!comm || w <= 0 || h <= 0 || slot < 0 || slot >= P2PState::kSlots || dest_rank < 0 ||
      dest_rank >= comm->nranks)
    return EQC_E_INVALID;
  const int n = comm->nranks, me = comm->rank;
  if (me == dest_rank && (!out_color || out_pitch < w)) return EQC_E_INVALID;
  if (n < 2) return EQC_E_UNSUPPORTED;
  P2PState &P = comm->p2p;
  if (P.capable != 1 || P.peer_slot_c[slot].size() != (size_t)n) return EQC_E_UNSUPPORTED;
  return scattered_body(comm, w, h, slot, dest_rank, out_color, out_pitch, flags, (cudaStream_t)stream);
}

extern "C" int eqc_comm_check(eqc_comm *comm, void *stream) {
  if (!comm) return EQC_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  EQC_CUDA_TRY(cudaStreamSynchronize(s));
  if (comm->nccl) {
    ncclResult_t ae = ncclSuccess;
    if (ncclCommGetAsyncError(comm->nccl, &ae) != ncclSuccess || ae != ncclSuccess) return EQC_E_NCCL;
  }
  P2PState &P = comm->p2p;
  if (P.flags.p) {
    int err = 0;
    EQC_CUDA_TRY(cudaMemcpy(&err, P.flags.as<int>() + kErrSlot, sizeof(int), cudaMemcpyDeviceToHost));
    if (err & kErrTimeout) return EQC_E_NCCL;
    if (err & kErrSlotMismatch) return EQC_E_INVALID;
  }
  return EQC_OK;
}

extern "C" int eqc_comm_abort(eqc_comm *comm) {
  if (!comm) return EQC_E_INVALID;
  if (comm->nccl) {
    ncclCommAbort(comm->nccl);
    comm->nccl = nullptr;
  }
  return EQC_OK;
}

// ---- virtual ranks of the peer-memory transport on one GPU ------------------
// nranks comms without NCCL whose P2P state points at each other's buffers
// (plain device pointers where the real transport has IPC mappings); every
// virtual rank's part of the call runs on its own stream (the flag barriers
// of different ranks must run concurrently), forked from and joined back to
// the caller's stream.  The same host code and kernels as the multi-process
// transport run; only the mapping step differs.
namespace {

// Every kernel of the library loaded (CUDA lazy loading otherwise loads a
// kernel at its first launch and waits for the device to do so: with one
// virtual rank's flag barrier spinning and the rank it waits for enqueued
// after it on the host, that wait never ends).
int eqc_preload_kernels() {
  static int rc = 1;
  if (rc == 1) {
    cudaFuncAttributes a;
    bool ok = cudaFuncGetAttributes(&a, p2p_barrier_kernel) == cudaSuccess &&
              cudaFuncGetAttributes(&a, p2p_signal_kernel) == cudaSuccess &&
              cudaFuncGetAttributes(&a, p2p_wait_kernel) == cudaSuccess &&
              cudaFuncGetAttributes(&a, roi_union_kernel) == cudaSuccess;
    rc = ok ? EQC_OK : EQC_E_CUDA;
    if (rc == EQC_OK) rc = eqc_preload_composite();
    if (rc == EQC_OK) rc = eqc_preload_rle();
    if (rc == EQC_OK) rc = eqc_preload_roi();
  }
  return rc;
}

struct VirtualP2P {
  std::vector<eqc_comm> c;
  std::vector<cudaStream_t> st;
  std::vector<cudaEvent_t> ev;
  int n = 0;
  int init(int nranks, int64_t px, cudaStream_t s) {
    n = nranks;
    c.resize(n);
    st.assign(n, nullptr);
    ev.assign(n + 1, nullptr);
    const char *drop = getenv("EQC_P2P_DROP_RANK");  // test hook: this virtual rank never arrives
    const int dropped = drop ? atoi(drop) : -1;
    for (int q = 0; q < n; ++q) {
      c[q].nranks = n;
      c[q].rank = q;
      c[q].st.rank = q;
      P2PState &P = c[q].p2p;
      EQC_TRY(P.part_c.ensure((size_t)px * 4));
      EQC_TRY(P.part_d.ensure((size_t)px * 4));
      EQC_TRY(P.fin_c.ensure((size_t)px * 4));
      EQC_TRY(P.flags.ensure_zeroed(kFlagInts * sizeof(int)));
      // every allocation up front: a cudaMalloc while another virtual rank's
      // flag barrier spins would wait for the device (implicit sync) and so
      // for a rank whose launches come after it -- a deadlock
      EQC_TRY(P.roi_local.ensure(eqc_depth_bbox_scratch_bytes()));
      P.capable = 1;
      P.cap_px = px;
      P.skip_barriers = q == dropped;
      EQC_CUDA_TRY(cudaStreamCreateWithFlags(&st[q], cudaStreamNonBlocking));
      EQC_CUDA_TRY(cudaEventCreateWithFlags(&ev[q], cudaEventDisableTiming));
    }
    EQC_CUDA_TRY(cudaEventCreateWithFlags(&ev[n], cudaEventDisableTiming));
    EQC_TRY(eqc_preload_kernels());
    for (int q = 0; q < n; ++q) {
      P2PState &P = c[q].p2p;
      P.peer_part_c.assign(n, nullptr);
      P.peer_part_d.assign(n, nullptr);
      P.peer_fin_c.assign(n, nullptr);
      P.peer_flags.assign(n, nullptr);
      for (int r = 0; r < n; ++r) {
        P.peer_part_c[r] = c[r].p2p.part_c.as<uint32_t>();
        P.peer_part_d[r] = c[r].p2p.part_d.as<uint32_t>();
        P.peer_fin_c[r] = c[r].p2p.fin_c.as<uint32_t>();
        P.peer_flags[r] = c[r].p2p.flags.as<int>();
      }
    }
    EQC_CUDA_TRY(cudaEventRecord(ev[n], s));
    for (int q = 0; q < n; ++q) EQC_CUDA_TRY(cudaStreamWaitEvent(st[q], ev[n], 0));
    return EQC_OK;
  }
  // join every virtual rank's stream into s, wait, and report the ranks'
  // error words (a timed-out wait -> EQC_E_NCCL, a slot mismatch -> EQC_E_INVALID)
  int join(cudaStream_t s, int64_t *out_stats) {
    for (int q = 0; q < n; ++q) {
      EQC_CUDA_TRY(cudaEventRecord(ev[q], st[q]));
      EQC_CUDA_TRY(cudaStreamWaitEvent(s, ev[q], 0));
    }
    EQC_CUDA_TRY(cudaStreamSynchronize(s));
    int err = 0;
    for (int q = 0; q < n; ++q) {
      int e = 0;
      EQC_CUDA_TRY(cudaMemcpy(&e, c[q].p2p.flags.as<int>() + kErrSlot, sizeof(int), cudaMemcpyDeviceToHost));
      err |= e;
    }
    if (out_stats) {
      for (int i = 0; i < 4; ++i) out_stats[i] = 0;
      for (auto &x : c)
        for (int i = 0; i < 4; ++i) out_stats[i] += x.st.stats[i];
    }
    if (err & kErrTimeout) return EQC_E_NCCL;
    if (err & kErrSlotMismatch) return EQC_E_INVALID;
    return EQC_OK;
  }
  ~VirtualP2P() {
    cudaDeviceSynchronize();
    for (auto &x : c) {
      P2PState &P = x.p2p;
      P.peer_part_c.clear();  // plain pointers: nothing to unmap
      P.peer_part_d.clear();
      P.peer_fin_c.clear();
      P.peer_flags.clear();
      for (int i = 0; i < P2PState::kSlots; ++i) {
        P.peer_slot_c[i].clear();
        P.peer_slot_d[i].clear();
        P.peer_sslot[i].clear();
        P.slot_c[i].release();
        P.slot_d[i].release();
      }
      P.part_c.release();
      P.part_d.release();
      P.fin_c.release();
      P.flags.release();
      P.roi_local.release();
      P.xfer.release();
      if (P.aux) cudaStreamDestroy(P.aux);
      if (P.ev_start) cudaEventDestroy(P.ev_start);
      if (P.ev_pulled) cudaEventDestroy(P.ev_pulled);
      P.aux = nullptr;
      x.st.release();
    }
    for (auto s : st)
      if (s) cudaStreamDestroy(s);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
};

}  // namespace

extern "C" int compose_direct_send_p2p_local(int nranks, int n_local, const uint32_t *const *color,
                                             const uint32_t *const *depth, int w, int h, int64_t pitch, int op,
                                             int flags, int mode, int dest_rank, uint32_t *out_color,
                                             int64_t out_pitch, int64_t *out_stats, void *stream) {
  EQC_TRY(validate(nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch, true));
  if (nranks < 2 || (flags & (EQC_FLAG_RLE | EQC_FLAG_NCCL))) return EQC_E_INVALID;
  if (mode < EQC_P2P_PLAIN || mode > EQC_P2P_SLOTS) return EQC_E_INVALID;
  if (mode == EQC_P2P_PIPELINED && (flags & EQC_FLAG_ROI)) return EQC_E_INVALID;
  if (mode == EQC_P2P_SLOTS && (n_local != 1 || op != EQC_OP_DEPTH || !depth || (flags & EQC_FLAG_ROI)))
    return EQC_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t px = (int64_t)w * h;
  VirtualP2P V;
  EQC_TRY(V.init(nranks, px, s));
  std::vector<const uint32_t *> cs((size_t)nranks * n_local), dsv((size_t)nranks * n_local);
  for (size_t i = 0; i < cs.size(); ++i) {
    cs[i] = color[i];
    dsv[i] = depth ? depth[i] : nullptr;
  }
  if (mode == EQC_P2P_SLOTS) {
    // each virtual rank's partial frame lives in its slot 0 (the caller's
    // data copied in: the path under test reads the slots in place)
    for (int q = 0; q < nranks; ++q) {
      P2PState &P = V.c[q].p2p;
      EQC_TRY(P.slot_c[0].ensure((size_t)px * 4));
      EQC_TRY(P.slot_d[0].ensure((size_t)px * 4));
      EQC_TRY(P.slot_c[1].ensure(4));
      EQC_TRY(P.slot_d[1].ensure(4));
      EQC_CUDA_TRY(cudaMemcpy2DAsync(P.slot_c[0].p, (size_t)w * 4, color[q], (size_t)pitch * 4, (size_t)w * 4, h,
                                     cudaMemcpyDeviceToDevice, V.st[q]));
      EQC_CUDA_TRY(cudaMemcpy2DAsync(P.slot_d[0].p, (size_t)w * 4, depth[q], (size_t)pitch * 4, (size_t)w * 4, h,
                                     cudaMemcpyDeviceToDevice, V.st[q]));
      P.slot_px = px;
      cs[q] = P.slot_c[0].as<uint32_t>();
      dsv[q] = P.slot_d[0].as<uint32_t>();
    }
    for (int q = 0; q < nranks; ++q)
      for (int i = 0; i < P2PState::kSlots; ++i) {
        V.c[q].p2p.peer_slot_c[i].assign(nranks, nullptr);
        V.c[q].p2p.peer_slot_d[i].assign(nranks, nullptr);
        for (int r = 0; r < nranks; ++r) {
          V.c[q].p2p.peer_slot_c[i][r] = V.c[r].p2p.slot_c[i].as<uint32_t>();
          V.c[q].p2p.peer_slot_d[i][r] = V.c[r].p2p.slot_d[i].as<uint32_t>();
        }
      }
  }
  const int64_t use_pitch = mode == EQC_P2P_SLOTS ? w : pitch;
  for (int q = 0; q < nranks; ++q) {
    Geometry g;
    g.n = nranks;
    g.n_local = n_local;
    g.w = w;
    g.h = h;
    g.pitch = use_pitch;
    g.op = op;
    g.flags = flags;
    g.dest = dest_rank;
    g.out = q == dest_rank ? out_color : nullptr;
    g.out_pitch = q == dest_rank ? out_pitch : w;
    const uint32_t *const *cq = cs.data() + (size_t)q * n_local;
    const uint32_t *const *dq = depth ? dsv.data() + (size_t)q * n_local : nullptr;
    EQC_TRY(mode == EQC_P2P_PIPELINED ? direct_send_p2p_pipelined(&V.c[q], g, cq, dq, V.st[q])
                                      : direct_send_p2p(&V.c[q], g, cq, dq, V.st[q]));
  }
  return V.join(s, out_stats);
}

extern "C" int compose_binary_swap_p2p_local(int nranks, int n_local, const uint32_t *const *color,
                                             const uint32_t *const *depth, int w, int h, int64_t pitch, int op,
                                             int flags, int dest_rank, uint32_t *out_color, int64_t out_pitch,
                                             int64_t *out_stats, void *stream) {
  EQC_TRY(validate(nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch, true));
  if (nranks < 2 || (flags & (EQC_FLAG_RLE | EQC_FLAG_NCCL))) return EQC_E_INVALID;
  if (nranks & (nranks - 1)) return EQC_E_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  VirtualP2P V;
  EQC_TRY(V.init(nranks, (int64_t)w * h, s));
  for (int q = 0; q < nranks; ++q) {
    Geometry g;
    g.n = nranks;
    g.n_local = n_local;
    g.w = w;
    g.h = h;
    g.pitch = pitch;
    g.op = op;
    g.flags = flags;
    g.dest = dest_rank;
    g.out = q == dest_rank ? out_color : nullptr;
    g.out_pitch = q == dest_rank ? out_pitch : w;
    EQC_TRY(binary_swap_p2p(&V.c[q], g, color + (size_t)q * n_local, depth ? depth + (size_t)q * n_local : nullptr,
                            V.st[q]));
  }
  return V.join(s, out_stats);
}

extern "C" int compose_swap23_p2p_local(int nranks, int n_local, const uint32_t *const *color,
                                        const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                        int dest_rank, uint32_t *out_color, int64_t out_pitch, int64_t *out_stats,
                                        void *stream) {
  EQC_TRY(validate(nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch, true));
  if (nranks < 2 || (flags & (EQC_FLAG_RLE | EQC_FLAG_NCCL))) return EQC_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  VirtualP2P V;
  EQC_TRY(V.init(nranks, (int64_t)w * h, s));
  for (int q = 0; q < nranks; ++q) {
    Geometry g;
    g.n = nranks;
    g.n_local = n_local;
    g.w = w;
    g.h = h;
    g.pitch = pitch;
    g.op = op;
    g.flags = flags;
    g.dest = dest_rank;
    g.out = q == dest_rank ? out_color : nullptr;
    g.out_pitch = q == dest_rank ? out_pitch : w;
    EQC_TRY(swap23_p2p(&V.c[q], g, color + (size_t)q * n_local, depth ? depth + (size_t)q * n_local : nullptr,
                       V.st[q]));
  }
  return V.join(s, out_stats);
}

extern "C" int compose_direct_send_rle_pull_local(int nranks, int n_local, const uint8_t *const *rank_streams,
                                                  int64_t cap_bytes, int w, int h, int dest_rank,
                                                  uint32_t *out_color, int64_t out_pitch, int32_t *d_status,
                                                  int64_t *out_stats, void *stream) {
  if (nranks < 2 || n_local < 1 || !rank_streams || cap_bytes <= 0 || w <= 0 || h <= 0 || dest_rank < 0 ||
      dest_rank >= nranks || !out_color || out_pitch < w || !d_status)
    return EQC_E_INVALID;
  if ((int64_t)nranks * n_local > EQC_MAX_SOURCES) return EQC_E_INVALID;
  for (int q = 0; q < nranks; ++q)
    if (!rank_streams[q]) return EQC_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  VirtualP2P V;
  EQC_TRY(V.init(nranks, (int64_t)w * h, s));
  for (int q = 0; q < nranks; ++q) {
    P2PState &P = V.c[q].p2p;
    P.sn = 2 * n_local;
    P.scap = cap_bytes;
    P.peer_sslot[0].assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) P.peer_sslot[0][r] = const_cast<uint8_t *>(rank_streams[r]);
  }
  for (int q = 0; q < nranks; ++q)
    EQC_TRY(rle_pull_body(&V.c[q], n_local, w, h, 0, dest_rank, q == dest_rank ? out_color : nullptr,
                          q == dest_rank ? out_pitch : w, d_status, V.st[q]));
  return V.join(s, out_stats);
}

// Virtual ranks on one GPU (test executor): rank q's n_local colour / depth
// streams are color_rle[q * n_local + i] / depth_rle[q * n_local + i]; every
// rank gets its own frame slot (plain device memory as "peer" memory).
extern "C" int compose_direct_send_scatter_local(int nranks, int n_local, const uint8_t *const *color_rle,
                                                 const uint8_t *const *depth_rle, const int64_t *color_bytes,
                                                 const int64_t *depth_bytes, int w, int h, int dest_rank,
                                                 uint32_t *out_color, int64_t out_pitch, int32_t *d_status,
                                                 int64_t *out_stats, void *stream) {
  if (nranks < 2 || nranks > EQC_MAX_SOURCES || n_local < 1 || n_local > EQC_MAX_SOURCES || !color_rle ||
      !depth_rle || !color_bytes || !depth_bytes || w <= 0 || h <= 0 || dest_rank < 0 || dest_rank >= nranks ||
      !out_color || out_pitch < w || !d_status)
    return EQC_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  VirtualP2P V;
  EQC_TRY(V.init(nranks, (int64_t)w * h, s));
  const int64_t spx = (int64_t)w * h + (int64_t)w * nranks;  // the scattered layout (as eqc_comm_frame_buffers)
  for (int q = 0; q < nranks; ++q) {  // every allocation before any launch (see VirtualP2P::init)
    P2PState &P = V.c[q].p2p;
    EQC_TRY(P.slot_c[0].ensure((size_t)spx * 4));
    EQC_TRY(P.slot_d[0].ensure((size_t)spx * 4));
    P.slot_px = spx;
  }
  for (int q = 0; q < nranks; ++q) {
    P2PState &P = V.c[q].p2p;
    P.peer_slot_c[0].assign(nranks, nullptr);
    P.peer_slot_d[0].assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
      P.peer_slot_c[0][r] = V.c[r].p2p.slot_c[0].as<uint32_t>();
      P.peer_slot_d[0][r] = V.c[r].p2p.slot_d[0].as<uint32_t>();
    }
  }
  for (int q = 0; q < nranks; ++q) {
    const size_t o = (size_t)q * n_local;
    EQC_TRY(scatter_body(&V.c[q], n_local, color_rle + o, depth_rle + o, color_bytes + o, depth_bytes + o, w, h, 0,
                         d_status, V.st[q]));
    EQC_TRY(scattered_body(&V.c[q], w, h, 0, dest_rank, q == dest_rank ? out_color : nullptr,
                           q == dest_rank ? out_pitch : w, 0, V.st[q]));
  }
  return V.join(s, out_stats);
}

extern "C" int eqc_comm_stats(const eqc_comm *comm, int64_t out[4]) {
  if (!comm || !out) return EQC_E_INVALID;
  for (int i = 0; i < 4; ++i) out[i] = comm->st.stats[i];
  return EQC_OK;
}

extern "C" int eqc_plan_bands(int h, int n, int *row0) {
  if (h <= 0 || n < 1 || !row0) return EQC_E_INVALID;
  plan_bands(h, n, row0);
  return EQC_OK;
}

extern "C" int eqc_plan_bands_gather(int h, int n, int dest, int *row0) {
  if (h <= 0 || n < 1 || dest < 0 || dest >= n || !row0) return EQC_E_INVALID;
  plan_bands_gather(h, n, dest, row0);
  return EQC_OK;
}

extern "C" int eqc_plan_binary_swap(int h, int n, int rank, int *rounds, int max_rounds) {
  if (h <= 0 || n < 1 || rank < 0 || rank >= n) return EQC_E_INVALID;
  std::vector<BsRound> rr;
  const int k = plan_bs(h, n, rank, rr);
  if (k < 0) return k;
  if (k > max_rounds || (k > 0 && !rounds)) return EQC_E_CAPACITY;
  for (int i = 0; i < k; ++i) {
    const BsRound &b = rr[i];
    const int v[6] = {b.partner, b.low, b.keep_y0, b.keep_y1, b.send_y0, b.send_y1};
    std::memcpy(rounds + 6 * i, v, sizeof(v));
  }
  return k;
}

enum Algo { kDirectSend, kBinarySwap, kSwap23, kStream };

static int compose_nccl(Algo algo, eqc_comm *comm, int n_local, const uint32_t *const *color,
                        const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags, int dest_rank,
                        uint32_t *out_color, int64_t out_pitch, void *stream, const int32_t *src_roi = nullptr) {
  if (!comm) return EQC_E_INVALID;
  EQC_TRY(validate(comm->nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch,
                   comm->rank == dest_rank));
  if (algo == kBinarySwap && (comm->nranks & (comm->nranks - 1))) return EQC_E_UNSUPPORTED;
  const bool ds = algo == kDirectSend;
  Geometry g;
  g.n = comm->nranks;
  g.n_local = n_local;
  g.w = w;
  g.h = h;
  g.pitch = pitch;
  g.op = op;
  g.flags = flags;
  g.dest = dest_rank;
  g.out = out_color;
  g.out_pitch = comm->rank == dest_rank ? out_pitch : w;
  comm->st.color = color;
  comm->st.depth = depth;
  g.src_roi = src_roi;
  cudaStream_t s = (cudaStream_t)stream;
  if (ds && comm->nranks > 1 && !(flags & (EQC_FLAG_RLE | EQC_FLAG_NCCL))) {
    EQC_TRY(p2p_setup(comm, (int64_t)w * h, s));
    if (comm->p2p.capable == 1) {
      // pieces pay off only when each rank's pre-composite is substantial
      // (measured: >= 2 sources and >= 6 Mpx per band; below that the extra
      // launches and flag round trips cost more than the overlap gains)
      const bool big = n_local >= 2 && (int64_t)w * (h / comm->nranks) >= (int64_t)6 << 20;
      return (!(flags & EQC_FLAG_ROI) && big) ? direct_send_p2p_pipelined(comm, g, color, depth, s)
                                              : direct_send_p2p(comm, g, color, depth, s);
    }
  }
  if ((algo == kBinarySwap || algo == kSwap23) && comm->nranks > 1 && !(flags & (EQC_FLAG_RLE | EQC_FLAG_NCCL))) {
    EQC_TRY(p2p_setup(comm, (int64_t)w * h, s));
    if (comm->p2p.capable == 1)
      return algo == kBinarySwap ? binary_swap_p2p(comm, g, color, depth, s) : swap23_p2p(comm, g, color, depth, s);
  }
  NcclTransport T(comm->nccl, s);
  std::vector<RankState *> ranks{&comm->st};
  return ds ? run_direct_send(ranks, g, T, s)
         : algo == kBinarySwap ? run_binary_swap(ranks, g, T, s)
         : algo == kSwap23     ? run_swap23(ranks, g, T, s)
                               : run_stream(ranks, g, T, s);
}

extern "C" int compose_direct_send(eqc_comm *comm, int n_local, const uint32_t *const *color,
                                   const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                   int dest_rank, uint32_t *out_color, int64_t out_pitch, void *stream) {
  return compose_nccl(kDirectSend, comm, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch,
                      stream);
}

extern "C" int compose_binary_swap(eqc_comm *comm, int n_local, const uint32_t *const *color,
                                   const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                   int dest_rank, uint32_t *out_color, int64_t out_pitch, void *stream) {
  return compose_nccl(kBinarySwap, comm, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch,
                      stream);
}

static int compose_local(Algo algo, int nranks, int n_local, const uint32_t *const *color,
                         const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags, int dest_rank,
                         uint32_t *out_color, int64_t out_pitch, int64_t *out_stats, void *stream,
                         const int32_t *src_roi = nullptr) {
  EQC_TRY(validate(nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch, true));
  if (algo == kBinarySwap && (nranks & (nranks - 1))) return EQC_E_UNSUPPORTED;
  Geometry g;
  g.n = nranks;
  g.n_local = n_local;
  g.w = w;
  g.h = h;
  g.pitch = pitch;
  g.op = op;
  g.flags = flags;
  g.dest = dest_rank;
  g.out = out_color;
  g.out_pitch = out_pitch;
  g.src_roi = src_roi;
  g.src_roi_all_ranks = true;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<RankState> states(nranks);
  std::vector<RankState *> ranks;
  for (int q = 0; q < nranks; ++q) {
    states[q].rank = q;
    states[q].color = color + (size_t)q * n_local;
    states[q].depth = depth ? depth + (size_t)q * n_local : nullptr;
    ranks.push_back(&states[q]);
  }
  LocalTransport T(s);
  int rc = algo == kDirectSend ? run_direct_send(ranks, g, T, s)
           : algo == kBinarySwap ? run_binary_swap(ranks, g, T, s)
           : algo == kSwap23     ? run_swap23(ranks, g, T, s)
                                 : run_stream(ranks, g, T, s);
  cudaStreamSynchronize(s);  // scratch is freed below
  if (out_stats) {
    for (int i = 0; i < 4; ++i) out_stats[i] = 0;
    for (auto &st : states)
      for (int i = 0; i < 4; ++i) out_stats[i] += st.stats[i];
  }
  for (auto &st : states) st.release();
  return rc;
}

static int tiles_validate(int nranks, int n_local, const void *color, const void *depth, int w, int h, int64_t pitch,
                          int tiles_x, int tiles_y, int flags, const void *out, int64_t out_pitch) {
  if (nranks < 1 || n_local < 1 || n_local > EQC_MAX_SOURCES || nranks > EQC_MAX_SOURCES) return EQC_E_INVALID;
  if (!color || !depth || w <= 0 || h <= 0 || pitch < w || !out || out_pitch < w) return EQC_E_INVALID;
  if (tiles_x < 1 || tiles_y < 1 || tiles_x > w || tiles_y > h || (int64_t)tiles_x * tiles_y > 4096)
    return EQC_E_INVALID;
  if (flags & ~EQC_FLAG_RLE) return EQC_E_INVALID;
  return EQC_OK;
}

static Geometry tiles_geometry(int nranks, int n_local, int w, int h, int64_t pitch, int flags, uint32_t *out,
                               int64_t out_pitch) {
  Geometry g;
  g.n = nranks;
  g.n_local = n_local;
  g.w = w;
  g.h = h;
  g.pitch = pitch;
  g.op = EQC_OP_DEPTH;
  g.flags = flags;
  g.out = out;
  g.out_pitch = out_pitch;
  return g;
}

extern "C" int eqc_plan_tiles(int w, int h, int tiles_x, int tiles_y, int nranks, int tile, int *rect) {
  if (w <= 0 || h <= 0 || tiles_x < 1 || tiles_y < 1 || tiles_x > w || tiles_y > h || nranks < 1 || !rect ||
      tile < 0 || tile >= tiles_x * tiles_y)
    return EQC_E_INVALID;
  const TileRect r = plan_tile(w, h, tiles_x, tiles_y, nranks, tile);
  rect[0] = r.x0, rect[1] = r.y0, rect[2] = r.w, rect[3] = r.h, rect[4] = r.owner;
  return EQC_OK;
}

extern "C" int compose_tiles(eqc_comm *comm, int n_local, const uint32_t *const *color, const uint32_t *const *depth,
                             int w, int h, int64_t pitch, int tiles_x, int tiles_y, int flags, uint32_t *out_color,
                             int64_t out_pitch, void *stream) {
  if (!comm) return EQC_E_INVALID;
  EQC_TRY(tiles_validate(comm->nranks, n_local, color, depth, w, h, pitch, tiles_x, tiles_y, flags, out_color,
                         out_pitch));
  Geometry g = tiles_geometry(comm->nranks, n_local, w, h, pitch, flags, out_color, out_pitch);
  comm->st.color = color;
  comm->st.depth = depth;
  cudaStream_t s = (cudaStream_t)stream;
  NcclTransport T(comm->nccl, s);
  std::vector<RankState *> ranks{&comm->st};
  return run_tiles(ranks, g, T, s, tiles_x, tiles_y);
}

extern "C" int compose_tiles_local(int nranks, int n_local, const uint32_t *const *color,
                                   const uint32_t *const *depth, int w, int h, int64_t pitch, int tiles_x,
                                   int tiles_y, int flags, uint32_t *out_color, int64_t out_pitch,
                                   int64_t *out_stats, void *stream) {
  EQC_TRY(tiles_validate(nranks, n_local, color, depth, w, h, pitch, tiles_x, tiles_y, flags, out_color, out_pitch));
  Geometry g = tiles_geometry(nranks, n_local, w, h, pitch, flags, out_color, out_pitch);
  cudaStream_t s = (cudaStream_t)stream;
  // the virtual ranks' scratch (GBs at wall size) is kept for the next call
  // with the same number of ranks (EQC_TILES_LOCAL_KEEP=0: freed every call)
  static std::vector<RankState> states;
  static const bool keep = !getenv("EQC_TILES_LOCAL_KEEP") || atoi(getenv("EQC_TILES_LOCAL_KEEP")) != 0;
  if ((int)states.size() != nranks) {
    cudaStreamSynchronize(s);
    for (auto &st : states) st.release();
    states.clear();
    states.resize(nranks);
  }
  std::vector<RankState *> ranks;
  for (int q = 0; q < nranks; ++q) {
    states[q].rank = q;
    states[q].color = color + (size_t)q * n_local;
    states[q].depth = depth + (size_t)q * n_local;
    if (states[q].status.p) cudaMemsetAsync(states[q].status.p, 0, sizeof(int32_t), s);
    ranks.push_back(&states[q]);
  }
  LocalTransport T(s);
  int rc = run_tiles(ranks, g, T, s, tiles_x, tiles_y);
  cudaStreamSynchronize(s);
  if (rc == EQC_OK) {
    for (auto &st : states) {
      int32_t bad = 0;
      if (st.status.p) cudaMemcpy(&bad, st.status.p, sizeof(bad), cudaMemcpyDeviceToHost);
      if (bad) rc = EQC_E_CORRUPT;
    }
  }
  if (out_stats) {
    for (int i = 0; i < 4; ++i) out_stats[i] = 0;
    for (auto &st : states)
      for (int i = 0; i < 4; ++i) out_stats[i] += st.stats[i];
  }
  if (!keep || rc != EQC_OK) {
    for (auto &st : states) st.release();
    states.clear();
  }
  return rc;
}

extern "C" int compose_direct_send_local(int nranks, int n_local, const uint32_t *const *color,
                                         const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                         int dest_rank, uint32_t *out_color, int64_t out_pitch, int64_t *out_stats,
                                         void *stream) {
  return compose_local(kDirectSend, nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch,
                       out_stats, stream);
}

extern "C" int compose_binary_swap_local(int nranks, int n_local, const uint32_t *const *color,
                                         const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                         int dest_rank, uint32_t *out_color, int64_t out_pitch, int64_t *out_stats,
                                         void *stream) {
  return compose_local(kBinarySwap, nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch,
                       out_stats, stream);
}

extern "C" int compose_swap23(eqc_comm *comm, int n_local, const uint32_t *const *color,
                              const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                              int dest_rank, uint32_t *out_color, int64_t out_pitch, void *stream) {
  return compose_nccl(kSwap23, comm, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch,
                      stream);
}

extern "C" int compose_swap23_local(int nranks, int n_local, const uint32_t *const *color,
                                    const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                    int dest_rank, uint32_t *out_color, int64_t out_pitch, int64_t *out_stats,
                                    void *stream) {
  return compose_local(kSwap23, nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color,
                       out_pitch, out_stats, stream);
}

extern "C" int eqc_plan_swap23(int h, int n, int rank, int *out, int max_ints) {
  if (h <= 0 || n < 1 || rank < 0 || rank >= n || !out) return EQC_E_INVALID;
  S23Plan P;
  const int k = plan_swap23(h, n, rank, P);
  if (k < 0) return k;
  const int need = 5 + 9 * k;
  if (need > max_ints) return EQC_E_CAPACITY;
  out[0] = P.fold_role;
  out[1] = P.fold_partner;
  out[2] = k;
  out[3] = P.fy0;
  out[4] = P.fy1;
  for (int i = 0; i < k; ++i) {
    const S23Round &R = P.rounds[i];
    int *o = out + 5 + 9 * i;
    o[0] = R.k;
    o[1] = R.t;
    for (int u = 0; u < 3; ++u) o[2 + u] = R.members[u];
    for (int u = 0; u < 4; ++u) o[5 + u] = R.bnd[u];
  }
  return k;
}

extern "C" int compose_stream(eqc_comm *comm, int n_local, const uint32_t *const *color,
                              const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                              int dest_rank, uint32_t *out_color, int64_t out_pitch, void *stream) {
  return compose_nccl(kStream, comm, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color, out_pitch,
                      stream);
}

extern "C" int compose_stream_local(int nranks, int n_local, const uint32_t *const *color,
                                    const uint32_t *const *depth, int w, int h, int64_t pitch, int op, int flags,
                                    int dest_rank, uint32_t *out_color, int64_t out_pitch, int64_t *out_stats,
                                    void *stream) {
  return compose_local(kStream, nranks, n_local, color, depth, w, h, pitch, op, flags, dest_rank, out_color,
                       out_pitch, out_stats, stream);
}

extern "C" int compose_direct_send_roi(eqc_comm *comm, int n_local, const uint32_t *const *color,
                                       const uint32_t *const *depth, const int32_t *d_src_roi, int w, int h,
                                       int64_t pitch, int flags, int dest_rank, uint32_t *out_color,
                                       int64_t out_pitch, void *stream) {
  if (!d_src_roi || ((uintptr_t)d_src_roi & 15) != 0) return EQC_E_INVALID;
  return compose_nccl(kDirectSend, comm, n_local, color, depth, w, h, pitch, EQC_OP_DEPTH, flags, dest_rank,
                      out_color, out_pitch, stream, d_src_roi);
}

extern "C" int compose_direct_send_roi_local(int nranks, int n_local, const uint32_t *const *color,
                                             const uint32_t *const *depth, const int32_t *d_src_roi, int w, int h,
                                             int64_t pitch, int flags, int dest_rank, uint32_t *out_color,
                                             int64_t out_pitch, int64_t *out_stats, void *stream) {
  if (!d_src_roi || ((uintptr_t)d_src_roi & 15) != 0) return EQC_E_INVALID;
  return compose_local(kDirectSend, nranks, n_local, color, depth, w, h, pitch, EQC_OP_DEPTH, flags, dest_rank,
                       out_color, out_pitch, out_stats, stream, d_src_roi);
}
