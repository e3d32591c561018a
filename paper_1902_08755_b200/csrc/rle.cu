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
// Encoder: two kernels, no inter-CTA waiting.  rle_encode_kernel: every warp
// codes one run of 16 consecutive chunks (classify all, code the non-constant
// ones in registers/shared memory), appends the records to its slice of an
// (L2-resident) record scratch, and writes its run size and its table entries
// relative to the run.  rle_compact_kernel then gives every run its payload
// offset (the sum of the preceding runs' sizes of the same image -- a few
// thousand values, summed directly, no look-back chain), moves the records
// to their final place, rebases the table entries and writes the header.
#include <algorithm>

#include "rle.cuh"
#include "rle_enc.cuh"

#ifndef EQC_ENC_WARPS
#define EQC_ENC_WARPS 1
#endif
#ifndef EQC_ENC_MINB
#define EQC_ENC_MINB 28  // 1-warp CTAs at 72 registers (measured best: no spills, no intra-CTA imbalance)
#endif
#ifndef EQC_DEC_MINB
#define EQC_DEC_MINB 3  // 80 registers (measured best for the v1 decoder)
#endif
#ifndef EQC_FUSED_MINB
#define EQC_FUSED_MINB (32 / EQC_FWARPS)  // 32 warps per SM (64 registers)
#endif
#ifndef EQC_CLS_BATCH
#define EQC_CLS_BATCH 8
#endif

using namespace eqc_rle;

namespace {

constexpr int kWarps = 8;            // warps per CTA
#ifndef EQC_RUN_CHUNKS
#define EQC_RUN_CHUNKS 16
#endif
constexpr int kSTChunksPerWarp = EQC_RUN_CHUNKS;  // encoder: consecutive chunks per warp run (small: balances uneven chunks)
static_assert(kSTChunksPerWarp <= 64, "two table-entry registers per lane");
constexpr int kEncWarps = EQC_ENC_WARPS;  // coder warps per CTA (encoder); warps are independent
constexpr int kCompactWarps = 8;          // runs per CTA of the compaction kernel
constexpr int kRecMax = 4 * (kC + 2);                  // worst-case chunk record bytes (520)
// a run's scratch slot: whole 128-byte lines (the compaction discards them)
constexpr int kScratchPerWarp = (kSTChunksPerWarp * kRecMax + 127) / 128 * 128;  // 16 chunks: 8320 = 65 x 128 B
constexpr int kMaxBatch = 64;

// workspace layout: run_size[count * runs_per_image] int32 (the coded bytes
// of every run of kSTChunksPerWarp consecutive chunks), then (256-byte
// aligned) the record scratch: kScratchPerWarp bytes per run.  No state
// survives between calls (no zeroing needed).

struct EncImage {
  const uint32_t *src;
  uint8_t *dst;
  int64_t *d_size;
  int kind, flags;
};

struct EncParams {
  EncImage img[kMaxBatch];
  int32_t *run_size;     // inside the workspace
  uint8_t *scratch;      // record scratch (inside the workspace)
  int64_t pitch;
  int64_t nchunks;       // per image
  int count, w, h, S;    // S = chunks per row
  int tiles_per_image;   // encoder CTAs per image
  int runs_per_image;
  int vec;               // 128-bit loads allowed
};

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

// Copy `size` bytes from a 16-byte aligned global source (the warp's record
// scratch) to an arbitrary global destination: whole 4-byte destination
// words are funnel-shifted out of aligned source words; the <= 3 head and
// <= 3 tail bytes are byte copies.
__device__ __forceinline__ void copy_run(uint8_t *g, const uint8_t *src, int64_t size, int lane) {
  const uintptr_t ga = (uintptr_t)g;
  const uintptr_t first_w = (ga + 3) & ~(uintptr_t)3;
  const uintptr_t end = ga + (uintptr_t)size;
  const uintptr_t last_w = end & ~(uintptr_t)3;
  if (first_w >= last_w) {
    for (int64_t k = lane; k < size; k += 32) g[k] = __ldcg(src + k);
    return;
  }
  const int head = (int)(first_w - ga);
  const int tail = (int)(end - last_w);
  if (lane < head) g[lane] = __ldcg(src + lane);
  if (lane >= 8 && lane < 8 + tail) {
    const int64_t q = (int64_t)(last_w - ga) + lane - 8;
    g[q] = __ldcg(src + q);
  }
  const int64_t nw = (int64_t)((last_w - first_w) >> 2);
  const uint32_t *s32 = reinterpret_cast<const uint32_t *>(src) + (head >> 2);
  const int sh = head & 3;
  uint32_t *gw = reinterpret_cast<uint32_t *>(first_w);
  // 8 independent loads in flight per lane per step (the scratch usually
  // comes back from DRAM: enough bytes in flight to cover its latency)
  int64_t k = lane;
  for (; k + 224 < nw; k += 256) {
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      lo[u] = __ldcg(s32 + k + 32 * u);
      hi[u] = sh ? __ldcg(s32 + k + 32 * u + 1) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) gw[k + 32 * u] = sh ? __funnelshift_r(lo[u], hi[u], 8 * sh) : lo[u];
  }
  uint32_t lo[8], hi[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int64_t kk = k + 32 * u;
    lo[u] = kk < nw ? __ldcg(s32 + kk) : 0u;
    hi[u] = (kk < nw && sh) ? __ldcg(s32 + kk + 1) : 0u;
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int64_t kk = k + 32 * u;
    if (kk < nw) gw[kk] = sh ? __funnelshift_r(lo[u], hi[u], 8 * sh) : lo[u];
  }
}

__device__ __forceinline__ void discard_l2(const void *p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// Per-warp shared memory of the encoder.
struct WarpEnc {
  uint8_t stage[kStageBytes];        // one coded record
  uint8_t toks[kTokBytes];           // token-start scratch of encode_chunk
  uint32_t cval[kSTChunksPerWarp];   // constant chunks: the (swizzled) value
  uint32_t cps[kSTChunksPerWarp];    // plane sizes of each chunk record
  uint16_t csize[kSTChunksPerWarp];  // record size of each chunk
  uint8_t gidx[kSTChunksPerWarp];    // positions of the non-constant chunks
};

struct EncSmem {
  WarpEnc w[kEncWarps];
};

// Encoder.  Every warp codes one run of kSTChunksPerWarp consecutive chunks,
// independently of the other warps of its (small) CTA -- no CTA barrier, so a
// warp whose chunks are cheap never waits for a busy neighbour:
//  A. classify: stream the run's chunks (coalesced 128-bit loads, several in
//     flight per lane); a chunk whose pixels are all equal (76 % of the target
//     workload) only records its value -- about a dozen instructions;
//  B. code every other chunk with encode_chunk (SIMD-within-a-word flags,
//     packed-byte scans, per-plane classes) from a second, L2-resident read,
//     the next chunk's load in flight, and store its record at its offset in
//     the warp's run (the offsets of the constant chunks are known from A);
//  C. write the constant chunks' 12-byte records lane-parallel and the
//     table entries.
// The compaction kernel then moves the runs to their final offsets.
// R64: the RLE-64 codec (R-C17); constant chunks (all 128 pixels equal) get a
// 10-byte record [1][0x80 | 63][v v] instead of four 3-byte planes.
template <bool R64>
__global__ void __launch_bounds__(kEncWarps * 32, EQC_ENC_MINB) rle_encode_kernel(const __grid_constant__ EncParams p) {
  constexpr int kCRec = R64 ? 10 : 12;  // record bytes of a constant chunk
  extern __shared__ __align__(16) uint8_t smem_raw[];
  EncSmem &sm = *reinterpret_cast<EncSmem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  WarpEnc &W = sm.w[warp];
  const int m = (int)(blockIdx.x / p.tiles_per_image);
  const int lr = (int)(blockIdx.x - m * p.tiles_per_image) * kEncWarps + warp;  // run of image m
  if (lr >= p.runs_per_image) return;  // no CTA-wide barrier below: warps are independent
  const int64_t gr = (int64_t)m * p.runs_per_image + lr;
  const EncImage im = p.img[m];
  const int nch = (int)p.nchunks;
  const bool swz = (im.flags & EQC_FLAG_SWIZZLE) != 0;
  uint8_t *scr = p.scratch + (size_t)gr * kScratchPerWarp;
  const int c0 = lr * kSTChunksPerWarp;
  const int cnt = min(kSTChunksPerWarp, nch - c0);
  const int Llast = p.w - (p.S - 1) * kC;
  const int k0 = c0 % p.S;
  const uint32_t *row0 = im.src + (int64_t)(c0 / p.S) * p.pitch;
  const bool contig = p.vec && (p.w % kC) == 0 && p.pitch == p.w;
  // chunk j of the run -> (pointer, length)
  auto chunk_ptr = [&](int j, int &L) -> const uint32_t * {
    if (contig) {  // one contiguous span of full chunks
      L = kC;
      return row0 + (int64_t)(k0 + j) * kC;
    }
    const int kk = k0 + j;
    const int dy = kk / p.S, k = kk - dy * p.S;
    L = k == p.S - 1 ? Llast : kC;
    return row0 + (int64_t)dy * p.pitch + k * kC;
  };
  // ---- A: classify (4 chunks in flight per lane; row pointer advanced
  // incrementally; the swizzle of constant values is deferred to C).  When
  // the warp's chunks are one contiguous span of full 128-pixel chunks
  // (pitch == w, w % 128 == 0) the loads use immediate offsets, 8 in flight.
  int ng = 0;
  uint64_t cmask = 0;
  if (contig) {
    const uint4 *base = reinterpret_cast<const uint4 *>(row0 + (int64_t)k0 * kC) + lane;
    for (int j0 = 0; j0 < cnt; j0 += EQC_CLS_BATCH) {
      uint4 v[EQC_CLS_BATCH];
#pragma unroll
      for (int u = 0; u < EQC_CLS_BATCH; ++u)
        v[u] = (j0 + u < cnt) ? ld_stream_u4(base + 32 * (j0 + u)) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < EQC_CLS_BATCH; ++u) {
        if (j0 + u >= cnt) break;
        const uint32_t v0 = __shfl_sync(EQC_FULL, v[u].x, 0);
        const bool same = v[u].x == v0 && v[u].y == v0 && v[u].z == v0 && v[u].w == v0;
        if (__all_sync(EQC_FULL, same)) {
          cmask |= 1ull << (j0 + u);
          if (lane == 0) W.cval[j0 + u] = v0;
        } else {
          if (lane == 0) W.gidx[ng] = (uint8_t)(j0 + u);
          ++ng;
        }
      }
    }
  } else {
    int ka = k0;
    const uint32_t *rowa = row0;
    for (int j0 = 0; j0 < cnt; j0 += 4) {
      uint32_t px[4][4];
      int Ls[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        Ls[u] = 0;
        if (j0 + u < cnt) {
          Ls[u] = ka == p.S - 1 ? Llast : kC;
          load_chunk(rowa + ka * kC, Ls[u], lane, p.vec != 0, px[u]);
          if (++ka == p.S) {
            ka = 0;
            rowa += p.pitch;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j0 + u >= cnt) break;
        uint32_t v0;
        const bool cst = chunk_is_constant(px[u], Ls[u], lane, v0) && (!R64 || (Ls[u] & 1) == 0);
        if (cst) {
          cmask |= 1ull << (j0 + u);
          if (lane == 0) W.cval[j0 + u] = v0;
        } else {
          if (lane == 0) W.gidx[ng] = (uint8_t)(j0 + u);
          ++ng;
        }
      }
    }
  }
  __syncwarp();
  // ---- B: the other chunks, SIMD coder, next chunk's load in flight
  int gen_bytes = 0;
  uint32_t nxt[4] = {0, 0, 0, 0};
  int Ln = 0;
  if (ng > 0) load_chunk(chunk_ptr(W.gidx[0], Ln), Ln, lane, p.vec != 0, nxt);
#pragma unroll 1
  for (int g = 0; g < ng; ++g) {
    uint32_t px[4] = {nxt[0], nxt[1], nxt[2], nxt[3]};
    const int L = Ln;
    const int j = W.gidx[g];
    if (g + 1 < ng) load_chunk(chunk_ptr(W.gidx[g + 1], Ln), Ln, lane, p.vec != 0, nxt);
    const EncodeOut eo = R64 ? encode_chunk64(px, L, lane, W.stage, W.toks)
                             : encode_chunk(px, L, lane, swz, W.stage, W.toks);
    const int off = kCRec * __popcll(cmask & ((1ull << j) - 1)) + gen_bytes;
    store_record(scr + off, W.stage, eo.size, lane);
    if (lane == 0) {
      W.csize[j] = (uint16_t)eo.size;
      W.cps[j] = eo.psizes;
    }
    gen_bytes += eo.size;
    __syncwarp();
  }
  // ---- C: offsets of all chunks, constant records, table entries
  const int j1 = lane, j2 = lane + 32;
  const bool cst1 = j1 < cnt && ((cmask >> j1) & 1ull), cst2 = j2 < cnt && ((cmask >> j2) & 1ull);
  const int s1 = j1 < cnt ? (cst1 ? kCRec : (int)W.csize[j1]) : 0;
  const int s2 = j2 < cnt ? (cst2 ? kCRec : (int)W.csize[j2]) : 0;
  const int i1 = (int)warp_incl_scan_add((uint32_t)s1, lane);
  const int t1 = __shfl_sync(EQC_FULL, i1, 31);
  const int i2 = (int)warp_incl_scan_add((uint32_t)s2, lane) + t1;
  const int off1 = i1 - s1, off2 = i2 - s2;
  const int run = __shfl_sync(EQC_FULL, i2, 31);
  const uint32_t cps = R64 ? (uint32_t)kCRec : 0x03030303u;  // RLE-64: the table holds the record size
  uint32_t ps1 = cst1 ? cps : (j1 < cnt ? W.cps[j1] : 0u);
  uint32_t ps2 = cst2 ? cps : (j2 < cnt ? W.cps[j2] : 0u);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = h ? j2 : j1;
    const int off = h ? off2 : off1;
    if (h ? cst2 : cst1) {
      int L;
      chunk_ptr(j, L);
      uint8_t *gp = scr + off;
      if (R64) {  // [1][0x80 | (L/2 - 1)][v v], L even
        const uint32_t v = W.cval[j];
        gp[0] = 1;
        gp[1] = (uint8_t)(0x80 | (L / 2 - 1));
#pragma unroll
        for (int q = 0; q < 8; ++q) gp[2 + q] = (uint8_t)(v >> (8 * (q & 3)));
      } else {
        const uint32_t v = swz ? swizzle(W.cval[j]) : W.cval[j];
        const uint8_t c = (uint8_t)(0x80 | (L - 1));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          gp[3 * q] = 1;
          gp[3 * q + 1] = c;
          gp[3 * q + 2] = (uint8_t)(v >> (8 * q));
        }
      }
    }
  }
  if (lane == 0) p.run_size[gr] = run;
  // table entries relative to the run (rebased by the compaction)
  uint2 *table = reinterpret_cast<uint2 *>(im.dst + 32) + c0;
  if (j1 < cnt) table[j1] = make_uint2((uint32_t)off1, ps1);
  if (j2 < cnt) table[j2] = make_uint2((uint32_t)off2, ps2);
}

struct CompactParams {
  EncImage img[kMaxBatch];
  const int32_t *run_size;
  const uint32_t *run_off;  // per image: exclusive prefix of run sizes, then the total
  const uint8_t *scratch;
  int64_t nchunks;
  int w, h, groups_per_image, runs_per_image;
};

// One CTA per image: exclusive prefix of the image's run sizes (the payload
// offset of every run) and the payload total, so the compaction needs no
// per-CTA summation of all preceding runs.
__global__ void __launch_bounds__(1024) rle_runscan_kernel(const int32_t *run_size, uint32_t *run_off, int runs) {
  __shared__ uint32_t s_w[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t *rs = run_size + (int64_t)blockIdx.x * runs;
  uint32_t *ro = run_off + (int64_t)blockIdx.x * (runs + 1);
  const int per = (runs + blockDim.x - 1) / blockDim.x;  // consecutive runs per thread
  const int q0 = tid * per, q1 = min(runs, q0 + per);
  uint32_t local = 0;
  for (int q = q0; q < q1; ++q) local += (uint32_t)__ldg(rs + q);
  const uint32_t inc = warp_incl_scan_add(local, lane);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0u;
    const uint32_t wi = warp_incl_scan_add(v, lane);
    s_w[lane] = wi - v;
  }
  __syncthreads();
  uint32_t acc = s_w[warp] + inc - local;
  for (int q = q0; q < q1; ++q) {
    ro[q] = acc;
    acc += (uint32_t)__ldg(rs + q);
  }
  if (q1 == runs && q0 < q1) ro[runs] = acc;
  if (runs == 0 && tid == 0) ro[0] = 0;
}

// One warp per run (kCompactWarps per CTA, independent): moves the run from
// the scratch to its payload offset, rebases its table entries and discards
// its scratch lines from L2; the warp of an image's last run writes the
// header and the stream size.
__global__ void __launch_bounds__(kCompactWarps * 32) rle_compact_kernel(const __grid_constant__ CompactParams p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = (int)(blockIdx.x / p.groups_per_image);
  const int r = (int)(blockIdx.x - m * p.groups_per_image) * kCompactWarps + warp;  // run of image m
  if (r >= p.runs_per_image) return;
  const EncImage im = p.img[m];
  const uint32_t *ro = p.run_off + (int64_t)m * (p.runs_per_image + 1);
  const int64_t base = __ldg(ro + r);
  const int64_t run = __ldg(p.run_size + (int64_t)m * p.runs_per_image + r);
  if (r == p.runs_per_image - 1 && lane == 0) {
    const int64_t payload = __ldg(ro + p.runs_per_image);
    uint32_t *h32 = reinterpret_cast<uint32_t *>(im.dst);
    h32[0] = kMagic;
    h32[1] = (uint32_t)kVersion | ((uint32_t)im.kind << 8) | ((uint32_t)im.flags << 16) | ((uint32_t)kLog2C << 24);
    h32[2] = (uint32_t)p.w;
    h32[3] = (uint32_t)p.h;
    h32[4] = (uint32_t)p.nchunks;
    h32[5] = 0u;
    h32[6] = (uint32_t)(uint64_t)payload;
    h32[7] = (uint32_t)((uint64_t)payload >> 32);
    *im.d_size = 32 + 8 * p.nchunks + payload;
  }
  const int nch = (int)p.nchunks;
  const int c0 = r * kSTChunksPerWarp;
  const int cnt = min(kSTChunksPerWarp, nch - c0);
  const uint8_t *scr = p.scratch + ((size_t)m * p.runs_per_image + r) * kScratchPerWarp;
  uint2 *table = reinterpret_cast<uint2 *>(im.dst + 32) + c0;
  for (int j = lane; j < cnt; j += 32) {
    uint2 e = table[j];
    e.x = (uint32_t)(base + e.x);
    table[j] = e;
  }
  if (run > 0) {
    copy_run(im.dst + 32 + 8 * p.nchunks + base, scr, run, lane);
    __syncwarp();
    for (int l = lane; (int64_t)l * 128 < run; l += 32) discard_l2(scr + 128 * l);
  }
}

// ---------------------------------------------------------------------------
// v1 encoder (image_compress_rle_batch without RLE-64): two launches.
//   rle_encode3_kernel   persistent warps take runs (kRun3 consecutive chunks
//                        of one image) by ticket, in image order: classify the
//                        run's chunks, code the non-constant ones
//                        (eqc_enc::code_chunk) into a per-warp shared span at
//                        run-relative offsets, write the constant chunks'
//                        12-byte records and the run-relative table entries,
//                        copy the span to the run's record-scratch slot (L2
//                        evict-last), store the run size and add it to its
//                        block of 64 runs;
//   rle_compact3_kernel  moves every run to its payload offset (below).
// (A single launch with the compaction overlapped was measured slower: the
// completion signalling costs every run a release fence.)
// ---------------------------------------------------------------------------
#ifndef EQC_E3_GROUP_MB
#define EQC_E3_GROUP_MB 4096  // raw megabytes of images per encoder/compaction launch pair
#endif
#ifndef EQC_E3_WARPS
#define EQC_E3_WARPS 4
#endif
#ifndef EQC_E3_MINB
#define EQC_E3_MINB 6
#endif
constexpr int kRun3 = kSTChunksPerWarp;  // chunks per encode item (same scratch layout as the RLE-64 path)
constexpr int kE3Warps = EQC_E3_WARPS;

struct __align__(16) E3Warp {  // (16-aligned: warps' spans are read as uint4)
  uint8_t span[kRun3 * kRecMax + 16];    // the run's records (+ garbage slack)
  uint8_t tp[(eqc_enc::kTpBytes + 4 + 15) & ~15];  // start list + trash bytes
  uint32_t cps[kRun3];
  uint16_t csz[kRun3];
  uint8_t q[kRun3];
};

struct Enc3Params {
  EncImage img[kMaxBatch];
  int32_t *run_size;   // [count][R]
  uint8_t *scratch;    // [count][R] slots of kScratchPerWarp bytes
  uint32_t *ctr;       // [0] encode ticket
  uint32_t *blk;       // [count][NB] block totals (sum of the sizes of 64 consecutive runs)
  int64_t pitch, nchunks;
  int count, w, h, S, R, NB;  // NB = blocks of 64 runs per image
  float invS, invR;           // 1 / S, 1 / R
  int total_enc;
  int vec;             // 128-bit loads allowed
};


#ifndef EQC_E3_L2HINT
#define EQC_E3_L2HINT 2  // 1: record scratch stored L2 evict_last; 2: + classify loads L2 evict_first
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_u4_hint(void *a, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint4 ld_stream_u4_if_hint(const void *p, bool pred, uint64_t pol) {
  uint4 r = make_uint4(0, 0, 0, 0);
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %6;\n\t}"
      : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
      : "l"(p), "r"((uint32_t)pred), "l"(pol));
  return r;
}

// q = a / b for 0 <= a < 2^22 by a float reciprocal (inv = 1/b), corrected
// by one; larger a: the integer division.
__device__ __forceinline__ int div_small(int a, int b, float inv) {
  if (a >= (1 << 22)) return a / b;
  int q = (int)((float)a * inv);
  const int r = a - q * b;
  q += r < 0 ? -1 : (r >= b ? 1 : 0);
  return q;
}

// CONTIG: pitch == w, w % 128 == 0, 16-byte aligned: a run is one contiguous
// span of full chunks (straight-line loads with immediate offsets).
// FULL: w % 128 == 0 (every chunk has 128 pixels).
template <bool FULL, bool CONTIG>
__device__ void e3_encode_run(const Enc3Params &p, int m, int r, int lane, E3Warp &W, const eqc_enc::LaneK &K,
                              const uint32_t *lut_sel, const uint32_t *lut_st) {
  const EncImage im = p.img[m];
  const int nch = (int)p.nchunks;
  const bool swz = (im.flags & EQC_FLAG_SWIZZLE) != 0;
  const int c0 = r * kRun3;
  const int cnt = min(kRun3, nch - c0);
  const int Llast = p.w - (p.S - 1) * kC;
  const int y0 = div_small(c0, p.S, p.invS), k0 = c0 - y0 * p.S;
  const uint32_t *row0 = im.src + (int64_t)y0 * p.pitch;
  auto chunk_ptr = [&](int j, int &L) -> const uint32_t * {
    if (CONTIG) {
      L = kC;
      return row0 + (int64_t)(k0 + j) * kC;
    }
    const int kk = k0 + j;
    const int dy = kk / p.S, k = kk - dy * p.S;
    L = (!FULL && k == p.S - 1) ? Llast : kC;
    return row0 + (int64_t)dy * p.pitch + k * kC;
  };
  // ---- A: classify (8 chunks in flight per lane)
  uint32_t cmask = 0, myc = 0;  // myc: lane j keeps the value of constant chunk j
  int ng = 0;
  for (int j0 = 0; j0 < cnt; j0 += 8) {
    uint32_t px[8][4];
    int Ls[8];
    if (CONTIG) {
      const uint4 *base = reinterpret_cast<const uint4 *>(row0 + (int64_t)(k0 + j0) * kC) + lane;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 v = EQC_E3_L2HINT >= 2 ? ld_stream_u4_if_hint(base + 32 * u, j0 + u < cnt, l2_policy_evict_first())
                                           : ld_stream_u4_if(base + 32 * u, j0 + u < cnt);
        px[u][0] = v.x, px[u][1] = v.y, px[u][2] = v.z, px[u][3] = v.w;
        Ls[u] = kC;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        Ls[u] = 0;
        px[u][0] = px[u][1] = px[u][2] = px[u][3] = 0u;
        if (j0 + u < cnt) {
          const uint32_t *cp = chunk_ptr(j0 + u, Ls[u]);
          if (p.vec && (FULL || 4 * lane + 4 <= Ls[u])) {
            const uint4 v = ld_stream_u4(cp + 4 * lane);
            px[u][0] = v.x, px[u][1] = v.y, px[u][2] = v.z, px[u][3] = v.w;
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) px[u][q] = 4 * lane + q < Ls[u] ? ld_stream_u32(cp + 4 * lane + q) : 0u;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j0 + u >= cnt) break;
      const int L = Ls[u];
      const uint32_t v0 = __shfl_sync(EQC_FULL, px[u][0], 0);
      bool same;
      if (FULL) {
        same = ((px[u][0] ^ v0) | (px[u][1] ^ v0) | (px[u][2] ^ v0) | (px[u][3] ^ v0)) == 0u;
      } else {
        same = true;
#pragma unroll
        for (int q = 0; q < 4; ++q) same = same && (px[u][q] == v0 || 4 * lane + q >= L);
      }
      if (__all_sync(EQC_FULL, same) && (FULL || L >= 3)) {
        cmask |= 1u << (j0 + u);
        myc = lane == j0 + u ? v0 : myc;
      } else {
        if (lane == 0) W.q[ng] = (uint8_t)(j0 + u);
        ++ng;
      }
    }
  }
  __syncwarp();
  // ---- B: code the other chunks (re-read from L2, the next one in flight)
  int coded = 0;
  uint32_t nx[4] = {0u, 0u, 0u, 0u};
  int Ln = kC;
  auto load = [&](int j) {
    const uint32_t *cp = chunk_ptr(j, Ln);
    if (CONTIG || (p.vec && (FULL || 4 * lane + 4 <= Ln))) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(cp + 4 * lane));
      nx[0] = v.x, nx[1] = v.y, nx[2] = v.z, nx[3] = v.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) nx[q] = 4 * lane + q < Ln ? __ldcg(cp + 4 * lane + q) : 0u;
    }
  };
  if (ng > 0) load(W.q[0]);
#pragma unroll 1
  for (int g = 0; g < ng; ++g) {
    uint32_t x[4] = {nx[0], nx[1], nx[2], nx[3]};
    const int L = Ln;
    const int j = W.q[g];
    if (g + 1 < ng) load(W.q[g + 1]);
    if (swz) {
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = swizzle(x[q]);
    }
    const int off = 12 * __popc(cmask & ((1u << j) - 1u)) + coded;
    uint32_t ps;
    const int sz = eqc_enc::code_chunk<FULL>(x, L, lane, K, W.span + off, W.tp, lut_sel, lut_st, &ps);
    if (lane == 0) {
      W.csz[j] = (uint16_t)sz;
      W.cps[j] = ps;
    }
    coded += sz;
  }
  __syncwarp();
  // ---- C: offsets, constant records, table entries, run -> scratch
  const int j = lane;
  const bool isc = j < cnt && ((cmask >> j) & 1u);
  const int s = j < cnt ? (isc ? 12 : (int)W.csz[j]) : 0;
  const int inc = (int)warp_incl_scan_add((uint32_t)s, lane);
  const int run = __shfl_sync(EQC_FULL, inc, 31);
  const int off = inc - s;
  if (isc) {
    int L = kC;
    if (!FULL) chunk_ptr(j, L);
    const uint32_t v = swz ? swizzle(myc) : myc;
    const uint32_t c = 0x80u | (uint32_t)(L - 1);
    // [01][c][v0] [01][c][v1] [01][c][v2] [01][c][v3] as three words, stored bytewise
    const uint32_t w0 = 1u | (c << 8) | ((v & 0xFFu) << 16) | (1u << 24);
    const uint32_t w1 = c | (((v >> 8) & 0xFFu) << 8) | (1u << 16) | (c << 24);
    const uint32_t w2 = ((v >> 16) & 0xFFu) | (1u << 8) | (c << 16) | ((v >> 24) << 24);
    uint8_t *g = W.span + off;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      g[q] = (uint8_t)(w0 >> (8 * q));
      g[4 + q] = (uint8_t)(w1 >> (8 * q));
      g[8 + q] = (uint8_t)(w2 >> (8 * q));
    }
  }
  if (j < cnt) {
    uint2 *table = reinterpret_cast<uint2 *>(im.dst + 32) + c0;
    table[j] = make_uint2((uint32_t)off, isc ? 0x03030303u : W.cps[j]);
  }
  __syncwarp();
  const int64_t gr = (int64_t)m * p.R + r;
  uint4 *slot = reinterpret_cast<uint4 *>(p.scratch + (size_t)gr * kScratchPerWarp);
  const uint4 *sp = reinterpret_cast<const uint4 *>(W.span);
  if (EQC_E3_L2HINT >= 1) {
    const uint64_t pol = l2_policy_evict_last();
    for (int i = lane; 16 * i < run; i += 32) st_u4_hint(slot + i, sp[i], pol);
  } else {
    for (int i = lane; 16 * i < run; i += 32) slot[i] = sp[i];
  }
  if (lane == 0) p.run_size[gr] = run;
  if (lane == 0) atomicAdd(p.blk + (int64_t)m * p.NB + (r >> 6), (uint32_t)run);  // the run's block of 64 runs
}

// Compaction (v1): one warp per run.  The run's payload offset is the sum of
// the block totals before its block of 64 runs plus the sizes of the runs of
// its block before it; every load of the run -- those partial sums, its size,
// its table entries and the first 512 B of its records -- is issued at once
// (one memory round trip for a background run), then the records are stored at
// their offset (whole destination words funnel-shifted, the <= 3 head and tail
// bytes by byte stores), the table entries rebased, and the scratch lines
// dropped from L2.  The warp of an image's last run writes the header.
struct Cmp3Params {
  EncImage img[kMaxBatch];
  const int32_t *run_size;  // [count][R]
  const uint32_t *blk;      // [count][NB]
  const uint8_t *scratch;
  int64_t nchunks;
  int count, w, h, R, NB;
};

constexpr int kCmp3Warps = 8;
#ifndef EQC_CMP_U
#define EQC_CMP_U 4
#endif
#ifndef EQC_CMP_REVERSE
#define EQC_CMP_REVERSE 1
#endif

__global__ void __launch_bounds__(kCmp3Warps * 32) rle_compact3_kernel(const __grid_constant__ Cmp3Params p) {
  const int lane = threadIdx.x & 31;
  // grid (runs / kCmp3Warps, images); EQC_CMP_REVERSE: the images coded last
  // (whose scratch is the most likely to be still in L2) first
  const int r = blockIdx.x * kCmp3Warps + (threadIdx.x >> 5);
  if (r >= p.R) return;
  const int m = EQC_CMP_REVERSE ? p.count - 1 - (int)blockIdx.y : (int)blockIdx.y;
  const int64_t gr = (int64_t)m * p.R + r;
  const EncImage im = p.img[m];
  const int nch = (int)p.nchunks;
  const int c0 = r * kRun3, cnt = min(kRun3, nch - c0);
  const int32_t *rs = p.run_size + (int64_t)m * p.R;
  const uint32_t *blk = p.blk + (int64_t)m * p.NB;
  const uint32_t *src = reinterpret_cast<const uint32_t *>(p.scratch + (size_t)gr * kScratchPerWarp);
  uint2 *table = reinterpret_cast<uint2 *>(im.dst + 32) + c0;
  // ---- every load at once
  const int b = r >> 6, q0 = b << 6;
  uint32_t part = 0;
  for (int i = lane; i < b; i += 32) part += __ldcg(blk + i);
  for (int i = q0 + lane; i < r; i += 32) part += (uint32_t)__ldcg(rs + i);
  const int run = __ldcg(rs + r);
  uint2 e = make_uint2(0u, 0u);
  if (lane < cnt) e = __ldcg(table + lane);
  constexpr int U = EQC_CMP_U;  // words per lane in the first round (128 B per warp each)
  uint32_t w[U];
#pragma unroll
  for (int u = 0; u < U; ++u) w[u] = __ldcg(src + 32 * u + lane);
  const uint32_t base = __reduce_add_sync(EQC_FULL, part);
  if (lane < cnt) {
    e.x += base;
    table[lane] = e;
  }
  uint8_t *dst = im.dst + 32 + 8 * p.nchunks + base;
  if (r == p.R - 1 && lane == 0) {
    const uint32_t total = base + (uint32_t)run;
    uint32_t *h32 = reinterpret_cast<uint32_t *>(im.dst);
    h32[0] = kMagic;
    h32[1] = (uint32_t)kVersion | ((uint32_t)im.kind << 8) | ((uint32_t)im.flags << 16) | ((uint32_t)kLog2C << 24);
    h32[2] = (uint32_t)p.w;
    h32[3] = (uint32_t)p.h;
    h32[4] = (uint32_t)p.nchunks;
    h32[5] = 0u;
    h32[6] = total;
    h32[7] = 0u;
    *im.d_size = 32 + 8 * p.nchunks + (int64_t)total;
  }
  if (run <= 0) return;
  // destination word k (k >= 0) = bytes [4k - a, 4k - a + 4) of the run, a =
  // dst & 3; for a > 0 it is funnel(src word k-1, src word k); its bytes
  // outside [0, run) belong to the neighbouring runs (byte stores there)
  const int a = (int)((uintptr_t)dst & 3u);
  uint32_t *dw = reinterpret_cast<uint32_t *>(dst - a);
  const int nk = (run + a + 3) >> 2;  // destination words touched
  auto put = [&](int k, uint32_t lo, uint32_t hi) {
    // lo = src word k - 1 (unused when a == 0), hi = src word k
    const uint32_t v = a ? __funnelshift_r(lo, hi, 8 * (4 - a)) : hi;
    const int b0 = 4 * k - a;  // run byte at the word's first byte
    if (b0 >= 0 && b0 + 4 <= run) {
      dw[k] = v;
    } else {
      uint8_t *d8 = reinterpret_cast<uint8_t *>(dw + k);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (b0 + q >= 0 && b0 + q < run) d8[q] = (uint8_t)(v >> (8 * q));
    }
  };
#pragma unroll
  for (int u = 0; u < U; ++u) {
    // src word k - 1 of k = 32u + lane: the previous lane's word u, or (lane 0)
    // lane 31's word u - 1
    const uint32_t up = __shfl_up_sync(EQC_FULL, w[u], 1);
    const uint32_t wrap = __shfl_sync(EQC_FULL, u ? w[u - 1] : 0u, 31);
    const int k = 32 * u + lane;
    if (k < nk) put(k, lane ? up : wrap, w[u]);
  }
  for (int k0 = 32 * U; k0 < nk; k0 += 4 * 32) {  // longer runs: the rest, 4 words per lane in flight
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + 32 * u + lane;
      lo[u] = k < nk ? __ldcg(src + k - 1) : 0u;
      hi[u] = k < nk ? __ldcg(src + k) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + 32 * u + lane;
      if (k < nk) put(k, lo[u], hi[u]);
    }
  }
  __syncwarp();
  for (int l = lane; l * 128 < run; l += 32) discard_l2(reinterpret_cast<const uint8_t *>(src) + 128 * l);
}

template <bool FULL, bool CONTIG>
__global__ void __launch_bounds__(kE3Warps * 32, EQC_E3_MINB) rle_encode3_kernel(const __grid_constant__ Enc3Params p) {
  __shared__ uint32_t s_lut[16 + 256];
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 16 + 256; i += blockDim.x) s_lut[i] = reinterpret_cast<const uint32_t *>(&eqc_enc::g_enc_luts)[i];
  __syncthreads();  // the only CTA-wide barrier: warps are independent below
  uint32_t *const ectr = p.ctr;
  // ---- encode warp
  E3Warp &W = reinterpret_cast<E3Warp *>(smem_raw)[warp];
  const eqc_enc::LaneK K = eqc_enc::lane_consts(lane);
  int e = 0;  // encode ticket
  if (lane == 0) e = (int)atomicAdd(ectr, 1u);
  e = __shfl_sync(EQC_FULL, e, 0);
  while (e < p.total_enc) {
    int en = 0;
    if (lane == 0) en = (int)atomicAdd(ectr, 1u);  // the next ticket, in flight meanwhile
    const int m = div_small(e, p.R, p.invR);
    e3_encode_run<FULL, CONTIG>(p, m, e - m * p.R, lane, W, K, s_lut, s_lut + 16);
    e = __shfl_sync(EQC_FULL, en, 0);
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
// allow64: also accept RLE-64 streams (flags == EQC_FLAG_RLE64, 128-pixel chunks)
__device__ StreamHdr read_header(const uint8_t *src, int64_t src_bytes, int w, int h, bool allow64 = false) {
  StreamHdr hd{};
  hd.ok = 0;
  if (src_bytes < 32) return hd;
  const uint32_t *h32 = reinterpret_cast<const uint32_t *>(src);
  const uint32_t w0 = h32[0], w1 = h32[1];
  const int ver = w1 & 0xFF, kind = (w1 >> 8) & 0xFF, flags = (w1 >> 16) & 0xFF, log2c = w1 >> 24;
  const bool r64 = allow64 && flags == EQC_FLAG_RLE64 && log2c == kLog2C;
  if (w0 != kMagic || ver != kVersion || kind > 1 || ((flags & ~1) && !r64) || (kind == 1 && (flags & 1)) ||
      log2c < 5 || log2c > 7)
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

// Constant-chunk probe (lane-local): a record of four 3-byte planes
// [01][0x80 | (L-1)][v] is one value for the whole chunk.  Reads the 12
// bytes as aligned words (an aligned word that starts inside the stream
// never leaves its allocation) and funnel-shifts them into place.
__device__ __forceinline__ bool probe_const(const uint8_t *rec, uint32_t ps, int L, uint32_t &v) {
  if (ps != 0x03030303u) return false;
  const uint32_t *a = reinterpret_cast<const uint32_t *>((uintptr_t)rec & ~(uintptr_t)3);
  const int sh = 8 * (int)((uintptr_t)rec & 3);
  const uint32_t q0 = __ldg(a), q1 = __ldg(a + 1), q2 = __ldg(a + 2);
  const uint32_t q3 = sh ? __ldg(a + 3) : 0u;
  const uint32_t w0 = __funnelshift_r(q0, q1, sh), w1 = __funnelshift_r(q1, q2, sh),
                 w2 = __funnelshift_r(q2, q3, sh);
  // bytes: [01 c v0 01][c v1 01 c][v2 01 c v3]
  const uint32_t c = 0x80u | (uint32_t)(L - 1);
  const bool ok = (w0 & 0xFF00FFFFu) == (0x01000001u | (c << 8)) &&
                  (w1 & 0xFFFF00FFu) == (c | 0x00010000u | (c << 24)) && (w2 & 0x00FFFF00u) == (0x0100u | (c << 16));
  v = __byte_perm(w0, w1, 0x0652) | 0u;  // v0 = byte 2 of w0, v1 = byte 1 of w1 (= byte 5)
  v = (v & 0xFFFFu) | (__byte_perm(w2, 0, 0x3000) & 0xFF000000u) | ((w2 & 0xFFu) << 16);
  return ok;
}

#ifndef EQC_PLANE_UNROLL
#define EQC_PLANE_UNROLL 1
#endif
constexpr int kPlaneUnroll = EQC_PLANE_UNROLL;  // (1: one decode_plane_w call site per pass)

// Decode a staged record into px[0..3], planes in the order 3, 0, 1, 2 (the
// most significant byte first).  With `check`, when that byte alone makes the
// source deeper than the current best at every pixel of the chunk (bm: byte j
// = the best depth's most significant byte at pixel j; vinv: 0xFF bytes for
// pixels past the chunk) it cannot win (ties keep the lower index): planes
// 0-2 are not decoded and `skip` is set.
// One decode_plane_w call site (the kernels must stay inside the instruction
// cache).  Warp-uniform result; false on a malformed record.
__device__ __forceinline__ bool decode_staged(const uint8_t *r, uint32_t ps, int L, int lane, uint16_t *info,
                                              uint32_t px[4], bool check, uint32_t bm, uint32_t vinv,
                                              bool &skip, bool swz = false) {
  // plane sizes and record offsets in decode order: rotate plane 3 first
  uint32_t sz = __funnelshift_l(ps, ps, 8);  // bytes: s3, s0, s1, s2
  int off = (int)__dp4a(ps, 0x00010101u, 0u);  // s0 + s1 + s2
  uint32_t X0 = 0, X1 = 0, X2 = 0, X3 = 0;  // shift register of plane words
  bool ok = true;
  skip = false;
#pragma unroll kPlaneUnroll
  for (int t = 0; t < 4; ++t) {
    const int size = (int)(sz & 0xFFu);
    const uint32_t w = decode_plane_w(r + off, size, L, lane, ok, info);
    X3 = X2;
    X2 = X1;
    X1 = X0;
    X0 = w;
    if (t == 0 && check && ok) {
      if (__all_sync(EQC_FULL, (__vcmpgtu4(w, bm) | vinv) == 0xFFFFFFFFu)) {
        skip = true;
        return true;
      }
    }
    off = t == 0 ? 0 : off + size;
    sz >>= 8;
  }
  // decode order 3, 0, 1, 2: X3 = plane 3, X2 = plane 0, X1 = plane 1, X0 = plane 2
  uint32_t W[4] = {X2, X1, X0, X3};
  if (swz) unswizzle_planes(W);
  planes_to_px(W, px);
  return ok;
}

// Stage a record from global memory (aligned 4-byte words; byte loads at the
// stream end) into `stage` (>= 3 + 520 + 8 bytes); returns the staged
// record's first byte.  Not inlined: the fallback for records that do not fit
// the prefetch buffer.
__device__ __noinline__ const uint8_t *stage_record(const uint8_t *src, int64_t src_bytes, const uint8_t *rec,
                                                    uint32_t ps, int lane, uint8_t *stage) {
  const int s0 = ps & 0xFF, s1 = (ps >> 8) & 0xFF, s2 = (ps >> 16) & 0xFF, s3 = ps >> 24;
  const int total = s0 + s1 + s2 + s3;
  const uintptr_t a0 = (uintptr_t)rec & ~(uintptr_t)3;
  const int sh = (int)((uintptr_t)rec & 3);
  const int nwords = (sh + total + 3) >> 2;
  const uintptr_t lim = (uintptr_t)src + (uintptr_t)src_bytes;
  uint32_t *st32 = reinterpret_cast<uint32_t *>(stage);
  __syncwarp();  // the previous record's readers are done with the stage
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
  return stage + sh;
}

// 16-byte units of the aligned window covering a record.
__device__ __forceinline__ int record_quads(const uint8_t *rec, uint32_t ps) {
  const int total = (int)__dp4a(ps, 0x01010101u, 0u);  // the four plane sizes
  return ((int)((uintptr_t)rec & 15) + total + 15) >> 4;
}

// Issue asynchronous 16-byte copies of the aligned window covering a record
// into `dst` (shared; the record starts at byte rec & 15 of dst).  The window
// never starts before the stream (records follow the header and table); a
// quad that would cross the stream end is copied byte by byte.
__device__ __forceinline__ void stage_async16(const uint8_t *src, int64_t src_bytes, const uint8_t *rec, int nquads,
                                              uint4 *dst, int lane) {
  const uintptr_t a0 = (uintptr_t)rec & ~(uintptr_t)15;
  const uintptr_t lim = (uintptr_t)src + (uintptr_t)src_bytes;
  for (int q = lane; q < nquads; q += 32) {
    const uintptr_t a = a0 + 16 * (uintptr_t)q;
    if (a + 16 <= lim) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + q);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(a) : "memory");
    } else {
      uint8_t *d = reinterpret_cast<uint8_t *>(dst + q);
      for (int b = 0; b < 16; ++b) d[b] = a + b < lim ? __ldg(reinterpret_cast<const uint8_t *>(a + b)) : 0;
    }
  }
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
  int64_t src_bytes;
};

struct DecParams {
  DecImage img[kMaxBatch];
  int32_t *status;
  int64_t pitch;
  int count, w, h;
  int64_t tiles_per_image;  // CTAs per image: 8 warps x 32 slots of 128 pixels
  int vec;
};

constexpr int kGroup = 32;  // chunks classified per warp pass (one per lane)

// Lane-parallel table read for chunk c (valid if `has`): entry, and the
// monotone/contiguous check against chunk c-1, whose entry lane
// `lane - delta` holds (lanes below `delta` load it).  Must be called by the
// whole warp.  Returns ok.
__device__ __forceinline__ bool entry_lane(const uint8_t *src, int64_t payload_bytes, int64_t nchunks, int64_t c,
                                           bool has, int L, int lane, int64_t &off, uint32_t &ps, int delta = 1) {
  uint2 te = make_uint2(0, 0);
  if (has) te = __ldg(reinterpret_cast<const uint2 *>(src + 32 + 8 * c));
  off = te.x;
  ps = te.y;
  const int s0 = ps & 0xFF, s1 = (ps >> 8) & 0xFF, s2 = (ps >> 16) & 0xFF, s3 = ps >> 24;
  const int64_t end = off + s0 + s1 + s2 + s3;
  int64_t prev = __shfl_up_sync(EQC_FULL, end, delta);
  if (lane < delta) {
    prev = 0;
    if (has && c > 0) {
      const uint2 tp = __ldg(reinterpret_cast<const uint2 *>(src + 32 + 8 * (c - 1)));
      prev = (int64_t)tp.x + (tp.y & 0xFF) + ((tp.y >> 8) & 0xFF) + ((tp.y >> 16) & 0xFF) + (tp.y >> 24);
    }
  }
  if (!has) return true;
  bool ok = off == prev && end <= payload_bytes && s0 <= L + 2 && s1 <= L + 2 && s2 <= L + 2 && s3 <= L + 2;
  if (c == nchunks - 1) ok = ok && end == payload_bytes;
  return ok;
}

// Lane-local variant: loads chunk c-1's entry itself (no warp collective).
__device__ __forceinline__ bool entry_local(const uint8_t *src, int64_t payload_bytes, int nchunks, int c, int L,
                                            int64_t &off, uint32_t &ps) {
  const uint2 te = __ldg(reinterpret_cast<const uint2 *>(src + 32 + 8 * c));
  const uint2 tp = c > 0 ? __ldg(reinterpret_cast<const uint2 *>(src + 32 + 8 * (c - 1))) : make_uint2(0u, 0u);
  off = te.x;
  ps = te.y;
  const int64_t end = off + (int64_t)__dp4a(ps, 0x01010101u, 0u);           // + the four plane sizes
  const int64_t prev = (int64_t)tp.x + (int64_t)__dp4a(tp.y, 0x01010101u, 0u);  // chunk c-1's end
  bool ok = off == prev && end <= payload_bytes && __vcmpgtu4(ps, (uint32_t)(L + 2) * 0x01010101u) == 0u;
  if (c == nchunks - 1) ok = ok && end == payload_bytes;
  return ok;
}

// One warp per 32 x (128 / C) chunks: lane-parallel table validation and
// constant-chunk classification, then constant chunks are filled with one
// 128-bit store per lane and the others decoded warp-cooperatively.
// ---- RLE-64 decode (R-C17): a warp decodes its group of chunks one by one --
// Lane l expands units 2l and 2l+1 (pixels 4l..4l+3).  Tokens t and t + 32
// live in lane t; their start units and payload units come from two packed
// warp scans; each unit finds its token by start markers + a running max.
__device__ __forceinline__ void rle64_decode_group(const DecImage im, const StreamHdr hd, int64_t cb, int w,
                                                int64_t pitch, bool vec, int32_t *status, uint8_t *mark) {
  const int lane = threadIdx.x & 31;
  const int64_t c = cb + lane;
  const bool has = c < hd.nchunks;
  const uint8_t *tab = im.src + 32;
  uint32_t off = 0, size = 0;
  if (has) {
    const uint2 e = __ldg(reinterpret_cast<const uint2 *>(tab + 8 * c));
    off = e.x;
    size = e.y;
  }
  // contiguity: chunk c starts where chunk c-1 ends; the last one ends the payload
  uint64_t prev = __shfl_up_sync(EQC_FULL, (uint64_t)off + size, 1);
  if (lane == 0) {
    prev = 0;
    if (cb > 0) {
      const uint2 e = __ldg(reinterpret_cast<const uint2 *>(tab + 8 * (cb - 1)));
      prev = (uint64_t)e.x + e.y;
    }
  }
  bool ok = !has || (off == prev && size >= 2 && (uint64_t)off + size <= (uint64_t)hd.payload_bytes &&
                     (c != hd.nchunks - 1 || (uint64_t)off + size == (uint64_t)hd.payload_bytes));
  const unsigned bad = __ballot_sync(EQC_FULL, !ok);
  if (bad) {
    if (lane == 0) set_corrupt(status);
    return;
  }
  const int nhere = (int)min((int64_t)32, hd.nchunks - cb);
  for (int i = 0; i < nhere; ++i) {
    const int64_t ci = cb + i;
    const int y = (int)(ci / hd.S), k = (int)(ci - (int64_t)y * hd.S);
    const int L = min(kC, w - k * kC), U = (L + 1) >> 1;
    const uint32_t oi = __shfl_sync(EQC_FULL, off, i), si = __shfl_sync(EQC_FULL, size, i);
    const uint8_t *rec = im.src + hd.payload0 + oi;
    const int ntok = __ldg(rec);
    bool good = ntok >= 1 && ntok <= U && (uint32_t)(1 + ntok) <= si;
    const int t0 = lane, t1 = lane + 32;
    const int c0 = (good && t0 < ntok) ? __ldg(rec + 1 + t0) : 0;
    const int c1 = (good && t1 < ntok) ? __ldg(rec + 1 + t1) : 0;
    const uint32_t l0 = (good && t0 < ntok) ? (c0 & 0x7F) + 1 : 0, l1 = (good && t1 < ntok) ? (c1 & 0x7F) + 1 : 0;
    const uint32_t v0 = l0 | ((c0 & 0x80 ? (l0 ? 1u : 0u) : l0) << 16);
    const uint32_t v1 = l1 | ((c1 & 0x80 ? (l1 ? 1u : 0u) : l1) << 16);
    const uint32_t inc0 = warp_incl_scan_add(v0, lane), inc1 = warp_incl_scan_add(v1, lane);
    const uint32_t tot0 = __shfl_sync(EQC_FULL, inc0, 31), tot1 = __shfl_sync(EQC_FULL, inc1, 31);
    const uint32_t ex0 = inc0 - v0, ex1 = inc1 - v1 + tot0, tot = tot0 + tot1;
    good = good && (int)(tot & 0xFFFFu) == U && 1u + (uint32_t)ntok + 8u * (tot >> 16) == si;
    if (!good) {  // warp-uniform
      if (lane == 0) set_corrupt(status);
      continue;
    }
    // token info: start unit | payload unit << 8 | literal << 16
    const uint32_t info0 = (ex0 & 0xFFFFu) | ((ex0 >> 16) << 8) | ((uint32_t)!(c0 & 0x80) << 16);
    const uint32_t info1 = (ex1 & 0xFFFFu) | ((ex1 >> 16) << 8) | ((uint32_t)!(c1 & 0x80) << 16);
    __syncwarp();
    reinterpret_cast<uint16_t *>(mark)[lane] = 0;
    __syncwarp();
    if (t0 < ntok) mark[ex0 & 0xFFFFu] = (uint8_t)(t0 + 1);
    if (t1 < ntok) mark[ex1 & 0xFFFFu] = (uint8_t)(t1 + 1);
    __syncwarp();
    const uint32_t mm = reinterpret_cast<const uint16_t *>(mark)[lane];
    const int ma = (int)(mm & 0xFFu), mb = (int)(mm >> 8);
    int run = max(ma, mb);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(EQC_FULL, run, d);
      if (lane >= d) run = max(run, o);
    }
    int pre = __shfl_up_sync(EQC_FULL, run, 1);
    if (lane == 0) pre = 0;
    const int ta = max(pre, ma) - 1, tb = max(pre, max(ma, mb)) - 1;
    const uint32_t ia0 = __shfl_sync(EQC_FULL, info0, ta & 31), ia1 = __shfl_sync(EQC_FULL, info1, ta & 31);
    const uint32_t ib0 = __shfl_sync(EQC_FULL, info0, tb & 31), ib1 = __shfl_sync(EQC_FULL, info1, tb & 31);
    const uint32_t ia = ta >= 32 ? ia1 : ia0, ib = tb >= 32 ? ib1 : ib0;
    uint32_t px[4] = {0, 0, 0, 0};
    bool pad_ok = true;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = 2 * lane + h;
      if (u >= U) continue;
      const uint32_t inf = h ? ib : ia;
      const int su = (int)(inf & 0xFFu), sp = (int)((inf >> 8) & 0xFFu);
      const int idx = sp + ((inf >> 16) ? u - su : 0);
      const uint8_t *q = rec + 1 + ntok + 8 * idx;
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        lo |= (uint32_t)__ldg(q + b) << (8 * b);
        hi |= (uint32_t)__ldg(q + 4 + b) << (8 * b);
      }
      px[2 * h] = lo;
      px[2 * h + 1] = hi;
      if (2 * u + 1 >= L && hi != 0) pad_ok = false;  // canonical zero padding
    }
    if (!__all_sync(EQC_FULL, pad_ok)) {
      if (lane == 0) set_corrupt(status);
      continue;
    }
    store_px(im.dst + (int64_t)y * pitch + (int64_t)k * kC, L, lane, vec, px);
  }
}

// RLE-64 streams of a batch (R-C17): launched with the same geometry as
// rle_decode_kernel, each kernel skips the other codec's streams, so each
// keeps its own register allocation.
// Grid-stride over (image, tile): images of the other codec are skipped
// whole after one header read, so a batch without RLE-64 streams costs a
// couple of microseconds.
__global__ void __launch_bounds__(kWarps * 32) rle64_decode_kernel(const __grid_constant__ DecParams p) {
  __shared__ StreamHdr s_hd;
  __shared__ __align__(4) uint8_t s_mark[kWarps][64];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t ntiles = (int64_t)p.count * p.tiles_per_image;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int m = (int)(t / p.tiles_per_image);
    const int64_t lt = t - (int64_t)m * p.tiles_per_image;
    const DecImage im = p.img[m];
    __syncthreads();  // s_hd of the previous tile is no longer read
    if (tid == 0) s_hd = read_header(im.src, im.src_bytes, p.w, p.h, true);  // rle_decode_kernel flags bad ones
    __syncthreads();
    const StreamHdr hd = s_hd;
    if (!hd.ok || hd.flags != EQC_FLAG_RLE64) {
      t += (p.tiles_per_image - 1 - lt) / gridDim.x * gridDim.x;  // skip this image's remaining tiles
      continue;
    }
    const int64_t cb = (lt * kWarps + warp) * kGroup;
    if (cb < hd.nchunks) rle64_decode_group(im, hd, cb, p.w, p.pitch, p.vec != 0, p.status, s_mark[warp]);
  }
}

constexpr int kStage2 = 560;  // >= 15 + 520 record bytes, multiple of 16

__global__ void __launch_bounds__(kWarps * 32, EQC_DEC_MINB) rle_decode_kernel(const __grid_constant__ DecParams p) {
  __shared__ __align__(16) uint8_t stage[kWarps][2][kStage2];  // double buffer: next record in flight
  __shared__ __align__(16) uint16_t info[kWarps][kC];
  __shared__ StreamHdr s_hd;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = (int)(blockIdx.x / p.tiles_per_image);
  const int64_t lt = blockIdx.x - (int64_t)m * p.tiles_per_image;
  const DecImage im = p.img[m];
  if (tid == 0) {
    s_hd = read_header(im.src, im.src_bytes, p.w, p.h, true);
    if (!s_hd.ok) set_corrupt(p.status);
  }
  __syncthreads();
  const StreamHdr hd = s_hd;
  if (!hd.ok) return;
  if (hd.flags == EQC_FLAG_RLE64) return;  // decoded by rle64_decode_kernel (same launch geometry)
  const int C = 1 << hd.log2c;
  const int r = kC / C;
  const bool swz = (hd.flags & EQC_FLAG_SWIZZLE) != 0;
  for (int sub = 0; sub < r; ++sub) {
    const int64_t cb = ((lt * kWarps + warp) * r + sub) * kGroup;
    if (cb >= hd.nchunks) break;
    const int64_t c = cb + lane;
    const bool has = c < hd.nchunks;
    const int y = has ? (int)((uint32_t)c / (uint32_t)hd.S) : 0;
    const int k = has ? (int)c - y * hd.S : 0;
    const int L = has ? min(C, p.w - k * C) : 0;
    int64_t off;
    uint32_t ps;
    const bool ok = entry_lane(im.src, hd.payload_bytes, hd.nchunks, c, has, L, lane, off, ps);
    uint32_t v = 0;
    bool cst = false;
    if (has && ok) {
      cst = probe_const(im.src + hd.payload0 + off, ps, L, v);
      if (cst && swz) v = unswizzle(v);
    }
    const unsigned bad = __ballot_sync(EQC_FULL, has && !ok);
    if (bad && lane == 0) set_corrupt(p.status);
    const int nhere = (int)min((int64_t)kGroup, hd.nchunks - cb);
    // non-constant, valid chunks: their records are staged with 16-byte
    // cp.async, the next one in flight while the current one is decoded
    const unsigned live = nhere == 32 ? EQC_FULL : ((1u << nhere) - 1u);
    unsigned todo = __ballot_sync(EQC_FULL, has && ok && !cst) & ~bad & live;
    auto issue = [&](int j, int b) {
      const int64_t offj = __shfl_sync(EQC_FULL, off, j);
      const uint32_t psj = __shfl_sync(EQC_FULL, ps, j);
      const uint8_t *rec = im.src + hd.payload0 + offj;
      stage_async16(im.src, im.src_bytes, rec, record_quads(rec, psj), reinterpret_cast<uint4 *>(stage[warp][b]), lane);
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int buf = 0;
    if (todo) issue(__ffs(todo) - 1, 0);
    for (int i = 0; i < nhere; ++i) {
      if ((bad >> i) & 1u) continue;
      const int yi = __shfl_sync(EQC_FULL, y, i);
      const int ki = __shfl_sync(EQC_FULL, k, i);
      const int Li = __shfl_sync(EQC_FULL, L, i);
      const bool ci = __shfl_sync(EQC_FULL, (int)cst, i) != 0;
      uint32_t px[4];
      if (ci) {
        const uint32_t vi = __shfl_sync(EQC_FULL, v, i);
#pragma unroll
        for (int j = 0; j < 4; ++j) px[j] = vi;
      } else {
        const int64_t offi = __shfl_sync(EQC_FULL, off, i);
        const uint32_t psi = __shfl_sync(EQC_FULL, ps, i);
        todo &= ~(1u << i);
        if (todo) {  // the next record streams in while this one is decoded
          issue(__ffs(todo) - 1, buf ^ 1);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        const uint8_t *rec = im.src + hd.payload0 + offi;
        bool skip;
        const bool okr = decode_staged(stage[warp][buf] + ((uintptr_t)rec & 15u), psi, Li, lane, info[warp], px,
                                       false, 0u, 0u, skip, swz);
        __syncwarp();  // the buffer is refilled two records later
        buf ^= 1;
        if (!okr) {
          if (lane == 0) set_corrupt(p.status);
          continue;
        }
      }
      store_px(im.dst + (int64_t)yi * p.pitch + (int64_t)ki * C, Li, lane, p.vec != 0 && C == kC, px);
    }
  }
}

// ---------------------------------------------------------------------------
// fused decode + depth composite
// ---------------------------------------------------------------------------

struct FusedParams {
  const uint8_t *src[2 * EQC_MAX_SOURCES];  // colour streams 0..n-1, depth streams n..2n-1
  int64_t src_bytes[2 * EQC_MAX_SOURCES];
  uint32_t *out_color, *out_depth;
  int32_t *status;
  int64_t out_pitch;
  int n, w, h, S;
  float invS;  // 1 / S
  int y0, y1;  // rows composited (a band of the full-frame streams); out_* point at row y0
  int vec;
};

constexpr int kMaxStreams = 2 * EQC_MAX_SOURCES;
#ifndef EQC_FWARPS
#define EQC_FWARPS 4
#endif
constexpr int kFWarps = EQC_FWARPS;  // fused kernel: one chunk position per warp, EQC_FWARPS warps per CTA
constexpr int kPreWords = 1024; // per-warp record prefetch buffer (4 KB)

#ifndef EQC_FPOS
#define EQC_FPOS 16
#endif
constexpr int kFPos = EQC_FPOS;  // chunk positions per CTA (claimed by its warps from a shared counter)

// One chunk position (128 pixels of one row) of the fused decode, by one warp.
//  Phase A (n <= 16: lane q takes stream q; else lane i takes source i's two
//   streams, sources 32.. in a second pass unless ONE): the depth and colour
//   table entries of every stream are validated and probed for constant
//   chunks; if every chunk of the position is constant
//   the depth composite is evaluated on the scalar values (minimum depth, ties
//   to the lowest index) and written with one 128-bit store per lane.
//  Phase B: every non-constant record of the position is prefetched into the
//   warp's buffer (asynchronous copies, one round trip), then decoded depth
//   first: all depth records give the winning source of every pixel, then a
//   source's colour chunk is decoded only if it wins at least one pixel.
// Returns false (warp-uniform) on a corrupt stream (status already set).
template <bool ONE>
__device__ __forceinline__ bool fused_position(const FusedParams &p, int c, int lane, const int64_t *s_pb,
                                               const uint8_t *s_flags, uint8_t *stage, uint16_t *info,
                                               uint4 *pre, uint4 *desc) {
  const int n = p.n;
  const int nch = p.S * p.h;
  const int64_t payload0 = 32 + 8 * (int64_t)nch;
  // y = c / S by a float reciprocal corrected by one (its error is below
  // one row while h < 2^20; invS = 0 selects the integer division)
  int y = p.invS != 0.f ? (int)((float)c * p.invS) : c / p.S;
  int k = c - y * p.S;
  if (k < 0) {
    --y;
    k += p.S;
  } else if (k >= p.S) {
    ++y;
    k -= p.S;
  }
  const int L = min(kC, p.w - k * kC);
  constexpr int NP = ONE ? 1 : 2;
  const int npass = ONE ? 1 : (n + 31) >> 5;
  uint4 ed[NP], ec[NP];  // {offset, plane sizes, value (as coded), constant} per pass
  bool ok = true;
  bool allc = true;
  if (ONE && n <= 16) {
    // lane q validates and probes stream q (colour 0..n-1, depth n..2n-1);
    // lane i < n then takes its depth entry from lane n + i
    const int q = lane;
    uint4 e = make_uint4(0, 0, 0, 1);
    if (q < 2 * n) {
      int64_t o;
      uint32_t ps;
      ok = entry_local(p.src[q], s_pb[q], nch, c, L, o, ps);
      uint32_t v = 0;
      const bool cst = ok && probe_const(p.src[q] + payload0 + o, ps, L, v);
      e = make_uint4((uint32_t)o, ps, v, cst ? 1u : 0u);
      allc = cst;
    }
    const int sl = (n + lane) & 31;
    ed[0] = make_uint4(__shfl_sync(EQC_FULL, e.x, sl), __shfl_sync(EQC_FULL, e.y, sl), __shfl_sync(EQC_FULL, e.z, sl),
                       __shfl_sync(EQC_FULL, e.w, sl));
    ec[0] = e;
    if (lane >= n) ed[0] = ec[0] = make_uint4(0, 0, 0, 1);
  } else {
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      ed[ps] = ec[ps] = make_uint4(0, 0, 0, 1);
      if (ps >= npass) continue;
      const int i = ps * 32 + lane;
      if (i < n) {
        int64_t od, oc;
        uint32_t pd, pc;
        ok = entry_local(p.src[n + i], s_pb[n + i], nch, c, L, od, pd) && ok;
        ok = entry_local(p.src[i], s_pb[i], nch, c, L, oc, pc) && ok;
        uint32_t dv = 0, cv = 0;
        const bool dc = ok && probe_const(p.src[n + i] + payload0 + od, pd, L, dv);
        const bool cc = ok && probe_const(p.src[i] + payload0 + oc, pc, L, cv);
        ed[ps] = make_uint4((uint32_t)od, pd, dv, dc ? 1u : 0u);
        ec[ps] = make_uint4((uint32_t)oc, pc, cv, cc ? 1u : 0u);
        allc = allc && dc && cc;
      }
    }
  }
  if (!__all_sync(EQC_FULL, ok)) {
    if (lane == 0) set_corrupt(p.status);
    return false;
  }
  const int64_t row = (int64_t)(y - p.y0) * p.out_pitch + (int64_t)k * kC;
  if (__all_sync(EQC_FULL, allc)) {
    // every chunk of this position is one value: composite the scalars --
    // minimum depth, ties to the lowest source index
    uint32_t bdv = 0xFFFFFFFFu, bcv = 0;
    int bi = 0x7FFFFFFF;
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      if (ps >= npass) break;
      const int i = ps * 32 + lane;
      const uint32_t dv = i < n ? ed[ps].z : 0xFFFFFFFFu;
      const uint32_t m = __reduce_min_sync(EQC_FULL, dv);
      const unsigned who = __ballot_sync(EQC_FULL, i < n && dv == m);
      const int l0 = __ffs(who) - 1;
      const int ii = ps * 32 + l0;
      const uint32_t cv = __shfl_sync(EQC_FULL, ec[ps].z, l0);
      if (who && (m < bdv || (m == bdv && ii < bi))) {
        bdv = m;
        bcv = cv;
        bi = ii;
      }
    }
    if (s_flags[bi] & EQC_FLAG_SWIZZLE) bcv = unswizzle(bcv);  // (constant colour values are kept as coded)
    const uint32_t pc[4] = {bcv, bcv, bcv, bcv}, pd[4] = {bdv, bdv, bdv, bdv};
    store_px(p.out_color + row, L, lane, p.vec != 0, pc);
    if (p.out_depth) store_px(p.out_depth + row, L, lane, p.vec != 0, pd);
    return true;
  }
  // ---- phase B
  uint32_t bd[4] = {0, 0, 0, 0};
  int bi[4] = {0, 0, 0, 0};
  uint32_t bc[4] = {0, 0, 0, 0};
  uint32_t bm = 0;  // byte j: most significant byte of bd[j]
  const int nv = min(max(L - 4 * lane, 0), 4);
  const uint32_t vinv = nv >= 4 ? 0u : ~((1u << (8 * nv)) - 1u);  // 0xFF bytes: pixels past the chunk
  constexpr int kPreQuads = kPreWords / 4;
  if constexpr (ONE) {
    // Lane i plans source i: 16-byte slots of its depth and colour records in
    // the prefetch buffer, and a descriptor per record in shared memory
    // {offset, plane sizes, value, w}: w bit 0 = constant, bits 1-4 = the
    // record's address mod 16, bits 5.. = slot + 1 (0: not prefetched).
    const bool act = lane < n;
    const int qd = act ? n + lane : 0, qc = act ? lane : 0;
    const uint8_t *recd = p.src[qd] + payload0 + ed[0].x, *recc = p.src[qc] + payload0 + ec[0].x;
    const int nwd = (act && !ed[0].w) ? record_quads(recd, ed[0].y) : 0;
    const int nwc = (act && !ec[0].w) ? record_quads(recc, ec[0].y) : 0;
    const int tot = nwd + nwc;
    const int ex = (int)warp_incl_scan_add((uint32_t)tot, lane) - tot;
    // a record is prefetched if it fits the buffer and its aligned window
    // ends inside the stream (else it is staged when decoded)
    const uintptr_t ad = (uintptr_t)recd & ~(uintptr_t)15, ac = (uintptr_t)recc & ~(uintptr_t)15;
    const bool fd = nwd && ex + nwd <= kPreQuads && ad + 16 * (uintptr_t)nwd <= (uintptr_t)p.src[qd] + p.src_bytes[qd];
    const bool fc = nwc && ex + tot <= kPreQuads && ac + 16 * (uintptr_t)nwc <= (uintptr_t)p.src[qc] + p.src_bytes[qc];
    const int sd0 = fd ? ex : -1, sc0 = fc ? ex + nwd : -1;
    __syncwarp();  // the previous position's readers are done with the buffer and descriptors
    if (act) {
      desc[lane] = make_uint4(ed[0].x, ed[0].y, ed[0].z,
                              ed[0].w ? 1u : ((((uint32_t)(uintptr_t)recd & 15u) << 1) | ((uint32_t)(sd0 + 1) << 5)));
      desc[32 + lane] = make_uint4(ec[0].x, ec[0].y, ec[0].z,
                                   ec[0].w ? 1u : ((((uint32_t)(uintptr_t)recc & 15u) << 1) | ((uint32_t)(sc0 + 1) << 5)));
    }
    const unsigned ncd = __ballot_sync(EQC_FULL, act && !ed[0].w);  // non-constant depth chunks
    // prefetch: the depth records in one round trip now; the colour records
    // of the winning sources only, after the depth pass
    auto prefetch = [&](unsigned m, uintptr_t a, uint32_t sn) {
      while (m) {
        const int i = __ffs(m) - 1;
        m &= m - 1;
        const uintptr_t ai = ((uintptr_t)__shfl_sync(EQC_FULL, (uint32_t)((uint64_t)a >> 32), i) << 32) |
                             __shfl_sync(EQC_FULL, (uint32_t)a, i);
        const uint32_t si = __shfl_sync(EQC_FULL, sn, i);
        const int slot = (int)(si & 0xFFFFu), nq = (int)(si >> 16);  // nq <= 34
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(pre + slot + lane);
        const uintptr_t ga = ai + 16 * (uintptr_t)lane;
        if (lane < nq) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(ga) : "memory");
        if (lane + 32 < nq)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + 512u), "l"(ga + 512) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
    };
    prefetch(__ballot_sync(EQC_FULL, fd), ad, (uint32_t)sd0 | ((uint32_t)nwd << 16));
    // depth pass.  The constant depth chunks are reduced first (minimum, ties
    // to the lowest index: one warp reduction); the non-constant records are
    // then merged in index order, a tie going to the lower index.
    {
      const uint32_t cd = (lane < n && ed[0].w) ? ed[0].z : 0xFFFFFFFFu;
      const uint32_t m = __reduce_min_sync(EQC_FULL, cd);
      const unsigned who = __ballot_sync(EQC_FULL, lane < n && ed[0].w && cd == m);
      const int ci = who ? __ffs(who) - 1 : n;  // n: no constant chunk (any source ties it)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bd[j] = m;
        bi[j] = ci;
      }
      bm = m >> 24 | (m >> 24) << 8 | (m >> 24) << 16 | (m >> 24) << 24;
    }
    for (unsigned todo = ncd; todo; todo &= todo - 1) {
      const int i = __ffs(todo) - 1;
      const uint4 e = desc[i];
      uint32_t d[4];
      const int slot = (int)(e.w >> 5) - 1;
      const uint8_t *r = slot >= 0 ? reinterpret_cast<const uint8_t *>(pre + slot) + ((e.w >> 1) & 15u)
                                   : stage_record(p.src[n + i], p.src_bytes[n + i], p.src[n + i] + payload0 + e.x,
                                                  e.y, lane, stage);
      bool skip = false;
      if (!decode_staged(r, e.y, L, lane, info, d, true, bm, vinv, skip)) {
        if (lane == 0) set_corrupt(p.status);
        return false;
      }
      if (skip) continue;  // deeper than the current best everywhere: cannot win
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool t = d[j] < bd[j] || (d[j] == bd[j] && i < bi[j]);
        bd[j] = t ? d[j] : bd[j];
        bi[j] = t ? i : bi[j];
      }
      bm = __byte_perm(__byte_perm(bd[0], bd[1], 0x0073), __byte_perm(bd[2], bd[3], 0x0073), 0x5410);
    }
    // colour pass: only the sources that win at least one pixel of the chunk
    const unsigned wins = __reduce_or_sync(EQC_FULL, (1u << bi[0]) | (1u << bi[1]) | (1u << bi[2]) | (1u << bi[3]));
    prefetch(__ballot_sync(EQC_FULL, fc) & wins, ac, (uint32_t)sc0 | ((uint32_t)nwc << 16));
    for (unsigned todo = wins; todo; todo &= todo - 1) {
      const int i = __ffs(todo) - 1;
      const uint4 e = desc[32 + i];
      uint32_t col[4];
      if (e.w & 1u) {
        const uint32_t v = (s_flags[i] & EQC_FLAG_SWIZZLE) ? unswizzle(e.z) : e.z;
#pragma unroll
        for (int j = 0; j < 4; ++j) col[j] = v;
      } else {
        const int slot = (int)(e.w >> 5) - 1;
        const uint8_t *r = slot >= 0 ? reinterpret_cast<const uint8_t *>(pre + slot) + ((e.w >> 1) & 15u)
                                     : stage_record(p.src[i], p.src_bytes[i], p.src[i] + payload0 + e.x, e.y, lane,
                                                    stage);
        bool skip;
        if (!decode_staged(r, e.y, L, lane, info, col, false, 0u, 0u, skip, (s_flags[i] & EQC_FLAG_SWIZZLE) != 0)) {
          if (lane == 0) set_corrupt(p.status);
          return false;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bc[j] = bi[j] == i ? col[j] : bc[j];
    }
  } else {
    // n > 32 (two phase-A passes): each record is staged when it is decoded
    for (int i = 0; i < n; ++i) {
      const int li = i & 31;
      const uint4 e1 = i < 32 ? ed[0] : ed[NP - 1];
      const uint32_t dx = __shfl_sync(EQC_FULL, e1.x, li), dy = __shfl_sync(EQC_FULL, e1.y, li),
                     dz = __shfl_sync(EQC_FULL, e1.z, li), dw = __shfl_sync(EQC_FULL, e1.w, li);
      uint32_t d[4];
      if (dw) {
#pragma unroll
        for (int j = 0; j < 4; ++j) d[j] = dz;
      } else {
        bool skip = false;
        const uint8_t *r = stage_record(p.src[n + i], p.src_bytes[n + i], p.src[n + i] + payload0 + dx, dy, lane, stage);
        if (!decode_staged(r, dy, L, lane, info, d, i > 0, bm, vinv, skip)) {
          if (lane == 0) set_corrupt(p.status);
          return false;
        }
        if (skip) continue;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool t = (i == 0) || d[j] < bd[j];
        bd[j] = t ? d[j] : bd[j];
        bi[j] = t ? i : bi[j];
      }
      bm = __byte_perm(__byte_perm(bd[0], bd[1], 0x0073), __byte_perm(bd[2], bd[3], 0x0073), 0x5410);
    }
    for (int i = 0; i < n; ++i) {
      if (!__any_sync(EQC_FULL, bi[0] == i || bi[1] == i || bi[2] == i || bi[3] == i)) continue;
      const int li = i & 31;
      const uint4 e2 = i < 32 ? ec[0] : ec[NP - 1];
      const uint32_t cx = __shfl_sync(EQC_FULL, e2.x, li), cy = __shfl_sync(EQC_FULL, e2.y, li),
                     cz = __shfl_sync(EQC_FULL, e2.z, li), cw = __shfl_sync(EQC_FULL, e2.w, li);
      uint32_t col[4];
      if (cw) {
        const uint32_t v = (s_flags[i] & EQC_FLAG_SWIZZLE) ? unswizzle(cz) : cz;
#pragma unroll
        for (int j = 0; j < 4; ++j) col[j] = v;
      } else {
        bool skip;
        const uint8_t *r = stage_record(p.src[i], p.src_bytes[i], p.src[i] + payload0 + cx, cy, lane, stage);
        if (!decode_staged(r, cy, L, lane, info, col, false, 0u, 0u, skip)) {
          if (lane == 0) set_corrupt(p.status);
          return false;
        }
        if (s_flags[i] & EQC_FLAG_SWIZZLE) {
#pragma unroll
          for (int j = 0; j < 4; ++j) col[j] = unswizzle(col[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bc[j] = bi[j] == i ? col[j] : bc[j];
    }
  }
  store_px(p.out_color + row, L, lane, p.vec != 0, bc);
  if (p.out_depth) store_px(p.out_depth + row, L, lane, p.vec != 0, bd);
  return true;
}

// A CTA takes kFPos consecutive chunk positions; its warps claim them one at
// a time from a shared counter (the stream headers are validated once per
// CTA).  ONE: n <= 32 (one phase-A pass; the entries stay in registers).
template <bool ONE>
__global__ void __launch_bounds__(kFWarps * 32, EQC_FUSED_MINB) depth_rle_kernel(const __grid_constant__ FusedParams p) {
  __shared__ __align__(16) uint8_t stage[kFWarps][kStageBytes];
  __shared__ __align__(16) uint16_t info[kFWarps][kC];
  __shared__ int64_t s_pb[kMaxStreams];
  __shared__ uint8_t s_flags[kMaxStreams];
  __shared__ int s_bad, s_next;
  __shared__ __align__(16) uint32_t s_pre[kFWarps * kPreWords + 4];  // + 16 B: decode_plane_w reads past a record
  __shared__ uint4 s_desc[kFWarps][64];  // per-record descriptors of the warp's position (n <= 32)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = p.n, ns = 2 * n;
  if (tid == 0) {
    s_bad = 0;
    s_next = kFWarps;
  }
  __syncthreads();
  for (int q = tid; q < ns; q += blockDim.x) {
    const bool is_depth = q >= n;
    StreamHdr hd = read_header(p.src[q], p.src_bytes[q], p.w, p.h);
    if (!hd.ok || hd.kind != (is_depth ? 1 : 0) || hd.log2c != kLog2C) s_bad = 1;
    s_pb[q] = hd.payload_bytes;
    s_flags[q] = (uint8_t)hd.flags;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) set_corrupt(p.status);
    return;
  }
  const int c0 = p.y0 * p.S + blockIdx.x * kFPos;
  const int cnt = min(kFPos, p.y1 * p.S - c0);
  uint4 *pre = reinterpret_cast<uint4 *>(s_pre + (size_t)warp * kPreWords);
  for (int j = warp; j < cnt;) {
    int nj = 0;
    if (lane == 0) nj = atomicAdd(&s_next, 1);  // claimed ahead: the atomic overlaps the work
    if (!fused_position<ONE>(p, c0 + j, lane, s_pb, s_flags, stage[warp], info[warp], pre, s_desc[warp])) return;
    j = __shfl_sync(EQC_FULL, nj, 0);
  }
}

inline bool aligned(const void *q, uintptr_t a) { return ((uintptr_t)q & (a - 1)) == 0; }

inline int64_t rle_max_size(int w, int h) {
  const int64_t S = (w + kC - 1) / kC;
  return 32 + 16 * S * (int64_t)h + 4 * (int64_t)w * h;
}

inline int64_t enc_runs_per_image(int w, int h) {
  const int64_t S = (w + kC - 1) / kC;
  return (S * h + kSTChunksPerWarp - 1) / kSTChunksPerWarp;
}

// workspace: run_size[runs] int32, run_off[runs + count] uint32, then (256-byte
// aligned) the record scratch
inline size_t enc_runoff_offset(int64_t runs) { return (size_t)runs * sizeof(int32_t); }
inline size_t enc_ctr_offset(int64_t runs, int count) {
  return enc_runoff_offset(runs) + ((size_t)runs + count) * sizeof(uint32_t);
}
// fused v1 encoder counters: ticket, done runs per image, size of every block
// of 64 runs per image
inline size_t enc_ctr_words(int count, int64_t runs_per_image) {
  return 32 * (size_t)count + (size_t)count * (size_t)((runs_per_image + 63) / 64);  // <= count group tickets
}
inline size_t enc_scratch_offset(int64_t runs, int count) {
  return (enc_ctr_offset(runs, count) + 4 * enc_ctr_words(count, runs / count) + 255) & ~(size_t)255;
}

}  // namespace

extern "C" int64_t image_rle_max_size(int w, int h) {
  if (w <= 0 || h <= 0) return EQC_E_INVALID;
  return rle_max_size(w, h);
}

extern "C" size_t image_rle_workspace_size_batch(int count, int w, int h) {
  if (count <= 0 || w <= 0 || h <= 0) return 0;
  const int64_t runs = (int64_t)count * enc_runs_per_image(w, h);
  // + 256: the record scratch is aligned to 256 bytes in absolute address
  // (its L2 lines are discarded whole), whatever the workspace's alignment
  return enc_scratch_offset(runs, count) + 256 + (size_t)runs * kScratchPerWarp;
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
  const bool r64 = (flags[0] & EQC_FLAG_RLE64) != 0;  // one codec per batch
  for (int i = 0; i < count; ++i) {
    if (!src[i] || !dst[i]) return EQC_E_INVALID;
    if (kind[i] != EQC_KIND_RGBA8 && kind[i] != EQC_KIND_DEPTH32) return EQC_E_INVALID;
    if (flags[i] & ~(EQC_FLAG_SWIZZLE | EQC_FLAG_RLE64)) return EQC_E_INVALID;
    if (((flags[i] & EQC_FLAG_RLE64) != 0) != r64) return EQC_E_INVALID;
    if ((flags[i] & EQC_FLAG_SWIZZLE) && (kind[i] == EQC_KIND_DEPTH32 || r64)) return EQC_E_UNSUPPORTED;
    if (!aligned(dst[i], 8) || !aligned(src[i], 4)) return EQC_E_INVALID;
    vec = vec && aligned(src[i], 16);
    p.img[i] = EncImage{src[i], dst[i], d_sizes + i, kind[i], flags[i]};
  }
  p.pitch = pitch;
  p.S = (w + kC - 1) / kC;
  p.nchunks = (int64_t)p.S * h;
  p.count = count;
  p.w = w;
  p.h = h;
  p.runs_per_image = (int)enc_runs_per_image(w, h);
  p.tiles_per_image = (p.runs_per_image + kEncWarps - 1) / kEncWarps;
  p.vec = vec ? 1 : 0;
  const int64_t runs = (int64_t)count * p.runs_per_image;
  const int64_t tiles = (int64_t)count * p.tiles_per_image;
  if (runs > 0x7FFFFFFFll || p.nchunks > 0x7FFFFFFFll) return EQC_E_INVALID;
  p.run_size = reinterpret_cast<int32_t *>(workspace);
  p.scratch = reinterpret_cast<uint8_t *>(
      ((uintptr_t)workspace + enc_scratch_offset(runs, count) + 255) & ~(uintptr_t)255);
  uint32_t *run_off = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(workspace) + enc_runoff_offset(runs));
  static bool configured = false;
  const size_t smem = sizeof(EncSmem);
  if (!configured) {
    if (cudaFuncSetAttribute(rle_encode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(rle_encode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      return EQC_E_CUDA;
    configured = true;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (!r64) {
    // v1: the batch in groups of images whose raw size stays below
    // EQC_E3_GROUP_MB (so a group's record scratch is still L2-resident when
    // its compaction runs): per group an encoder launch and a compaction
    // launch, after one zeroing of all groups' counters
    const bool full = (w % kC) == 0;
    const bool contig = full && vec && pitch == w;
    static bool configured3 = false;
    const size_t smem3 = sizeof(E3Warp) * kE3Warps;
    if (!configured3) {
      if (cudaFuncSetAttribute(rle_encode3_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem3) != cudaSuccess ||
          cudaFuncSetAttribute(rle_encode3_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem3) != cudaSuccess ||
          cudaFuncSetAttribute(rle_encode3_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem3) != cudaSuccess)
        return EQC_E_CUDA;
      configured3 = true;
    }
    const int R = p.runs_per_image, NB = (R + 63) / 64;
    uint32_t *ctr = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(workspace) + enc_ctr_offset(runs, count));
    EQC_CUDA_TRY(cudaMemsetAsync(ctr, 0, 4 * enc_ctr_words(count, R), st));
    const int64_t img_bytes = 4 * (int64_t)w * h;
    const int per = (int)std::max<int64_t>(1, std::min<int64_t>(count, ((int64_t)EQC_E3_GROUP_MB << 20) / img_bytes));
    for (int g0 = 0; g0 < count; g0 += per) {
      const int gc = std::min(per, count - g0);
      Enc3Params e;
      for (int i = 0; i < gc; ++i) e.img[i] = p.img[g0 + i];
      e.run_size = p.run_size + (int64_t)g0 * R;
      e.scratch = p.scratch + (size_t)g0 * R * kScratchPerWarp;
      e.ctr = ctr + 32 * (g0 / per);  // the group's ticket (its own 128-byte line)
      e.blk = ctr + 32 * ((count + per - 1) / per) + (int64_t)g0 * NB;
      e.pitch = pitch;
      e.nchunks = p.nchunks;
      e.count = gc;
      e.w = w;
      e.h = h;
      e.S = p.S;
      e.R = R;
      e.NB = NB;
      e.invS = 1.0f / (float)p.S;
      e.invR = 1.0f / (float)R;
      e.total_enc = gc * R;
      e.vec = vec ? 1 : 0;
      const int64_t item_ctas = ((int64_t)e.total_enc + kE3Warps - 1) / kE3Warps;
      auto launch = [&](auto kern) {
        const int res = eqc_resident_ctas(kern, kE3Warps * 32, smem3);
        kern<<<(unsigned)std::min<int64_t>(res, item_ctas), kE3Warps * 32, smem3, st>>>(e);
      };
      if (contig) launch(rle_encode3_kernel<true, true>);
      else if (full) launch(rle_encode3_kernel<true, false>);
      else launch(rle_encode3_kernel<false, false>);
      Cmp3Params c;
      for (int i = 0; i < gc; ++i) c.img[i] = e.img[i];
      c.run_size = e.run_size;
      c.blk = e.blk;
      c.scratch = e.scratch;
      c.nchunks = e.nchunks;
      c.count = gc;
      c.w = w;
      c.h = h;
      c.R = R;
      c.NB = NB;
      rle_compact3_kernel<<<dim3((unsigned)((R + kCmp3Warps - 1) / kCmp3Warps), (unsigned)gc), kCmp3Warps * 32, 0,
                            st>>>(c);
    }
    return eqc_launch_status();
  }
  rle_encode_kernel<true><<<(unsigned)tiles, kEncWarps * 32, smem, st>>>(p);
  CompactParams c;
  for (int i = 0; i < count; ++i) c.img[i] = p.img[i];
  rle_runscan_kernel<<<count, 1024, 0, st>>>(p.run_size, run_off, p.runs_per_image);
  c.run_size = p.run_size;
  c.run_off = run_off;
  c.scratch = p.scratch;
  c.nchunks = p.nchunks;
  c.w = w;
  c.h = h;
  c.runs_per_image = p.runs_per_image;
  c.groups_per_image = (p.runs_per_image + kCompactWarps - 1) / kCompactWarps;
  rle_compact_kernel<<<(unsigned)(count * c.groups_per_image), kCompactWarps * 32, 0, st>>>(c);
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

extern "C" int image_decompress_rle_batch(int count, const uint8_t *const *src, const int64_t *src_bytes,
                                          uint32_t *const *dst, int64_t pitch, int w, int h,
                                          int32_t *d_status, void *stream) {
  if (count < 1 || count > kMaxBatch || !src || !src_bytes || !dst || !d_status) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w) return EQC_E_INVALID;
  DecParams p;
  bool vec = (pitch % 4) == 0;
  for (int i = 0; i < count; ++i) {
    if (!src[i] || !dst[i] || src_bytes[i] < 32) return EQC_E_INVALID;
    if (!aligned(src[i], 8) || !aligned(dst[i], 4)) return EQC_E_INVALID;
    vec = vec && aligned(dst[i], 16);
    p.img[i] = DecImage{src[i], dst[i], src_bytes[i]};
  }
  p.status = d_status;
  p.pitch = pitch;
  p.count = count;
  p.w = w;
  p.h = h;
  p.tiles_per_image = ((int64_t)((w + kC - 1) / kC) * h + kWarps * kGroup - 1) / (kWarps * kGroup);
  p.vec = vec ? 1 : 0;
  const int64_t grid = (int64_t)count * p.tiles_per_image;
  if (grid > 0x7FFFFFFFll) return EQC_E_INVALID;
  rle_decode_kernel<<<(unsigned)grid, kWarps * 32, 0, (cudaStream_t)stream>>>(p);
  rle64_decode_kernel<<<(unsigned)std::min<int64_t>(grid, (int64_t)eqc_num_sms() * 32), kWarps * 32, 0,
                        (cudaStream_t)stream>>>(p);
  return eqc_launch_status();
}

extern "C" int image_decompress_rle(const uint8_t *src, int64_t src_bytes, uint32_t *dst, int64_t pitch,
                                    int w, int h, int32_t *d_status, void *stream) {
  const uint8_t *s[1] = {src};
  uint32_t *d[1] = {dst};
  return image_decompress_rle_batch(1, s, &src_bytes, d, pitch, w, h, d_status, stream);
}

// Internal (compose.cu): compositor_depth_rle over rows [y0, y1) of the
// full-frame streams (any device / peer-mapped pointers); out_* point at row y0.
int eqc_depth_rle_band(int n, const uint8_t *const *color_rle, const uint8_t *const *depth_rle,
                       const int64_t *color_bytes, const int64_t *depth_bytes, int w, int h, int y0, int y1,
                       uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch, int32_t *d_status,
                       void *stream);

extern "C" int compositor_depth_rle(int n, const uint8_t *const *color_rle, const uint8_t *const *depth_rle,
                                    const int64_t *color_bytes, const int64_t *depth_bytes, int w, int h,
                                    uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch,
                                    int32_t *d_status, void *stream) {
  return eqc_depth_rle_band(n, color_rle, depth_rle, color_bytes, depth_bytes, w, h, 0, h, out_color, out_depth,
                            out_pitch, d_status, stream);
}

int eqc_depth_rle_band(int n, const uint8_t *const *color_rle, const uint8_t *const *depth_rle,
                       const int64_t *color_bytes, const int64_t *depth_bytes, int w, int h, int y0, int y1,
                       uint32_t *out_color, uint32_t *out_depth, int64_t out_pitch, int32_t *d_status,
                       void *stream) {
  if (y0 < 0 || y1 > h || y0 > y1) return EQC_E_INVALID;
  if (y0 == y1) return EQC_OK;
  if (n < 1 || n > EQC_MAX_SOURCES || !color_rle || !depth_rle || !color_bytes || !depth_bytes || !out_color ||
      !d_status)
    return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || out_pitch < w) return EQC_E_INVALID;
  FusedParams p;
  for (int i = 0; i < n; ++i) {
    if (!color_rle[i] || !depth_rle[i] || color_bytes[i] < 32 || depth_bytes[i] < 32) return EQC_E_INVALID;
    if (!aligned(color_rle[i], 8) || !aligned(depth_rle[i], 8)) return EQC_E_INVALID;
    p.src[i] = color_rle[i];
    p.src[n + i] = depth_rle[i];
    p.src_bytes[i] = color_bytes[i];
    p.src_bytes[n + i] = depth_bytes[i];
  }
  if (!aligned(out_color, 4) || (out_depth && !aligned(out_depth, 4))) return EQC_E_INVALID;
  p.out_color = out_color;
  p.out_depth = out_depth;
  p.status = d_status;
  p.out_pitch = out_pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.S = (w + kC - 1) / kC;
  p.invS = h < (1 << 20) ? 1.0f / (float)p.S : 0.f;
  p.y0 = y0;
  p.y1 = y1;
  p.vec = ((out_pitch % 4) == 0 && aligned(out_color, 16) && (!out_depth || aligned(out_depth, 16))) ? 1 : 0;
  const int64_t grid = ((int64_t)p.S * (y1 - y0) + kFPos - 1) / kFPos;
  if (grid > 0x7FFFFFFFll || (int64_t)p.S * h > 0x7FFFFFFFll) return EQC_E_INVALID;
  if (n <= 32)
    depth_rle_kernel<true><<<(unsigned)grid, kFWarps * 32, 0, (cudaStream_t)stream>>>(p);
  else
    depth_rle_kernel<false><<<(unsigned)grid, kFWarps * 32, 0, (cudaStream_t)stream>>>(p);
  return eqc_launch_status();
}

// Load every kernel of this file now (see eqc_preload_composite).
int eqc_preload_rle() {
  cudaFuncAttributes a;
  bool ok = true;
  ok = ok && cudaFuncGetAttributes(&a, rle_encode_kernel<true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, rle_runscan_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, rle_compact_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, rle_compact3_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, rle_encode3_kernel<true, true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, rle_encode3_kernel<true, false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, rle_encode3_kernel<false, false>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, rle64_decode_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, rle_decode_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, depth_rle_kernel<true>) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, depth_rle_kernel<false>) == cudaSuccess;
  return ok ? EQC_OK : EQC_E_CUDA;
}
