// rle.cuh -- warp-level RLE-BP v1 chunk encoder/decoder (sm_100a).
//
// Thesis: per-component RLE, "four independent RLE-compressed output streams"
// (P:2402-2405); bit-swizzle preconditioner grouping bits "by significance"
// (P:2407-2425); data decomposition of the image into independently coded
// sub-images.  Wire format: reading R-C8, DESIGN.md §5.
//
// GPU mapping: one warp codes one 128-pixel row chunk.  Lane l
// owns pixels 4l..4l+3 (one 128-bit load), so the four byte planes of the
// chunk are processed SIMD-within-a-word: byte p of every register word is
// plane p.  Run detection is a per-byte equality flag (bit 7 of each byte);
// the REPEAT cover of a byte is local (a byte is in a run of >= 3 iff one of
// the three length-3 windows through it is constant), token starts and
// payload-emitting bytes follow from the cover and one neighbour, and all
// four planes' token / payload counts are prefix-summed at once as packed
// bytes in two warp scans.
#pragma once

#include "eqc_common.cuh"

namespace eqc_rle {

constexpr uint32_t kMagic = 0x4C525145u;  // "EQRL"
constexpr int kVersion = 1;
constexpr int kLog2C = 7;
constexpr int kC = 128;
constexpr int kStageBytes = 544;  // >= 4 planes * (128 + 2) bytes, 16-aligned
constexpr int kTokBytes = 512;    // token-start scratch: 4 planes * 128

// ---- swizzle (R-C9): out bit 4b + (3 - c) = bit b of channel c ------------
// As a permutation of the 5 bit-index bits: (c1 c0 b2 b1 b0) -> (b2 b1 b0 ~c1
// ~c0), a 5-cycle of index slots.  A byte permute that swaps bytes 0 and 3
// (complementing the byte index and exchanging its two bits, PRMT 0x0213)
// leaves a 3-cycle and a transposition of index slots: three delta swaps
// (slots 0 <-> 2, 0 <-> 4, 1 <-> 3), 13 operations instead of 17 for the
// plain rotation (four transpositions after the byte reversal).
__device__ __forceinline__ uint32_t delta_swap(uint32_t x, int d, uint32_t m) {
  uint32_t t = ((x >> d) ^ x) & m;
  return x ^ t ^ (t << d);
}
__device__ __forceinline__ uint32_t swizzle(uint32_t v) {
  v = __byte_perm(v, 0, 0x0213);
  v = delta_swap(v, 3, 0x0A0A0A0Au);   // index slots 0 <-> 2
  v = delta_swap(v, 15, 0x0000AAAAu);  // 0 <-> 4
  v = delta_swap(v, 6, 0x00CC00CCu);   // 1 <-> 3
  return v;
}
__device__ __forceinline__ uint32_t unswizzle(uint32_t v) {
  v = delta_swap(v, 6, 0x00CC00CCu);
  v = delta_swap(v, 15, 0x0000AAAAu);
  v = delta_swap(v, 3, 0x0A0A0A0Au);
  return __byte_perm(v, 0, 0x0213);
}

__device__ __forceinline__ uint32_t bytep(uint32_t v, int p) { return (v >> (8 * p)) & 0xFFu; }

// Position-validity flag word for position i of a chunk of length L.
__device__ __forceinline__ uint32_t vflag(bool ok) { return ok ? 0x80808080u : 0u; }

struct EncodeOut {
  int size;           // chunk record bytes
  uint32_t psizes;    // byte p = plane p record size
};

// Encode one chunk.  Lane `lane` holds the RAW pixels px[0..3] (positions
// 4*lane + j, valid while < L); `swz` applies the swizzle preconditioner.
// Writes the chunk record (planes 0..3 concatenated) into `st` (any byte
// alignment) and returns its size.  `tp` is per-warp scratch of kTokBytes.
//
// Plane classes (warp-uniform): CONSTANT (one REPEAT of L, 3 bytes),
// LITERAL-ONLY (no run of >= 3: one LITERAL, L + 2 bytes, the bytes in
// order), GENERAL (scatter of token starts and payload bytes by prefix
// counts).  Chunks whose pixels are all equal never get here: the caller
// emits them directly (chunk_is_constant / emit_constant_record).
template <bool FULL>
__device__ __forceinline__ EncodeOut encode_chunk_t(uint32_t px[4], int L_, int lane, bool swz, uint8_t *st,
                                                    uint8_t *tp) {
  // FULL: a 128-pixel chunk; the position-validity masks fold to constants
  const int L = FULL ? kC : L_;
  const int i0 = 4 * lane;
  if (swz) {
#pragma unroll
    for (int j = 0; j < 4; ++j) px[j] = swizzle(px[j]);
  }
  // ---- neighbours: W[-2], W[-1] from the previous lane, W[4], W[5] from the next
  const uint32_t wm2 = __shfl_up_sync(EQC_FULL, px[2], 1);
  const uint32_t wm1 = __shfl_up_sync(EQC_FULL, px[3], 1);
  const uint32_t wp4 = __shfl_down_sync(EQC_FULL, px[0], 1);
  const uint32_t wp5 = __shfl_down_sync(EQC_FULL, px[1], 1);
  // e[k] (position i0+k-1, k = 0..6): byte equals its predecessor, for
  // 1 <= position < L (no predecessor at the chunk start; nothing beyond L).
  uint32_t e[7];
  {
    const uint32_t W[8] = {wm2, wm1, px[0], px[1], px[2], px[3], wp4, wp5};
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      const int pos = i0 + k - 1;
      e[k] = bytes_eq(W[k + 1], W[k]) & vflag(pos >= 1 && pos < L);
    }
  }
  // p3[k] = e[k] & e[k+1]: window (pos-1, pos, pos+1) constant, pos = i0+k-1
  uint32_t p3[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) p3[k] = e[k] & e[k + 1];
  // R[j]: position i0+j lies in a run of >= 3 (REPEAT cover)
  uint32_t R[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) R[j] = p3[j] | p3[j + 1] | p3[j + 2];
  // ---- plane classes
  uint32_t allE = 0x80808080u, anyR = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (i0 + j >= 1 && i0 + j < L) allE &= e[j + 1];
    anyR |= R[j];
  }
  const uint32_t cst = __reduce_and_sync(EQC_FULL, allE);  // bit 7 of byte p: plane p constant
  const uint32_t rep = __reduce_or_sync(EQC_FULL, anyR);   // bit 7 of byte p: plane p has a REPEAT
  // class per plane: 0 literal-only, 1 constant, 2 general
  int cls[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const bool r = (rep >> (8 * p + 7)) & 1u, c = (cst >> (8 * p + 7)) & 1u;
    cls[p] = !r ? 0 : (c ? 1 : 2);
  }
  const bool any_general = cls[0] == 2 || cls[1] == 2 || cls[2] == 2 || cls[3] == 2;
  uint32_t nibT = 0, nibE = 0, nibR = 0, exT = 0, exE = 0, totT = 0, totE = 0;
  if (any_general) {
    uint32_t Rprev = __shfl_up_sync(EQC_FULL, R[3], 1);
    if (lane == 0) Rprev = 0;
    uint32_t T[4], E[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t valid = vflag(i0 + j < L);
      const uint32_t rp = (j == 0) ? Rprev : R[j - 1];
      const uint32_t first = vflag(i0 + j == 0);
      T[j] = (first | (R[j] ^ rp) | (R[j] & rp & ~e[j + 1])) & valid;
      E[j] = (~R[j] | T[j]) & valid;
    }
    nibT = ((T[0] >> 7) | (T[1] >> 6) | (T[2] >> 5) | (T[3] >> 4)) & 0x0F0F0F0Fu;
    nibE = ((E[0] >> 7) | (E[1] >> 6) | (E[2] >> 5) | (E[3] >> 4)) & 0x0F0F0F0Fu;
    nibR = ((R[0] >> 7) | (R[1] >> 6) | (R[2] >> 5) | (R[3] >> 4)) & 0x0F0F0F0Fu;
    const uint32_t cT = bytes_popc_nibble(nibT);
    const uint32_t cE = bytes_popc_nibble(nibE);
    const uint32_t incT = warp_incl_scan_add(cT, lane);
    const uint32_t incE = warp_incl_scan_add(cE, lane);
    totT = __shfl_sync(EQC_FULL, incT, 31);
    totE = __shfl_sync(EQC_FULL, incE, 31);
    exT = incT - cT;
    exE = incE - cE;
  }
  int size[4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
    size[p] = cls[p] == 0 ? L + 2 : cls[p] == 1 ? 3 : 1 + (int)bytep(totT, p) + (int)bytep(totE, p);
  const int b0 = 0, b1 = size[0], b2 = b1 + size[1], b3 = b2 + size[2], b4 = b3 + size[3];
  // ---- emit each plane by class
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int base = p == 0 ? b0 : p == 1 ? b1 : p == 2 ? b2 : b3;
    if (cls[p] == 1) {
      if (lane == 0) {
        st[base] = 1;
        st[base + 1] = (uint8_t)(0x80 | (L - 1));
        st[base + 2] = (uint8_t)bytep(px[0], p);
      }
    } else if (cls[p] == 0) {
      if (lane == 0) {
        st[base] = 1;
        st[base + 1] = (uint8_t)(L - 1);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i0 + j < L) st[base + 2 + i0 + j] = (uint8_t)bytep(px[j], p);
    } else {
      const uint32_t t = (nibT >> (8 * p)) & 15u, ev = (nibE >> (8 * p)) & 15u, r = (nibR >> (8 * p)) & 15u;
      int tk = (int)bytep(exT, p);
      int ek = base + 1 + (int)bytep(totT, p) + (int)bytep(exE, p);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if ((t >> j) & 1u) {
          tp[p * kC + tk] = (uint8_t)((i0 + j) | (((r >> j) & 1u) << 7));
          ++tk;
        }
        if ((ev >> j) & 1u) {
          st[ek] = (uint8_t)bytep(px[j], p);
          ++ek;
        }
      }
      if (lane == 0) st[base] = (uint8_t)bytep(totT, p);
    }
  }
  if (any_general) {
    __syncwarp();
    // ---- ctrl bytes of GENERAL planes: token length = next start - this start
    const int g0 = cls[0] == 2 ? (int)bytep(totT, 0) : 0;
    const int g1 = cls[1] == 2 ? (int)bytep(totT, 1) : 0;
    const int g2 = cls[2] == 2 ? (int)bytep(totT, 2) : 0;
    const int g3 = cls[3] == 2 ? (int)bytep(totT, 3) : 0;
    const int n0 = g0, n1 = n0 + g1, n2 = n1 + g2, n3 = n2 + g3;
    // token q of the concatenated lists: plane = last p with q >= n_{p-1};
    // per plane, tb = token scratch base - first q, sb = stage base - first q
    for (int q = lane; q < n3; q += 32) {
      int tb = 0, sb = b0 + 1, ne = n0;
      if (q >= n0) tb = kC - n0, sb = b1 + 1 - n0, ne = n1;
      if (q >= n1) tb = 2 * kC - n1, sb = b2 + 1 - n1, ne = n2;
      if (q >= n2) tb = 3 * kC - n2, sb = b3 + 1 - n2, ne = n3;
      const uint32_t a = tp[tb + q];
      const int next = (q + 1 < ne) ? (int)(tp[tb + q + 1] & 0x7Fu) : L;
      const int len = next - (int)(a & 0x7Fu);
      st[sb + q] = (uint8_t)((a & 0x80u) | (uint32_t)(len - 1));
    }
  }
  __syncwarp();
  const uint32_t ps = (uint32_t)size[0] | ((uint32_t)size[1] << 8) | ((uint32_t)size[2] << 16) |
                      ((uint32_t)size[3] << 24);
  return EncodeOut{b4, ps};
}

// ---- RLE-64 (reading R-C17): 64-bit units = pixel pairs -------
// Lane l holds units a = 2l (px0, px1) and b = 2l + 1 (px2, px3); positions at
// or beyond L hold 0 (the odd tail unit's high half is 0 by definition).
// Maximal runs of >= 2 equal units -> REPEAT (ctrl 0x80 | (len - 1), one
// 8-byte unit), other maximal spans -> LITERAL (ctrl len - 1, the units).
// Record = [ntok][ctrl x ntok][payload]; returns {size, size}.
__device__ __forceinline__ bool u64eq(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
  return a0 == b0 && a1 == b1;
}

__device__ __forceinline__ EncodeOut encode_chunk64(const uint32_t px[4], int L, int lane, uint8_t *st, uint8_t *tp) {
  const int U = (L + 1) >> 1;
  const int ua = 2 * lane, ub = ua + 1;
  const bool va = ua < U, vb = ub < U;
  // neighbours: unit a-1 (previous lane's b), unit b+1 (next lane's a)
  const uint32_t pm0 = __shfl_up_sync(EQC_FULL, px[2], 1), pm1 = __shfl_up_sync(EQC_FULL, px[3], 1);
  const uint32_t pn0 = __shfl_down_sync(EQC_FULL, px[0], 1), pn1 = __shfl_down_sync(EQC_FULL, px[1], 1);
  const bool ea = va && ua >= 1 && u64eq(px[0], px[1], pm0, pm1);    // a == a-1
  const bool eb = vb && u64eq(px[2], px[3], px[0], px[1]);           // b == a
  const bool en = (ub + 1 < U) && u64eq(pn0, pn1, px[2], px[3]);     // b+1 == b
  const bool Ra = va && (ea || eb), Rb = vb && (eb || en);           // inside a run of >= 2
  bool Rp = __shfl_up_sync(EQC_FULL, Rb, 1);                          // R of unit a-1
  if (lane == 0) Rp = false;
  const bool Ta = va && (ua == 0 || Ra != Rp || (Ra && Rp && !ea));
  const bool Tb = vb && (Rb != Ra || (Rb && Ra && !eb));
  const bool Ea = va && (!Ra || Ta), Eb = vb && (!Rb || Tb);
  const uint32_t cnt = (uint32_t)Ta + (uint32_t)Tb + (((uint32_t)Ea + (uint32_t)Eb) << 16);
  const uint32_t inc = warp_incl_scan_add(cnt, lane);
  const uint32_t tot = __shfl_sync(EQC_FULL, inc, 31);
  const uint32_t ex = inc - cnt;
  const int ntok = (int)(tot & 0xFFFFu), npay = (int)(tot >> 16);
  int tk = (int)(ex & 0xFFFFu), ek = 1 + ntok + 8 * (int)(ex >> 16);
  if (Ta) tp[tk++] = (uint8_t)(ua | ((uint32_t)Ra << 7));
  if (Tb) tp[tk] = (uint8_t)(ub | ((uint32_t)Rb << 7));
  if (Ea) {
#pragma unroll
    for (int q = 0; q < 8; ++q) st[ek + q] = (uint8_t)((q < 4 ? px[0] : px[1]) >> (8 * (q & 3)));
    ek += 8;
  }
  if (Eb) {
#pragma unroll
    for (int q = 0; q < 8; ++q) st[ek + q] = (uint8_t)((q < 4 ? px[2] : px[3]) >> (8 * (q & 3)));
  }
  if (lane == 0) st[0] = (uint8_t)ntok;
  __syncwarp();
  for (int q = lane; q < ntok; q += 32) {
    const uint32_t a = tp[q];
    const int next = q + 1 < ntok ? (int)(tp[q + 1] & 0x7Fu) : U;
    st[1 + q] = (uint8_t)((a & 0x80u) | (uint32_t)(next - (int)(a & 0x7Fu) - 1));
  }
  __syncwarp();
  const int size = 1 + ntok + 8 * npay;
  return EncodeOut{size, (uint32_t)size};
}

__device__ __forceinline__ EncodeOut encode_chunk(uint32_t px[4], int L, int lane, bool swz, uint8_t *st,
                                                  uint8_t *tp) {
  return L == kC ? encode_chunk_t<true>(px, L, lane, swz, st, tp) : encode_chunk_t<false>(px, L, lane, swz, st, tp);
}

// Whole-chunk constancy test on the RAW pixels (the swizzle is a bijection,
// so this equals constancy after it); v0 receives the value.
__device__ __forceinline__ bool chunk_is_constant(const uint32_t px[4], int L, int lane, uint32_t &v0) {
  const int i0 = 4 * lane;
  v0 = __shfl_sync(EQC_FULL, px[0], 0);
  bool same = true;
#pragma unroll
  for (int j = 0; j < 4; ++j) same = same && (i0 + j >= L || px[j] == v0);
  return __all_sync(EQC_FULL, same) && L >= 3;
}

// The 12-byte record of a constant chunk (four planes [01][0x80|(L-1)][v_p]),
// written straight to global memory by lanes 0..11 (one byte each).
__device__ __forceinline__ void emit_constant_record(uint8_t *g, uint32_t v, int L, int lane) {
  if (lane < 12) {
    const int p = lane / 3, q = lane - 3 * p;
    const uint32_t b = q == 0 ? 1u : q == 1 ? (0x80u | (uint32_t)(L - 1)) : bytep(v, p);
    g[lane] = (uint8_t)b;
  }
}

// Copy the warp's staged record (st[0..size)) to global bytes [g, g+size).
// Interior 4-byte-aligned words are stored whole (funnel-shifted out of the
// staging words); the <= 3 head and <= 3 tail bytes are byte stores.
__device__ __forceinline__ void store_record(uint8_t *g, const uint8_t *st, int size, int lane) {
  const uintptr_t ga = (uintptr_t)g;
  const uintptr_t first_w = (ga + 3) & ~(uintptr_t)3;
  const uintptr_t end = ga + (uintptr_t)size;
  const uintptr_t last_w = end & ~(uintptr_t)3;
  if (first_w >= last_w) {  // no whole word: all bytes individually
    for (int k = lane; k < size; k += 32) g[k] = st[k];
    return;
  }
  const int head = (int)(first_w - ga);
  const int tail = (int)(end - last_w);
  if (lane < head) g[lane] = st[lane];
  if (lane >= 8 && lane < 8 + tail) g[(int)(last_w - ga) + lane - 8] = st[(int)(last_w - ga) + lane - 8];
  const int nw = (int)((last_w - first_w) >> 2);
  const uint32_t *st32 = reinterpret_cast<const uint32_t *>(st);
  const int sh = head & 3;  // staging byte offset of each word's first byte, mod 4
  uint32_t *gw = reinterpret_cast<uint32_t *>(first_w);
  for (int k = lane; k < nw; k += 32) {
    const int q = head + 4 * k;  // staging index of the word's first byte
    const uint32_t lo = st32[q >> 2];
    const uint32_t hi = sh ? st32[(q >> 2) + 1] : 0u;
    gw[k] = sh ? __funnelshift_r(lo, hi, 8 * sh) : lo;
  }
}

// ---- decoder ---------------------------------------------------------------

// ---- word-per-lane decoder --------------------------------------------------
// A plane record r[0..size) = [ntok][ctrl x ntok][payload] (R-C8).  Position i
// takes payload byte r[ntok + A(i)], where A(i) counts the positions k <= i
// that advance the payload: token starts and positions inside a LITERAL token.
// The advancing positions are disjoint ranges [s, e) (literal: e = s + len,
// repeat: e = s + 1); with S = {s} and E = {e} as 128-bit masks their mask is
// the integer E - S (an end at 128 wraps to 0).  Lane l forms the word of
// positions 4l..4l+3 with one byte permute of the 8 payload bytes at its first
// position's index: byte j is offset by the advancing positions among
// 4l+1..4l+j (bits 1..j of the lane's nibble of the mask).

// PRMT selector offsets (byte j: o_j << 4j) for the advance nibble `nib`.
__device__ __forceinline__ uint32_t adv_sel(uint32_t nib) {
  // byte t of the table = o2 | o3 << 4 for t = nib >> 1 = (b1, b2, b3):
  // o2 = b1 + b2, o3 = o2 + b3
  const uint32_t hi = __byte_perm(0x22111100u, 0x32212110u, nib >> 1);
  return ((nib & 2u) << 3) | (hi << 8);
}

// Bytes r[pi + o_j], j = 0..3 (o_j from the selector offsets): two aligned
// word loads and a permute.
__device__ __forceinline__ uint32_t ld_window(const uint8_t *r, int pi, uint32_t sel) {
  const uint8_t *b = r + pi;
  const uint32_t mis = (uint32_t)(uintptr_t)b & 3u;
  // pointer arithmetic (not an integer round trip) keeps the shared-memory
  // address space visible to the compiler: LDS, not generic loads
  const uint32_t *w = reinterpret_cast<const uint32_t *>(b - mis);
  return __byte_perm(w[0], w[1], mis * 0x1111u + sel);
}

// Word of positions 4*lane .. 4*lane+3 (byte j = position 4*lane + j; bytes of
// positions >= L unspecified) of the plane record r[0..size), size <= L + 2.
// `ok` is cleared if the record is malformed (warp-uniform); a malformed
// record is still read only inside r[0 .. size + 8) (callers' buffers keep 8
// bytes of slack past every record), so validation is deferred to one test
// per record.  `info`: per-warp scratch of 128 uint16 (records of more than
// 32 tokens).
__device__ __forceinline__ uint32_t decode_plane_w(const uint8_t *r, int size, int L, int lane, bool &ok,
                                                   uint16_t *info) {
  // (size 0: ntok is a byte of the next plane or the slack.)  The checks of
  // each path below imply size >= 2, 1 <= ntok, 1 + ntok <= size, ntok <= L:
  // a path that sums all ntok lengths to L and their payload bytes to
  // size - 1 - ntok cannot accept a record that breaks one of them.
  const int ntok = r[0];
  const int i0 = 4 * lane;
  uint32_t nib;  // advancing positions among 4*lane .. 4*lane+3
  int cntb;      // advancing positions before 4*lane
  if (ntok <= 1) {  // single-token fast paths
    const int c = r[1];
    const bool rep = (c & 0x80) != 0;
    ok = ok && ntok == 1 && (c & 0x7F) + 1 == L && size == (rep ? 3 : 2 + L);
    if (rep) return (uint32_t)r[2] * 0x01010101u;
    // (lanes past L, and a malformed size: reads stay within r[0, size + 8))
    return ld_window(r, min(2 + min(i0, L), size), 0x3210u);
  }
  if (ntok <= 4) {
    // token boundaries computed by every lane (uniform); the lane's nibble and
    // count are sums over the <= 4 ranges
    int pos = 0, pay = 0;
    nib = 0;
    cntb = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (t < ntok) {
        const int c = r[1 + t];
        const int len = (c & 0x7F) + 1;
        const bool lit = !(c & 0x80);
        const int e = lit ? pos + len : pos + 1;
        const int lo = min(max(pos - i0, 0), 4), hi = min(max(e - i0, 0), 4);
        nib |= (1u << hi) - (1u << lo);
        cntb += max(min(e, i0) - pos, 0);
        pos += len;
        pay += lit ? len : 1;
      }
    }
    ok = ok && pos == L && pay == size - 1 - ntok;
  } else {
    uint32_t A[4];
    if (ntok <= 32) {
      // lane t holds token t: starts and payload sums by one packed warp
      // scan, then the mask words by OR-reductions of the token ranges
      const bool act = lane < ntok && 1 + lane < size;  // (the second test only for a malformed record)
      const int c = act ? r[1 + lane] : 0;
      const int len = act ? (c & 0x7F) + 1 : 0;
      const bool lit = !(c & 0x80);
      const int pay = lit ? len : 1;
      const uint32_t packed = (uint32_t)len | ((uint32_t)pay << 16);
      const uint32_t inc = warp_incl_scan_add(packed, lane);
      const uint32_t tot = __shfl_sync(EQC_FULL, inc, 31);
      ok = ok && (int)(tot & 0xFFFFu) == L && (int)(tot >> 16) == size - 1 - ntok;
      const int s = (int)((inc - packed) & 0xFFFFu);
      const int e = lit ? s + len : s + 1;  // (an absent token: e = s, an empty range)
      // word w of the mask: OR over the tokens of [s, e) within the word
      // (mask_ge(n) = ~0 << n, 0 for n >= 32: a clamped funnel shift)
#pragma unroll
      for (int w = 0; w < 4; ++w)
        A[w] = __reduce_or_sync(EQC_FULL, __funnelshift_lc(0u, ~0u, max(s - 32 * w, 0)) &
                                              ~__funnelshift_lc(0u, ~0u, max(e - 32 * w, 0)));
    } else {
      // lane l holds tokens 4l .. 4l+3 (of at most 128: ntok <= L); S and E
      // as byte markers in the scratch, gathered into words by shuffles
      const int nt = min(min(ntok, L), size - 1);  // (reads stay inside a malformed record)
      ok = ok && ntok <= L;                        // (tokens past L are not summed)
      int sl = 0, sp = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = i0 + k;
        if (t < nt) {
          const int c = r[1 + t];
          const int len = (c & 0x7F) + 1;
          sl += len;
          sp += (c & 0x80) ? 1 : len;
        }
      }
      const uint32_t packed = (uint32_t)sl | ((uint32_t)sp << 16);
      const uint32_t inc = warp_incl_scan_add(packed, lane);
      const uint32_t tot = __shfl_sync(EQC_FULL, inc, 31);
      ok = ok && (int)(tot & 0xFFFFu) == L && (int)(tot >> 16) == size - 1 - ntok;
      uint8_t *mS = reinterpret_cast<uint8_t *>(info), *mE = mS + 128;
      __syncwarp();  // the scratch may still be read by a previous plane
      reinterpret_cast<uint2 *>(info)[lane] = make_uint2(0u, 0u);
      __syncwarp();
      int spos = (int)((inc - packed) & 0xFFFFu);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = i0 + k;
        if (t < nt) {
          const int c = r[1 + t];
          const int len = (c & 0x7F) + 1;
          const int e = (c & 0x80) ? spos + 1 : spos + len;
          if (spos < 128) mS[spos] = 1;
          if (e < 128) mE[e] = 1;
          spos += len;
        }
      }
      __syncwarp();
      // lane l reads its 4 marker bytes (positions 4l..4l+3) of each mask
      const uint32_t ms = reinterpret_cast<const uint32_t *>(mS)[lane];
      const uint32_t me = reinterpret_cast<const uint32_t *>(mE)[lane];
      // bytes 0/1 -> nibble (byte j -> bit j)
      const uint32_t ns = (ms | (ms >> 7) | (ms >> 14) | (ms >> 21)) & 0xFu;
      const uint32_t ne = (me | (me >> 7) | (me >> 14) | (me >> 21)) & 0xFu;
      // word w of a mask = nibbles of lanes 8w .. 8w+7
      uint32_t vs = ns << (4 * (lane & 7)), ve = ne << (4 * (lane & 7));
#pragma unroll
      for (int d = 1; d < 8; d <<= 1) {
        vs |= __shfl_xor_sync(EQC_FULL, vs, d);
        ve |= __shfl_xor_sync(EQC_FULL, ve, d);
      }
      uint32_t S[4], E[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        S[w] = __shfl_sync(EQC_FULL, vs, 8 * w);
        E[w] = __shfl_sync(EQC_FULL, ve, 8 * w);
      }
      const uint64_t lo = ((uint64_t)E[1] << 32 | E[0]) - ((uint64_t)S[1] << 32 | S[0]);
      const uint64_t hi = ((uint64_t)E[3] << 32 | E[2]) - ((uint64_t)S[3] << 32 | S[2]) -
                          (((uint64_t)E[1] << 32 | E[0]) < ((uint64_t)S[1] << 32 | S[0]) ? 1u : 0u);
      A[0] = (uint32_t)lo;
      A[1] = (uint32_t)(lo >> 32);
      A[2] = (uint32_t)hi;
      A[3] = (uint32_t)(hi >> 32);
    }
    const int w = lane >> 3, sh = 4 * (lane & 7);
    const uint32_t Aw = w == 0 ? A[0] : w == 1 ? A[1] : w == 2 ? A[2] : A[3];
    const int pre = (w > 0 ? __popc(A[0]) : 0) + (w > 1 ? __popc(A[1]) : 0) + (w > 2 ? __popc(A[2]) : 0);
    cntb = pre + __popc(Aw & ((1u << sh) - 1u));
    nib = (Aw >> sh) & 0xFu;
  }
  // (a malformed record: the index is clamped into the record)
  return ld_window(r, min(ntok + cntb + (int)(nib & 1u), size), adv_sel(nib));
}

// unswizzle() of the four pixels held as plane words W[q] (byte j = byte q
// of pixel j): the same delta swaps, as swaps between two words (the steps
// that cross bytes) or within each word (inside a byte); the byte permute
// renames the words.  32 operations for four pixels instead of 4 x 13.
__device__ __forceinline__ void unswizzle_planes(uint32_t W[4]) {
  // slots 1 <-> 3: bits 2,3,6,7 of byte 0 (2) <-> bits 0,1,4,5 of byte 1 (3)
  uint32_t t = ((W[0] >> 2) ^ W[1]) & 0x33333333u;
  W[1] ^= t;
  W[0] ^= t << 2;
  t = ((W[2] >> 2) ^ W[3]) & 0x33333333u;
  W[3] ^= t;
  W[2] ^= t << 2;
  // slots 0 <-> 4: odd bits of byte 0 (1) <-> even bits of byte 2 (3)
  t = ((W[0] >> 1) ^ W[2]) & 0x55555555u;
  W[2] ^= t;
  W[0] ^= t << 1;
  t = ((W[1] >> 1) ^ W[3]) & 0x55555555u;
  W[3] ^= t;
  W[1] ^= t << 1;
  // slots 0 <-> 2 inside every byte
#pragma unroll
  for (int q = 0; q < 4; ++q) W[q] = delta_swap(W[q], 3, 0x0A0A0A0Au);
  // bytes 0 <-> 3 of every pixel
  t = W[0];
  W[0] = W[3];
  W[3] = t;
}

// 4x4 byte transpose: pixel j = byte j of the plane words W[0..3].
__device__ __forceinline__ void planes_to_px(const uint32_t W[4], uint32_t px[4]) {
  const uint32_t t0 = __byte_perm(W[0], W[1], 0x5140), t1 = __byte_perm(W[0], W[1], 0x7362);
  const uint32_t t2 = __byte_perm(W[2], W[3], 0x5140), t3 = __byte_perm(W[2], W[3], 0x7362);
  px[0] = __byte_perm(t0, t2, 0x5410);
  px[1] = __byte_perm(t0, t2, 0x7632);
  px[2] = __byte_perm(t1, t3, 0x5410);
  px[3] = __byte_perm(t1, t3, 0x7632);
}

}  // namespace eqc_rle
