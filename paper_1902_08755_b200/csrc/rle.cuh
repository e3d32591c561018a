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
// Byte reversal maps channel c to c' = 3 - c; the remaining permutation of the
// 5 bit-index bits (c'1 c'0 b2 b1 b0) -> (b2 b1 b0 c'1 c'0) is four
// transpositions of index bits, each one delta swap.
__device__ __forceinline__ uint32_t delta_swap(uint32_t x, int d, uint32_t m) {
  uint32_t t = ((x >> d) ^ x) & m;
  return x ^ t ^ (t << d);
}
__device__ __forceinline__ uint32_t swizzle(uint32_t v) {
  v = __byte_perm(v, 0, 0x0123);
  v = delta_swap(v, 12, 0x0000F0F0u);  // index bits 4 <-> 2
  v = delta_swap(v, 6, 0x00CC00CCu);   // 3 <-> 1
  v = delta_swap(v, 3, 0x0A0A0A0Au);   // 2 <-> 0
  v = delta_swap(v, 1, 0x22222222u);   // 1 <-> 0
  return v;
}
__device__ __forceinline__ uint32_t unswizzle(uint32_t v) {
  v = delta_swap(v, 1, 0x22222222u);
  v = delta_swap(v, 3, 0x0A0A0A0Au);
  v = delta_swap(v, 6, 0x00CC00CCu);
  v = delta_swap(v, 12, 0x0000F0F0u);
  return __byte_perm(v, 0, 0x0123);
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

// Decode plane record r[0..size) (staging bytes) of a chunk of length L into
// byte p of out[0..3] (positions 4*lane + j).  `info` is per-warp scratch of
// 128 uint16.  Returns false if the record is malformed (warp-uniform).
template <bool FULL>
__device__ __forceinline__ bool decode_plane_t(const uint8_t *r, int size, int L_, int lane, int p,
                                               uint32_t out[4], uint16_t *info) {
  // FULL: a 128-pixel chunk (every lane's 4 positions are valid)
  const int L = FULL ? kC : L_;
  const int i0 = 4 * lane;
  if (size < 2) return false;
  const int ntok = r[0];
  if (ntok < 1 || 1 + ntok > size) return false;
  if (ntok == 1) {  // single-token fast paths (uniform)
    const int c = r[1];
    const int len = (c & 0x7F) + 1;
    if (len != L) return false;
    if (c & 0x80) {
      if (size != 3) return false;
      const uint32_t v = (uint32_t)r[2] << (8 * p);
#pragma unroll
      for (int j = 0; j < 4; ++j) out[j] |= v;
    } else {
      if (size != 2 + L) return false;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (FULL || i0 + j < L) out[j] |= (uint32_t)r[2 + i0 + j] << (8 * p);
    }
    return true;
  }
  if (ntok <= 4) {
    // few tokens (typical of mixed background/foreground chunks): the token
    // boundaries are computed once (uniform), each position selects its token
    // by comparison -- no scans, no shuffles, no scratch
    // token t covers [st[t], st[t+1]); its byte for position i is
    // r[bs[t] + lt[t] * i] (literal: bs = payload index - start, lt = 1;
    // repeat: bs = payload index, lt = 0)
    int st[4], bs[4], lt[4];
    int pos = 0, pay = 1 + ntok;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      st[t] = 0x7FFF;  // never selected
      bs[t] = 0;
      lt[t] = 0;
      if (t < ntok) {
        const int c = r[1 + t];
        const int len = (c & 0x7F) + 1;
        const bool lit = !(c & 0x80);
        st[t] = pos;
        bs[t] = lit ? pay - pos : pay;
        lt[t] = lit;
        pos += len;
        pay += lit ? len : 1;
      }
    }
    if (pos != L || pay != size) return false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j;
      if (FULL || i < L) {
        // the covering token is the last one starting at or before i
        int b = bs[0], l = lt[0];
#pragma unroll
        for (int t = 1; t < 4; ++t) {
          const bool in = i >= st[t];
          b = in ? bs[t] : b;
          l = in ? lt[t] : l;
        }
        out[j] |= (uint32_t)r[b + l * i] << (8 * p);
      }
    }
    return true;
  }
  if (ntok <= 32) {
    // lane t holds token t: start positions and payload indices by one packed
    // warp scan; each position finds its token as the last start at or before
    // it (token-index markers + a running max over positions) and reads the
    // token's {start, payload index, type} with one shuffle.
    const int c = lane < ntok ? r[1 + lane] : 0;
    const int len = lane < ntok ? (c & 0x7F) + 1 : 0;
    const int pay = (c & 0x80) ? 1 : len;
    const uint32_t packed = (uint32_t)len | ((uint32_t)pay << 16);
    const uint32_t inc = warp_incl_scan_add(packed, lane);
    const uint32_t tot = __shfl_sync(EQC_FULL, inc, 31);
    if ((int)(tot & 0xFFFFu) != L || (int)(tot >> 16) != size - 1 - ntok) return false;
    const uint32_t ex = inc - packed;
    const int tstart = (int)(ex & 0xFFFFu);
    const int tpay = 1 + ntok + (int)(ex >> 16);
    const uint32_t tinfo = (uint32_t)tstart | ((uint32_t)tpay << 8) | ((uint32_t)(c & 0x80) << 24);
    uint8_t *mk = reinterpret_cast<uint8_t *>(info);
    __syncwarp();
    reinterpret_cast<uint32_t *>(mk)[lane] = 0u;
    __syncwarp();
    if (lane < ntok) mk[tstart] = (uint8_t)(lane + 1);
    __syncwarp();
    const uint32_t w4 = reinterpret_cast<const uint32_t *>(mk)[lane];
    // markers grow with position, so the running max is the last marker
    const int lmax = (int)max(max(w4 & 0xFFu, (w4 >> 8) & 0xFFu), max((w4 >> 16) & 0xFFu, w4 >> 24));
    int pre = lmax;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(EQC_FULL, pre, d);
      if (lane >= d) pre = max(pre, o);
    }
    int run = __shfl_up_sync(EQC_FULL, pre, 1);
    if (lane == 0) run = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      run = max(run, (int)((w4 >> (8 * j)) & 0xFFu));
      const uint32_t ti = __shfl_sync(EQC_FULL, tinfo, max(run - 1, 0));
      const int i = i0 + j;
      if (FULL || i < L) {
        const int pi = (int)((ti >> 8) & 0xFFFFu) + ((ti >> 31) ? 0 : i - (int)(ti & 0xFFu));
        out[j] |= (uint32_t)r[pi] << (8 * p);
      }
    }
    return true;
  }
  // many tokens: tokens 4*lane .. 4*lane+3 per lane, positions by prefix sums
  __syncwarp();  // the info scratch may still be read by the previous plane
  int sl = 0, sp = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int t = i0 + k;
    if (t < ntok) {
      const int c = r[1 + t];
      const int len = (c & 0x7F) + 1;
      const int pay = (c & 0x80) ? 1 : len;
      sl += len;
      sp += pay;
    }
  }
  const uint32_t packed = (uint32_t)sl | ((uint32_t)sp << 16);
  const uint32_t inc = warp_incl_scan_add(packed, lane);
  const uint32_t tot = __shfl_sync(EQC_FULL, inc, 31);
  if ((int)(tot & 0xFFFFu) != L || (int)(tot >> 16) != size - 1 - ntok) return false;
  uint32_t ex = inc - packed;
  int spos = (int)(ex & 0xFFFFu);
  int ppos = 1 + ntok + (int)(ex >> 16);
  // clear the per-position info table, then mark each token start with
  // (payload index | literal flag << 15)
  reinterpret_cast<uint2 *>(info)[lane] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int t = i0 + k;
    if (t < ntok) {
      const int c = r[1 + t];
      const int len = (c & 0x7F) + 1;
      info[spos] = (uint16_t)(ppos | ((c & 0x80) ? 0 : 0x8000));
      spos += len;
      ppos += (c & 0x80) ? 1 : len;
    }
  }
  __syncwarp();
  // covering token start of each position: running max of start positions
  const uint2 iw = reinterpret_cast<const uint2 *>(info)[lane];
  const uint16_t inf[4] = {(uint16_t)(iw.x & 0xFFFF), (uint16_t)(iw.x >> 16), (uint16_t)(iw.y & 0xFFFF),
                           (uint16_t)(iw.y >> 16)};
  int lmax = -1;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (inf[j] != 0xFFFF && i0 + j < L) lmax = i0 + j;
  int pre = lmax;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(EQC_FULL, pre, d);
    if (lane >= d) pre = max(pre, o);
  }
  int run = __shfl_up_sync(EQC_FULL, pre, 1);
  if (lane == 0) run = -1;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = i0 + j;
    if (i < L) {
      if (inf[j] != 0xFFFF) run = i;
      const uint32_t ti = info[run];
      const int pi = (int)(ti & 0x7FFFu) + ((ti & 0x8000u) ? (i - run) : 0);
      out[j] |= (uint32_t)r[pi] << (8 * p);
    }
  }
  return true;
}

__device__ __forceinline__ bool decode_plane(const uint8_t *r, int size, int L, int lane, int p, uint32_t out[4],
                                             uint16_t *info) {
  return L == kC ? decode_plane_t<true>(r, size, L, lane, p, out, info)
                 : decode_plane_t<false>(r, size, L, lane, p, out, info);
}

}  // namespace eqc_rle
