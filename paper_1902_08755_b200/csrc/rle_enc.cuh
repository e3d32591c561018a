// rle_enc.cuh -- RLE-BP v1 chunk coder, branch-free (sm_100a).
//
// Thesis: per-component RLE -- "four independent RLE-compressed output
// streams" -- over an image decomposed into independently coded
// sub-images; the encoder is "purely constrained by the
// available memory bandwidth" on the thesis's CPUs.  Wire
// format and token rule: reading R-C8 -- maximal runs of
// >= 3 equal bytes become REPEAT tokens, the maximal spans between them
// LITERAL tokens, record = [ntok][ctrl x ntok][payload].
//
// GPU mapping.  One warp codes one 128-pixel chunk;
// lane l holds pixels 4l..4l+3 (x[j], one 128-bit load), so word x[j] carries
// position 4l+j of all four byte planes.  Every per-position flag is a word
// whose byte p holds the flag of plane p in bit 0 (0x01010101 = "all planes"):
//   EQ[j]  byte equals its predecessor            (4 byte compares per word)
//   c3     window (i-1, i, i+1) constant          EQ[i] & EQ[i+1]
//   R[j]   position inside a run of >= 3          c3[i-1] | c3[i] | c3[i+1]
//   T[j]   token start                            R changes, or a run follows a run
//   E[j]   position emits a payload byte          literal byte or first byte of a run
// The neighbour lanes' EQ words come by four shuffles, so every flag is a
// handful of LOP3s for all four planes at once, with no branch on the plane's
// class (a CONSTANT or LITERAL-ONLY plane is just a special case of the
// rule).  Per plane and lane, the payload bytes are compacted by one PRMT
// (selector from a 16-entry table indexed by the E nibble) and stored with
// four byte stores at the lane's prefix offset; the token starts likewise
// (256-entry table indexed by the T and R nibbles) into a start list, from
// which one lane per token derives the ctrl byte (length = next start -
// start).  A lane writes all four bytes of its compacted word even when it
// owns fewer; the stores go in four byte-index phases, highest first, with
// __syncwarp between them, so every byte's owner writes it after any garbage
// aimed at it (see code_chunk).
#pragma once

#include "eqc_common.cuh"

namespace eqc_enc {

constexpr int kC = 128;

// ---- lookup tables --------------------------------------------------------
//  sel[m]   PRMT selector moving the bytes of a word whose nibble-mask bit j is
//           set to the low end, in order (the unused selector nibbles are
//           don't-cares: those bytes are rewritten by their owners)
//  st[t | r << 4]  the positions j of the set bits of t, compacted one per
//           byte, each j | (bit j of r) << 7 (token start + REPEAT flag)
struct EncLuts {
  uint32_t sel[16];
  uint32_t st[256];
};

constexpr EncLuts make_enc_luts() {
  EncLuts L{};
  for (int m = 0; m < 16; ++m) {
    uint32_t s = 0x3210u;  // don't-care default
    int k = 0;
    for (int j = 0; j < 4; ++j)
      if ((m >> j) & 1) {
        s = (s & ~(0xFu << (4 * k))) | ((uint32_t)j << (4 * k));
        ++k;
      }
    L.sel[m] = s;
  }
  for (int i = 0; i < 256; ++i) {
    const int t = i & 15, r = i >> 4;
    uint32_t v = 0;
    int k = 0;
    for (int j = 0; j < 4; ++j)
      if ((t >> j) & 1) {
        v |= ((uint32_t)j | ((uint32_t)((r >> j) & 1) << 7)) << (8 * k);
        ++k;
      }
    L.st[i] = v;
  }
  return L;
}

__device__ const EncLuts g_enc_luts = make_enc_luts();

// Per-lane constants of the coder (computed once per kernel).
struct LaneK {
  uint32_t m0;   // 0 for lane 0 (position 0 has no predecessor), else 0x01010101
  uint32_t f0;   // 0x01010101 for lane 0 (forces a token start at position 0)
  uint32_t m31;  // 0 for lane 31 (positions 128, 129 do not exist)
  uint32_t p4;   // 4 * lane in every byte (the lane's first position)
};

__device__ __forceinline__ LaneK lane_consts(int lane) {
  LaneK k;
  k.m0 = lane ? 0x01010101u : 0u;
  k.f0 = lane ? 0u : 0x01010101u;
  k.m31 = lane == 31 ? 0u : 0x01010101u;
  k.p4 = (uint32_t)(4 * lane) * 0x01010101u;
  return k;
}

// bit 0 of byte p: byte p of a equals byte p of b (masked by m)
__device__ __forceinline__ uint32_t eq_bytes01(uint32_t a, uint32_t b, uint32_t m) {
  const uint32_t t = a ^ b;
  const uint32_t nz = ((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t;  // bit 7: byte differs
  return ~(nz >> 7) & m;
}

__device__ __forceinline__ int bytei(uint32_t v, int p) { return (int)__byte_perm(v, 0u, 0x4440u + (uint32_t)p); }

// Inclusive warp prefix sum (shuffle with the in-range predicate: no select).
__device__ __forceinline__ uint32_t scan_add(uint32_t v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1)
    asm("{\n\t.reg .b32 o;\n\t.reg .pred q;\n\t"
        "shfl.sync.up.b32 o|q, %0, %1, 0, -1;\n\t"
        "@q add.u32 %0, %0, o;\n\t}"
        : "+r"(v)
        : "r"(d));
  return v;
}

// Code one chunk.  x[0..3]: lane's pixels (swizzled when the stream is), 0 at
// positions >= L.  The record (planes 0..3) is written to rec[0, size) in
// shared memory at any alignment; up to 3 bytes past rec + size may receive
// garbage (the caller writes whatever follows later, or ignores it).  tp is a
// per-warp shared scratch of >= kTpBytes.  Returns the record size; *psizes =
// the four plane record sizes (byte p = plane p).
constexpr int kTpBytes = 4 * kC + 4 + 4;
constexpr int kTrashOff = kTpBytes;       // 4 trash bytes after the start list (tp must hold kTpBytes + 4)

template <bool FULL>
__device__ __forceinline__ int code_chunk(const uint32_t x[4], int L, int lane, const LaneK &k, uint8_t *rec,
                                          uint8_t *tp, const uint32_t *lut_sel, const uint32_t *lut_st,
                                          uint32_t *psizes) {
  constexpr uint32_t ONE = 0x01010101u;
  uint32_t V[4];  // validity of position 4l + j (i < L)
#pragma unroll
  for (int j = 0; j < 4; ++j) V[j] = (FULL || 4 * lane + j < L) ? ONE : 0u;
  // ---- EQ flags of the own positions, then of the neighbours' (-2, -1, 4, 5)
  const uint32_t xm1 = __shfl_up_sync(EQC_FULL, x[3], 1);
  uint32_t EQ[4];
  EQ[0] = eq_bytes01(x[0], xm1, k.m0 & V[0]);
#pragma unroll
  for (int j = 1; j < 4; ++j) EQ[j] = eq_bytes01(x[j], x[j - 1], V[j]);
  const uint32_t em2 = __shfl_up_sync(EQC_FULL, EQ[2], 1);
  const uint32_t em1 = __shfl_up_sync(EQC_FULL, EQ[3], 1);
  const uint32_t e4 = __shfl_down_sync(EQC_FULL, EQ[0], 1);
  const uint32_t e5 = __shfl_down_sync(EQC_FULL, EQ[1], 1);
  // ---- c3 (window constant) at positions -2..4; lane 0's c3[-2] is forced
  // so that R[-1] = 1, which with EQ[0] = 0 makes position 0 a token start
  const uint32_t c3m2 = (em2 & em1) | k.f0;
  const uint32_t c3m1 = em1 & EQ[0];
  const uint32_t c30 = EQ[0] & EQ[1], c31 = EQ[1] & EQ[2], c32 = EQ[2] & EQ[3];
  const uint32_t c33 = EQ[3] & e4 & k.m31, c34 = e4 & e5 & k.m31;
  const uint32_t Rm1 = c3m2 | c3m1 | c30;
  uint32_t R[4];
  R[0] = c3m1 | c30 | c31;
  R[1] = c30 | c31 | c32;
  R[2] = c31 | c32 | c33;
  R[3] = c32 | c33 | c34;
  uint32_t T[4], E[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t rp = j ? R[j - 1] : Rm1;
    T[j] = (R[j] ^ rp) | (R[j] & rp & ~EQ[j]);
    if (!FULL) T[j] &= V[j];
    E[j] = (~R[j] | T[j]) & V[j];
  }
  // ---- per-plane nibbles (table indices) and counts, packed per byte
  const uint32_t iE = 4 * E[0] + 8 * E[1] + 16 * E[2] + 32 * E[3];  // 4 * E nibble
  const uint32_t iTR = T[0] + 2 * T[1] + 4 * T[2] + 8 * T[3] + 16 * R[0] + 32 * R[1] + 64 * R[2] + 128 * R[3];
  const uint32_t cT = T[0] + T[1] + T[2] + T[3];
  const uint32_t cE = E[0] + E[1] + E[2] + E[3];
  const uint32_t incT = scan_add(cT);
  const uint32_t incE = scan_add(cE);
  const uint32_t totT = __shfl_sync(EQC_FULL, incT, 31);
  const uint32_t totE = __shfl_sync(EQC_FULL, incE, 31);
  const uint32_t exT = incT - cT, exE = incE - cE;
  const uint32_t sz = ONE + totT + totE;  // plane record sizes (<= 130 each)
  *psizes = sz;
  int off[4], P[4], nt[4];
  off[0] = 0;
  P[0] = 0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    nt[p] = bytei(totT, p);
    if (p < 3) {
      off[p + 1] = off[p] + bytei(sz, p);
      P[p + 1] = P[p] + nt[p];
    }
  }
  const int size = off[3] + bytei(sz, 3);
  const int ntot = P[3] + nt[3];
  // ---- plane words: byte j of pw[p] = plane p at position 4l + j
  uint32_t pw[4];
  {
    const uint32_t a = __byte_perm(x[0], x[1], 0x5140), b = __byte_perm(x[2], x[3], 0x5140);
    const uint32_t c = __byte_perm(x[0], x[1], 0x7362), d = __byte_perm(x[2], x[3], 0x7362);
    pw[0] = __byte_perm(a, b, 0x5410);
    pw[1] = __byte_perm(a, b, 0x7632);
    pw[2] = __byte_perm(c, d, 0x5410);
    pw[3] = __byte_perm(c, d, 0x7632);
  }
  // ---- payload bytes and token starts.  A lane owning c >= 1 bytes of a
  // region writes all four bytes of its compacted word at its prefix offset;
  // the 4 - c it does not own belong to lanes (or, past the region's end, to
  // the next plane's header / start list / payload) that write them at a
  // LOWER byte index j.  So the stores go in four phases, j = 3, 2, 1, 0,
  // every plane's bytes j in phase j, __syncwarp between phases: each byte's
  // owner writes it after any garbage aimed at it.  (Lanes owning nothing
  // store into a trash word: two lanes never write one real byte in the same
  // phase.)
  uint32_t cw[4], sv[4];
  uint8_t *pa[4], *pb[4];
  uint8_t *const trash = tp + kTrashOff;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const uint32_t sel = *reinterpret_cast<const uint32_t *>(reinterpret_cast<const uint8_t *>(lut_sel) + bytei(iE, p));
    cw[p] = __byte_perm(pw[p], 0u, sel);                     // payload bytes, compacted by E
    sv[p] = lut_st[bytei(iTR, p)] + k.p4;                    // token starts (+ REPEAT flag), compacted by T
    // a lane owning no byte of a region writes into the trash bytes instead
    // (no predicate per store)
    pa[p] = (cE & (0xFFu << (8 * p))) ? rec + off[p] + 1 + nt[p] + bytei(exE, p) : trash;  // off + 1 + ntok + E prefix
    pb[p] = (cT & (0xFFu << (8 * p))) ? tp + P[p] + p + bytei(exT, p) : trash;              // P + p + T prefix
  }
#pragma unroll
  for (int j = 3; j >= 0; --j) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      pa[p][j] = (uint8_t)(cw[p] >> (8 * j));
      pb[p][j] = (uint8_t)(sv[p] >> (8 * j));
    }
    __syncwarp();
  }
  // sentinel after each plane's starts (the end of its last token) and the
  // ntok bytes
  if (lane < 4) {
    int sp = P[1], ro = off[0], n = nt[0];
    if (lane == 1) sp = P[2] + 1, ro = off[1], n = nt[1];
    if (lane == 2) sp = P[3] + 2, ro = off[2], n = nt[2];
    if (lane == 3) sp = ntot + 3, ro = off[3], n = nt[3];
    tp[sp] = (uint8_t)L;
    rec[ro] = (uint8_t)n;
  }
  __syncwarp();
  // ---- ctrl bytes: token q of the concatenated start lists (plane p's start
  // k is entry P[p] + p + k); length = next start - start (mod 128, so the
  // sentinel 128 of a full chunk works)
  const int D1 = off[1] + 1 - P[1], D2 = off[2] + 1 - P[2], D3 = off[3] + 1 - P[3];
  for (int q = lane; q < ntot; q += 32) {
    int o = 0, D = 1;
    if (q >= P[1]) o = 1, D = D1;
    if (q >= P[2]) o = 2, D = D2;
    if (q >= P[3]) o = 3, D = D3;
    const uint32_t s0 = tp[q + o], s1 = tp[q + o + 1];
    rec[q + D] = (uint8_t)((s0 & 0x80u) | ((s1 - s0 - 1u) & 0x7Fu));
  }
  __syncwarp();
  return size;
}

}  // namespace eqc_enc
