// eqc_common.cuh -- device/host helpers shared by the libeqc kernels
// (sm_100a only).  No arithmetic of the method lives here; see composite.cu,
// rle.cuh and rle.cu for the kernels and their paper citations.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/eqc.h"

#define EQC_WARP 32
#define EQC_FULL 0xFFFFFFFFu

#define EQC_CUDA_TRY(expr)                      \
  do {                                          \
    cudaError_t _e = (expr);                    \
    if (_e != cudaSuccess) return EQC_E_CUDA;   \
  } while (0)

// Launch-error check after a <<<>>> launch.
static inline int eqc_launch_status() {
  return cudaGetLastError() == cudaSuccess ? EQC_OK : EQC_E_CUDA;
}

static inline int eqc_num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// CTAs of `kernel` (at `threads` per CTA) resident on the whole GPU at once:
// grid-stride kernels launch at most this many, so there is no partial last
// wave (a 1.33-wave grid leaves most SMs idle for its last third).
template <typename K>
inline int eqc_resident_ctas(K kernel, int threads, size_t smem = 0) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  return occ * eqc_num_sms();
}

// ---- streaming 128-bit global access (inputs are read exactly once) -------
// The loads are not `volatile`: inputs are read-only for the kernel's lifetime,
// and the scheduler must be free to hoist a batch of loads above the
// arithmetic that consumes the previous ones (volatile asm pins their order
// relative to each other and lets the compiler interleave load / use).
__device__ __forceinline__ uint4 ld_stream_u4(const void *p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Predicated variant: no memory access (and zeros) when !pred.  Branch-free,
// so a batch of them can all be in flight (a load under an `if` is not
// hoisted above the branch of the next one).
__device__ __forceinline__ uint4 ld_stream_u4_if(const void *p, bool pred) {
  uint4 r = make_uint4(0, 0, 0, 0);
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
      : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
      : "l"(p), "r"((uint32_t)pred));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const void *p) {
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream_u4(void *p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream_u32(void *p, uint32_t v) {
  asm volatile("st.global.L1::no_allocate.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- byte-SIMD helpers on packed words (flag = bit 7 of each byte) -------
// Bit 7 of byte k set iff byte k of a equals byte k of b.
__device__ __forceinline__ uint32_t bytes_eq(uint32_t a, uint32_t b) {
  uint32_t t = a ^ b;
  // bit 7 of ((t & 0x7f) + 0x7f) | t is set iff the byte is non-zero
  uint32_t nz = ((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t;
  return ~nz & 0x80808080u;
}
// Bit 7 of byte k set iff byte k of a is non-zero.
__device__ __forceinline__ uint32_t bytes_nz(uint32_t a) {
  return (((a & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | a) & 0x80808080u;
}
// Expand a bit-7 flag word to full 0xFF/0x00 byte masks.
__device__ __forceinline__ uint32_t flags_to_mask(uint32_t f) {
  return (f >> 7) * 0xFFu;
}
// Per-byte population count of a word whose bytes hold values < 16.
__device__ __forceinline__ uint32_t bytes_popc_nibble(uint32_t x) {
  x = x - ((x >> 1) & 0x05050505u);
  return (x & 0x03030303u) + ((x >> 2) & 0x03030303u);
}

// ---- warp scans -----------------------------------------------------------
// Inclusive prefix sum over lanes (plain integer add; packed byte/halfword
// lanes are fine as long as no lane's field overflows).
// (The shuffle's in-range predicate guards the add: two instructions a step.)
__device__ __forceinline__ uint32_t warp_incl_scan_add(uint32_t v, int lane) {
  (void)lane;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1)
    asm("{\n\t.reg .b32 o;\n\t.reg .pred q;\n\t"
        "shfl.sync.up.b32 o|q, %0, %1, 0, -1;\n\t"
        "@q add.u32 %0, %0, o;\n\t}"
        : "+r"(v)
        : "r"(d));
  return v;
}
