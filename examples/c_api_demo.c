/*
 * c_api_demo.c -- the libeqc C ABI used from plain C with the CUDA runtime
 * (no Python, no torch): the boundary takes device pointers, sizes and a
 * stream.  Composites N synthetic sources, RLE-encodes the result, decodes it
 * and checks the round trip; prints one line.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_demo.c \
 *       -L paper_1902_08755_b200 -l:libeqc.so -Wl,-rpath,$PWD/paper_1902_08755_b200 \
 *       -L /usr/local/cuda/lib64 -lcudart -o c_api_demo && ./c_api_demo
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "eqc.h"

#define CK(x)                                                              \
  do {                                                                     \
    int _r = (int)(x);                                                     \
    if (_r != 0) {                                                         \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, _r, eqc_strerror(_r)); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main(void) {
  enum { N = 4, W = 640, H = 360 };
  const size_t px = (size_t)W * H, bytes = px * 4;
  uint32_t *h = (uint32_t *)malloc(bytes);
  uint32_t *color[N], *depth[N];
  for (int i = 0; i < N; ++i) {
    CK(cudaMalloc((void **)&color[i], bytes));
    CK(cudaMalloc((void **)&depth[i], bytes));
    for (size_t p = 0; p < px; ++p) h[p] = 0xFF000000u | (uint32_t)(i * 0x303030);  /* flat colour per source */
    CK(cudaMemcpy(color[i], h, bytes, cudaMemcpyHostToDevice));
    for (size_t p = 0; p < px; ++p) {  /* source i is nearest in vertical stripe i, background elsewhere */
      const int x = (int)(p % W);
      h[p] = (x * N / W == i) ? (uint32_t)(1000 + i) : ((x & 1) ? 0xFFFFFFFFu : (uint32_t)(5000 + i));
    }
    CK(cudaMemcpy(depth[i], h, bytes, cudaMemcpyHostToDevice));
  }
  uint32_t *out_c, *out_d, *back;
  CK(cudaMalloc((void **)&out_c, bytes));
  CK(cudaMalloc((void **)&out_d, bytes));
  CK(cudaMalloc((void **)&back, bytes));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  CK(compositor_depth(N, (const uint32_t *const *)color, (const uint32_t *const *)depth, W, H, W, out_c, out_d, W, s));
  /* RLE round trip of the composited colour */
  const int64_t cap = image_rle_max_size(W, H);
  const size_t wsb = image_rle_workspace_size(W, H);
  uint8_t *stream, *ws;
  int64_t *d_size;
  int32_t *d_status;
  CK(cudaMalloc((void **)&stream, (size_t)cap));
  CK(cudaMalloc((void **)&ws, wsb));
  CK(cudaMalloc((void **)&d_size, sizeof(int64_t)));
  CK(cudaMalloc((void **)&d_status, sizeof(int32_t)));
  CK(cudaMemsetAsync(d_status, 0, sizeof(int32_t), s));
  CK(image_compress_rle(out_c, W, H, W, EQC_KIND_RGBA8, EQC_FLAG_SWIZZLE, stream, cap, d_size, ws, wsb, s));
  CK(image_decompress_rle(stream, cap, back, W, W, H, d_status, s));
  CK(cudaStreamSynchronize(s));
  int64_t size = 0;
  int32_t status = 0;
  CK(cudaMemcpy(&size, d_size, sizeof(size), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&status, d_status, sizeof(status), cudaMemcpyDeviceToHost));
  uint32_t *a = (uint32_t *)malloc(bytes), *b = (uint32_t *)malloc(bytes);
  CK(cudaMemcpy(a, out_c, bytes, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b, back, bytes, cudaMemcpyDeviceToHost));
  /* expected: stripe i shows source i's colour */
  int bad = 0;
  for (size_t p = 0; p < px; ++p) {
    const int i = (int)(p % W) * N / W;
    bad += a[p] != (0xFF000000u | (uint32_t)(i * 0x303030));
  }
  const int same = memcmp(a, b, bytes) == 0;
  printf("c_api_demo: libeqc %d.%d.%d, composite %s, rle %lld bytes (%.1f%% of raw), decode %s, status %d\n",
         eqc_version() >> 16, (eqc_version() >> 8) & 0xFF, eqc_version() & 0xFF, bad ? "WRONG" : "ok",
         (long long)size, 100.0 * (double)size / (double)bytes, same ? "ok" : "WRONG", status);
  return (bad || !same || status) ? 1 : 0;
}
