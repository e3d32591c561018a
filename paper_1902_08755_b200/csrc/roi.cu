// roi.cu -- region of interest of a frame buffer.
//
//  image_roi   per-frame 2D bounding box of the rendered (non-background)
//              pixels: "the screen-space 2D bounding box fully enclosing the
//              data rendered by a single resource", computed
//              "by analysing the framebuffer".
//
// HBM-bound scan (4 B per pixel read once, 16 B per frame written): each CTA
// owns a contiguous row range of one frame, every thread streams 4-pixel
// groups with 128-bit loads and keeps its own (x0, y0, x1, y1); the CTA
// reduces them with warp reductions and merges its box into the frame's with
// four global atomics.  A one-warp init kernel before and a finalise kernel
// after turn the accumulator into {x, y, w, h} (all zero for an empty frame)
// on the device, so the result can feed compositor_*_roi with no host sync.
#include <algorithm>
#include <climits>

#include "eqc_common.cuh"

namespace {

struct RoiParams {
  const uint32_t *frame[EQC_MAX_SOURCES];
  int32_t *roi;  // device n x 4: accumulator {x0, y0, x1, y1} (inclusive), then {x, y, w, h}
  int64_t pitch;
  int n, w, h, ctas_per_frame, groups_per_row;
  uint32_t background;
  int vec;
};

__global__ void roi_init_kernel(int32_t *roi, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    reinterpret_cast<int4 *>(roi)[i] = make_int4(INT_MAX, INT_MAX, -1, -1);
}

__global__ void __launch_bounds__(256) roi_scan_kernel(const __grid_constant__ RoiParams p) {
  __shared__ int s_box[4][8];
  const int f = blockIdx.x / p.ctas_per_frame;
  const int part = blockIdx.x - f * p.ctas_per_frame;
  const int ya = (int)((int64_t)part * p.h / p.ctas_per_frame);
  const int yb = (int)((int64_t)(part + 1) * p.h / p.ctas_per_frame);
  const uint32_t *fr = p.frame[f];
  const uint32_t bg = p.background;
  int x0 = INT_MAX, y0 = INT_MAX, x1 = -1, y1 = -1;
  const uint32_t gpr = (uint32_t)p.groups_per_row;
  const uint32_t g0 = (uint32_t)ya * gpr, g1 = (uint32_t)yb * gpr;  // < 2^31 (host check)
  const uint32_t stride = blockDim.x;
  if (p.vec && (p.w & 3) == 0) {
    // every group is 4 full pixels: 8 predicated 128-bit loads in flight per
    // thread per step, no branches between them
    for (uint32_t gb = g0 + threadIdx.x; gb < g1; gb += 8 * stride) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t g = min(gb + u * stride, g1 - 1);
        const uint32_t y = g / gpr;
        v[u] = ld_stream_u4_if(fr + (int64_t)y * p.pitch + (g - y * gpr) * 4, gb + u * stride < g1);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t g = gb + u * stride;
        const uint32_t m = (v[u].x != bg) | ((v[u].y != bg) << 1) | ((v[u].z != bg) << 2) | ((v[u].w != bg) << 3);
        if (g < g1 && m) {
          const int y = (int)(g / gpr), x = (int)(g - (uint32_t)y * gpr) * 4;
          x0 = min(x0, x + __ffs(m) - 1);
          x1 = max(x1, x + 31 - __clz(m));
          y0 = min(y0, y);
          y1 = max(y1, y);
        }
      }
    }
  } else {
    for (uint32_t g = g0 + threadIdx.x; g < g1; g += stride) {
      const int y = (int)(g / gpr), x = (int)(g - (uint32_t)y * gpr) * 4;
      const uint32_t *q = fr + (int64_t)y * p.pitch + x;
      uint32_t m = 0;
      for (int j = 0; j < 4 && x + j < p.w; ++j) m |= (uint32_t)(ld_stream_u32(q + j) != bg) << j;
      if (m) {
        x0 = min(x0, x + __ffs(m) - 1);
        x1 = max(x1, x + 31 - __clz(m));
        y0 = min(y0, y);
        y1 = max(y1, y);
      }
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  x0 = __reduce_min_sync(EQC_FULL, x0);
  y0 = __reduce_min_sync(EQC_FULL, y0);
  x1 = __reduce_max_sync(EQC_FULL, x1);
  y1 = __reduce_max_sync(EQC_FULL, y1);
  if (lane == 0) {
    s_box[0][warp] = x0;
    s_box[1][warp] = y0;
    s_box[2][warp] = x1;
    s_box[3][warp] = y1;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int a = lane < nw ? s_box[0][lane] : INT_MAX, b = lane < nw ? s_box[1][lane] : INT_MAX;
    int c = lane < nw ? s_box[2][lane] : -1, d = lane < nw ? s_box[3][lane] : -1;
    a = __reduce_min_sync(EQC_FULL, a);
    b = __reduce_min_sync(EQC_FULL, b);
    c = __reduce_max_sync(EQC_FULL, c);
    d = __reduce_max_sync(EQC_FULL, d);
    if (lane == 0 && c >= 0) {
      int32_t *r = p.roi + 4 * f;
      atomicMin(r + 0, a);
      atomicMin(r + 1, b);
      atomicMax(r + 2, c);
      atomicMax(r + 3, d);
    }
  }
}

__global__ void roi_finalize_kernel(int32_t *roi, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int4 a = reinterpret_cast<int4 *>(roi)[i];
    reinterpret_cast<int4 *>(roi)[i] =
        a.z < 0 ? make_int4(0, 0, 0, 0) : make_int4(a.x, a.y, a.z - a.x + 1, a.w - a.y + 1);
  }
}

}  // namespace

extern "C" int image_roi(int n, const uint32_t *const *frames, int w, int h, int64_t pitch, uint32_t background,
                         int32_t *d_roi, void *stream) {
  if (n < 1 || n > EQC_MAX_SOURCES || !frames || !d_roi) return EQC_E_INVALID;
  if (w <= 0 || h <= 0 || pitch < w) return EQC_E_INVALID;
  if (((uintptr_t)d_roi & 15) != 0) return EQC_E_INVALID;
  RoiParams p;
  bool vec = pitch % 4 == 0;
  for (int i = 0; i < n; ++i) {
    if (!frames[i]) return EQC_E_INVALID;
    p.frame[i] = frames[i];
    vec = vec && ((uintptr_t)frames[i] & 15) == 0;
  }
  p.roi = d_roi;
  p.pitch = pitch;
  p.n = n;
  p.w = w;
  p.h = h;
  p.background = background;
  p.vec = vec ? 1 : 0;
  p.groups_per_row = (w + 3) / 4;
  if ((int64_t)p.groups_per_row * h > 0x7FFFFFFFll) return EQC_E_INVALID;
  // one full wave of resident CTAs over all frames, whole rows per CTA
  static const int resident = eqc_resident_ctas(roi_scan_kernel, 256);
  p.ctas_per_frame = std::max(1, std::min(h, resident / n));
  cudaStream_t s = (cudaStream_t)stream;
  roi_init_kernel<<<1, 64, 0, s>>>(d_roi, n);
  roi_scan_kernel<<<n * p.ctas_per_frame, 256, 0, s>>>(p);
  roi_finalize_kernel<<<1, 64, 0, s>>>(d_roi, n);
  return eqc_launch_status();
}

// Load every kernel of this file now (see eqc_preload_composite).
int eqc_preload_roi() {
  cudaFuncAttributes a;
  bool ok = cudaFuncGetAttributes(&a, roi_init_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, roi_scan_kernel) == cudaSuccess;
  ok = ok && cudaFuncGetAttributes(&a, roi_finalize_kernel) == cudaSuccess;
  return ok ? EQC_OK : EQC_E_CUDA;
}
