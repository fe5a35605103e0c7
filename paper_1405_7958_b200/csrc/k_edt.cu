// o6 distance map for PreWatershed: exact squared
// Euclidean distance transform, separable.
//
// Column phase: the tile is cut into 32-row segments; k_edt_seg summarises
// each (column, segment) by its first/last zero row, k_edt_col resolves the
// nearest zero above/below through the summaries and emits the 1-D column
// distance g (u16, 0xFFFF = no zero in the column).  262k threads for a
// 4096^2 tile instead of 4096 sequential column walkers.
// Row phase: one CTA per row stages g in shared memory; every foreground pixel
// searches outward, stopping as soon as k^2 >= best (exact: no farther column
// can win).  Rows whose search exceeds kCap fall back to a per-row exact
// lower-envelope pass (Meijster), so adversarial masks stay exact.
// The row pass also emits dq = floor(4*sqrt(d2)) and the HMAX marker.
//
// Roofline: HBM/L2 bound; algorithmic bytes mask 1 B in + dq/marker 4 B out.
#include "common.cuh"

namespace rtg {
namespace {

constexpr int kSeg = 32;
constexpr uint32_t kInfG = 0xFFFFu;
constexpr int kCap = 96;

__global__ void k_edt_seg(const uint8_t* __restrict__ mask, int h, int w,
                          uint16_t* __restrict__ seg, int32_t* __restrict__ any_zero) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  bool z = false;
  if (x < w) {
    int first = 0xFF, last = 0xFF;
    const int y0 = s * kSeg;
    for (int r = 0; r < kSeg && y0 + r < h; ++r) {
      if (!mask[(int64_t)(y0 + r) * w + x]) {
        if (first == 0xFF) first = r;
        last = r;
      }
    }
    seg[(int64_t)s * w + x] = (uint16_t)(first | (last << 8));
    z = first != 0xFF;
  }
  if (__any_sync(0xFFFFFFFFu, z) && (threadIdx.x & 31) == 0) atomicOr(any_zero, 1);
}

__global__ void k_edt_col(const uint8_t* __restrict__ mask, int h, int w,
                          const uint16_t* __restrict__ seg, uint16_t* __restrict__ g) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (x >= w) return;
  const int nseg = (h + kSeg - 1) / kSeg;
  const int y0 = s * kSeg;
  int above = -1;  // row of the nearest zero above the segment
  for (int t = s - 1; t >= 0; --t) {
    const int last = seg[(int64_t)t * w + x] >> 8;
    if (last != 0xFF) { above = t * kSeg + last; break; }
  }
  int below = -1;
  for (int t = s + 1; t < nseg; ++t) {
    const int first = seg[(int64_t)t * w + x] & 0xFF;
    if (first != 0xFF) { below = t * kSeg + first; break; }
  }
  const int rows = min(kSeg, h - y0);
  uint32_t zbits = 0;
  uint32_t du[kSeg];
#pragma unroll
  for (int r = 0; r < kSeg; ++r) {
    if (r < rows) {
      const int y = y0 + r;
      if (!mask[(int64_t)y * w + x]) { zbits |= 1u << r; above = y; }
      du[r] = above >= 0 ? (uint32_t)(y - above) : kInfG;
    }
  }
#pragma unroll
  for (int r = kSeg - 1; r >= 0; --r) {
    if (r < rows) {
      const int y = y0 + r;
      if (zbits & (1u << r)) below = y;
      const uint32_t dd = below >= 0 ? (uint32_t)(below - y) : kInfG;
      g[(int64_t)y * w + x] = (uint16_t)min(du[r], dd);
    }
  }
}

__device__ __forceinline__ uint32_t isqrt64(uint64_t v) {
  uint64_t r = (uint64_t)sqrt((double)v);
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return (uint32_t)r;
}

__device__ __forceinline__ void edt_emit(int64_t i, int64_t d2, int32_t* dist2,
                                         uint16_t* dq, uint16_t* mk, int32_t ws_h) {
  if (dist2) dist2[i] = (int32_t)d2;
  uint32_t v = d2 >= (int64_t)INT32_MAX ? 65535u : isqrt64(16ull * (uint64_t)d2);
  if (v > 65534u) v = 65534u;
  if (dq) dq[i] = (uint16_t)v;
  if (mk) mk[i] = (uint16_t)(v > (uint32_t)ws_h ? v - (uint32_t)ws_h : 0u);
}

__global__ void __launch_bounds__(256)
k_edt_row(const uint16_t* __restrict__ g, int h, int w,
          const int32_t* __restrict__ any_zero, int32_t* __restrict__ dist2,
          uint16_t* __restrict__ dq, uint16_t* __restrict__ mk, int32_t ws_h,
          int32_t* __restrict__ row_flag) {
  extern __shared__ uint16_t gs[];
  const int y = blockIdx.x;
  const int64_t rb = (int64_t)y * w;
  for (int x = threadIdx.x; x < w; x += blockDim.x) gs[x] = g[rb + x];
  __syncthreads();
  const bool none = *any_zero == 0;
  bool unresolved = false;
  // 32-bit arithmetic: g <= 8193 and k <= kCap, so k^2 + g^2 < 2^31
  for (int x = threadIdx.x; x < w; x += blockDim.x) {
    const uint32_t gx = gs[x];
    uint32_t best;
    if (none) {
      best = INT32_MAX;
    } else if (gx == 0) {
      best = 0;
    } else {
      best = gx == kInfG ? 0xFFFFFFFFu : gx * gx;
      uint32_t k = 1;
      for (; k * k < best && k <= (uint32_t)kCap; ++k) {
        const uint32_t k2 = k * k;
        const uint32_t gl = x >= (int)k ? gs[x - k] : kInfG;
        const uint32_t gr = x + (int)k < w ? gs[x + k] : kInfG;
        const uint32_t gm = min(gl, gr);
        if (gm != kInfG) best = min(best, k2 + gm * gm);
      }
      if (k * k < best) unresolved = true;  // hit the cap: exact row pass below
    }
    edt_emit(rb + x, (int64_t)best, dist2, dq, mk, ws_h);
  }
  if (__syncthreads_or(unresolved) && threadIdx.x == 0) row_flag[y] = 1;
  else if (threadIdx.x == 0) row_flag[y] = 0;
}

__device__ __forceinline__ int64_t floordiv64(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}

// Exact per-row lower envelope (Meijster phase 2) for flagged rows.
__global__ void k_edt_row_exact(const uint16_t* __restrict__ g, int h, int w,
                                const int32_t* __restrict__ row_flag,
                                int32_t* __restrict__ s_buf, int32_t* __restrict__ t_buf,
                                int32_t* __restrict__ dist2, uint16_t* __restrict__ dq,
                                uint16_t* __restrict__ mk, int32_t ws_h,
                                uint32_t* __restrict__ status) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= h || !row_flag[y]) return;
  atomicOr(status, kStatusEdtFallback);
  const int64_t rb = (int64_t)y * w;
  const int64_t INF = (int64_t)h + w + 1;
  int32_t* s = s_buf + rb;
  int32_t* t = t_buf + rb;
  auto G = [&](int64_t i) -> int64_t {
    const uint32_t v = g[rb + i];
    return v == kInfG ? INF : (int64_t)v;
  };
  auto F = [&](int64_t xx, int64_t i) -> int64_t {
    const int64_t gi = G(i);
    return (xx - i) * (xx - i) + gi * gi;
  };
  int q = 0;
  s[0] = 0;
  t[0] = 0;
  for (int u = 1; u < w; ++u) {
    while (q >= 0 && F(t[q], s[q]) > F(t[q], u)) --q;
    if (q < 0) {
      q = 0;
      s[0] = u;
    } else {
      const int64_t i = s[q];
      const int64_t gu = G(u), gi = G(i);
      const int64_t sep = floordiv64((int64_t)u * u - i * i + gu * gu - gi * gi, 2 * (u - i));
      const int64_t ww = 1 + sep;
      if (ww < w) {
        ++q;
        s[q] = u;
        t[q] = (int32_t)ww;
      }
    }
  }
  for (int u = w - 1; u >= 0; --u) {
    edt_emit(rb + u, F(u, s[q]), dist2, dq, mk, ws_h);
    if (u == t[q]) --q;
  }
}

}  // namespace

int edt(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w,
        int32_t* dist2, uint16_t* dq, uint16_t* mk, int32_t ws_h) {
  const int nseg = (int)ceil_div(h, kSeg);
  uint16_t* seg = reinterpret_cast<uint16_t*>(ctx->seg_summary);
  uint16_t* g = ctx->u16c;
  int32_t* any_zero = ctx->misc + 2;
  int32_t* row_flag = ctx->misc + 64;  // h entries
  RTG_CUDA(cudaMemsetAsync(any_zero, 0, sizeof(int32_t), ctx->stream));
  const dim3 gs((unsigned)ceil_div(w, 128), (unsigned)nseg);
  k_edt_seg<<<gs, 128, 0, ctx->stream>>>(mask, (int)h, (int)w, seg, any_zero);
  RTG_LAUNCH("k_edt_seg");
  k_edt_col<<<gs, 128, 0, ctx->stream>>>(mask, (int)h, (int)w, seg, g);
  RTG_LAUNCH("k_edt_col");
  const size_t smem = sizeof(uint16_t) * (size_t)w;
  k_edt_row<<<(unsigned)h, 256, smem, ctx->stream>>>(g, (int)h, (int)w, any_zero, dist2,
                                                      dq, mk, ws_h, row_flag);
  RTG_LAUNCH("k_edt_row");
  k_edt_row_exact<<<(unsigned)ceil_div(h, 128), 128, 0, ctx->stream>>>(
      g, (int)h, (int)w, row_flag, ctx->i32b, ctx->i32c, dist2, dq, mk, ws_h, ctx->status);
  RTG_LAUNCH("k_edt_row_exact");
  return RTG_OK;
}

}  // namespace rtg
