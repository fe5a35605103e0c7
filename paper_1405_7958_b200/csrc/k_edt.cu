// o6 distance map for PreWatershed: exact squared
// Euclidean distance transform.
//
// Fast path, k_edt_tile: one CTA per 64x64 output tile reads the mask of the
// tile plus a 16-pixel halo (a 96x96 window).  Columns of the window become
// 96-bit masks of background rows, the vertical distance g of every (tile
// row, window column) comes from one ffs / clz on them, and every foreground
// pixel searches outward along its row, stopping as soon as k^2 >= best.  The
// window holds every point within Chebyshev distance 16 of a tile pixel, so
// any result <= 16^2 is exact; a larger one raises a flag and the separable
// whole-tile pass below recomputes everything (it early-exits otherwise).
// Nuclei after the area filter have distances far below 16, so the fallback
// costs four empty launches in the normal case.
//
// Whole-tile pass (fallback, and the semantics the fast path reproduces):
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
#include <type_traits>
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rtg {
namespace {

constexpr int kSeg = 32;
constexpr int kET = 64;               // fast path: output tile edge
constexpr int kER = 16;               //   halo; exact while d2 <= kER^2
constexpr int kEW = kET + 2 * kER;    //   window edge (96 = 3 words)
constexpr uint32_t kInfG = 0xFFFFu;
constexpr int kCap = 96;

// Foreground test of pixel i from the mask bytes or from the 1-bit plane
// (the sparse path's plane; the joint fill/area stage writes only that).
struct ByteFg {
  const uint8_t* m;
  __device__ __forceinline__ bool operator()(int64_t i) const { return m[i] != 0; }
};
struct BitFg {
  const uint32_t* b;  // the plane after its kBitPad pad words
  __device__ __forceinline__ bool operator()(int64_t i) const { return (b[i >> 5] >> (i & 31)) & 1u; }
};

// Column segments: first/last zero row of every (32-row segment, column).
template <class Fg>
__device__ __forceinline__ void edt_seg_phase(const Fg& mask, int h, int w, uint16_t* seg,
                                              int32_t* any_zero) {
  // grid-stride over (segment, column block) pairs: a capped grid keeps the
  // gated (normally empty) launch cheap
  const int nbx = (w + blockDim.x - 1) / blockDim.x, nseg = (h + kSeg - 1) / kSeg;
  for (int blk = blockIdx.x; blk < nbx * nseg; blk += gridDim.x) {
    const int s = blk / nbx, x = (blk - s * nbx) * blockDim.x + threadIdx.x;
    bool z = false;
    if (x < w) {
      int first = 0xFF, last = 0xFF;
      const int y0 = s * kSeg;
      for (int r = 0; r < kSeg && y0 + r < h; ++r) {
        if (!mask((int64_t)(y0 + r) * w + x)) {
          if (first == 0xFF) first = r;
          last = r;
        }
      }
      seg[(int64_t)s * w + x] = (uint16_t)(first | (last << 8));
      z = first != 0xFF;
    }
    if (__any_sync(0xFFFFFFFFu, z) && (threadIdx.x & 31) == 0) atomicOr(any_zero, 1);
  }
}

template <class Fg>
__global__ void k_edt_seg(Fg mask, int h, int w, uint16_t* __restrict__ seg,
                          int32_t* __restrict__ any_zero, const int32_t* __restrict__ gate) {
  pdl_enter();
  if (gate && !*gate) return;
  edt_seg_phase(mask, h, w, seg, any_zero);
}

// Column distances g through the segment summaries.
template <class Fg>
__device__ __forceinline__ void edt_col_phase(const Fg& mask, int h, int w, const uint16_t* seg,
                                              uint16_t* g) {
  const int nbx = (w + blockDim.x - 1) / blockDim.x, nseg = (h + kSeg - 1) / kSeg;
  for (int blk = blockIdx.x; blk < nbx * nseg; blk += gridDim.x) {
    const int s = blk / nbx, x = (blk - s * nbx) * blockDim.x + threadIdx.x;
    if (x >= w) continue;
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
        if (!mask((int64_t)y * w + x)) { zbits |= 1u << r; above = y; }
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
}

template <class Fg>
__global__ void k_edt_col(Fg mask, int h, int w, const uint16_t* __restrict__ seg,
                          uint16_t* __restrict__ g, const int32_t* __restrict__ gate) {
  pdl_enter();
  if (gate && !*gate) return;
  edt_col_phase(mask, h, w, seg, g);
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

// Row search over the column distances (one CTA per row, g staged in shared
// memory); rows that hit kCap are flagged for the exact pass.
__device__ __forceinline__ void edt_row_phase(const uint16_t* g, int h, int w,
                                              const int32_t* any_zero, int32_t* dist2,
                                              uint16_t* dq, uint16_t* mk, int32_t ws_h,
                                              int32_t* row_flag, uint16_t* gs) {
  const bool none = *any_zero == 0;
  for (int y = blockIdx.x; y < h; y += gridDim.x) {  // grid-stride over rows
    const int64_t rb = (int64_t)y * w;
    __syncthreads();  // gs of the previous row fully consumed
    for (int x = threadIdx.x; x < w; x += blockDim.x) gs[x] = g[rb + x];
    __syncthreads();
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
    const bool any = __syncthreads_or(unresolved);
    if (threadIdx.x == 0) row_flag[y] = any ? 1 : 0;
  }
}

__global__ void __launch_bounds__(256)
k_edt_row(const uint16_t* __restrict__ g, int h, int w,
          const int32_t* __restrict__ any_zero, int32_t* __restrict__ dist2,
          uint16_t* __restrict__ dq, uint16_t* __restrict__ mk, int32_t ws_h,
          int32_t* __restrict__ row_flag, const int32_t* __restrict__ gate) {
  pdl_enter();
  extern __shared__ uint16_t gs[];
  if (gate && !*gate) return;  // k_edt_row_exact checks the same gate
  edt_row_phase(g, h, w, any_zero, dist2, dq, mk, ws_h, row_flag, gs);
}

__device__ __forceinline__ int64_t floordiv64(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}

// Exact per-row lower envelope (Meijster phase 2) of one flagged row.
__device__ __forceinline__ void edt_row_exact_one(int y, const uint16_t* g, int h, int w,
                                                  int32_t* s_buf, int32_t* t_buf, int32_t* dist2,
                                                  uint16_t* dq, uint16_t* mk, int32_t ws_h,
                                                  uint32_t* status) {
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

__global__ void k_edt_row_exact(const uint16_t* __restrict__ g, int h, int w,
                                const int32_t* __restrict__ row_flag,
                                int32_t* __restrict__ s_buf, int32_t* __restrict__ t_buf,
                                int32_t* __restrict__ dist2, uint16_t* __restrict__ dq,
                                uint16_t* __restrict__ mk, int32_t ws_h,
                                uint32_t* __restrict__ status,
                                const int32_t* __restrict__ gate = nullptr) {
  pdl_enter();
  if (gate && !*gate) return;
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= h || !row_flag[y]) return;
  edt_row_exact_one(y, g, h, w, s_buf, t_buf, dist2, dq, mk, ws_h, status);
}

// The whole-tile pass as ONE cooperative launch (grid-wide barriers between
// the phases) for the sparse path: when the gate is clear - the normal case
// - the stage pays one empty launch instead of four.
template <class Fg>
__global__ void __launch_bounds__(256)
k_edt_fallback(Fg mask, int h, int w, uint16_t* __restrict__ seg, uint16_t* __restrict__ g,
               int32_t* __restrict__ any_zero, uint16_t* __restrict__ dq,
               int32_t* __restrict__ row_flag, int32_t* __restrict__ s_buf,
               int32_t* __restrict__ t_buf, uint32_t* __restrict__ status,
               const int32_t* __restrict__ gate) {
  extern __shared__ uint16_t gs[];
  if (!*gate) return;  // the same value for every CTA: all leave together
  cg::grid_group grid = cg::this_grid();
  edt_seg_phase(mask, h, w, seg, any_zero);
  grid.sync();
  edt_col_phase(mask, h, w, seg, g);
  grid.sync();
  edt_row_phase(g, h, w, any_zero, nullptr, dq, nullptr, 0, row_flag, gs);
  grid.sync();
  for (int y = blockIdx.x * blockDim.x + threadIdx.x; y < h; y += gridDim.x * blockDim.x)
    if (row_flag[y]) edt_row_exact_one(y, g, h, w, s_buf, t_buf, nullptr, dq, nullptr, 0, status);
}

__device__ __forceinline__ uint32_t isqrt_small(uint32_t v) {  // v < 2^24
  uint32_t r = (uint32_t)__fsqrt_rn((float)v);
  if (r * r > v) --r;
  if ((r + 1) * (r + 1) <= v) ++r;
  return r;
}

__global__ void __launch_bounds__(256)
k_edt_tile(const uint8_t* __restrict__ mask, int h, int w, int32_t* __restrict__ dist2,
           uint16_t* __restrict__ dq, uint16_t* __restrict__ mk, int32_t ws_h,
           int32_t* __restrict__ need_full) {
  pdl_enter();
  __shared__ uint32_t colw[kEW][3];       // bit r of word k: window row 32k + r is background
  __shared__ uint8_t gdn[kET][kEW + 4];   // tile row -> nearest background row below / above
  __shared__ uint8_t gup[kET][kEW + 4];   //   (255: none in the window)
  const int x0 = blockIdx.x * kET, y0 = blockIdx.y * kET;
  const int wx0 = x0 - kER, wy0 = y0 - kER;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // 1. background bits of the window: a task is (4-column group, 32-row word),
  //    32 independent u32 loads when the rows are 4-byte aligned and inside
  const bool vec = (w & 3) == 0 && wx0 >= 0 && wx0 + kEW <= w &&
                   (reinterpret_cast<uintptr_t>(mask) & 3) == 0;
  if (vec) {
    if (tid < (kEW / 4) * 3) {
      const int k = tid / (kEW / 4), cg = tid - k * (kEW / 4);
      uint32_t v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int y = wy0 + 32 * k + r;
        v[r] = (y >= 0 && y < h)
                   ? __ldg(reinterpret_cast<const uint32_t*>(mask + (int64_t)y * w + wx0 + 4 * cg))
                   : 0x01010101u;  // outside the image: not background
      }
      uint32_t b0 = 0, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const uint32_t z = __vcmpeq4(v[r], 0u);  // 0xFF per background byte
        b0 |= ((z >> 7) & 1u) << r;
        b1 |= ((z >> 15) & 1u) << r;
        b2 |= ((z >> 23) & 1u) << r;
        b3 |= ((z >> 31) & 1u) << r;
      }
      colw[4 * cg + 0][k] = b0;
      colw[4 * cg + 1][k] = b1;
      colw[4 * cg + 2][k] = b2;
      colw[4 * cg + 3][k] = b3;
    }
  } else {
    for (int t = tid; t < kEW * 3; t += 256) {
      const int k = t / kEW, c = t - k * kEW;
      const int x = wx0 + c;
      uint32_t bits = 0;
      if (x >= 0 && x < w) {
#pragma unroll 8
        for (int r = 0; r < 32; ++r) {
          const int y = wy0 + 32 * k + r;
          if (y >= 0 && y < h && !__ldg(mask + (int64_t)y * w + x)) bits |= 1u << r;
        }
      }
      colw[c][k] = bits;
    }
  }
  __syncthreads();
  // 2. vertical distances: one thread sweeps one window column downwards
  //    (threads 0..95) or upwards (96..191); bits stay in registers
  if (tid < 2 * kEW) {
    const int c = tid < kEW ? tid : tid - kEW;
    const uint32_t cw[3] = {colw[c][0], colw[c][1], colw[c][2]};
    if (tid < kEW) {
      int last = -1000;
#pragma unroll
      for (int r = 0; r < kER + kET; ++r) {
        if ((cw[r >> 5] >> (r & 31)) & 1u) last = r;
        if (r >= kER) gdn[r - kER][c] = (uint8_t)min(r - last, 255);
      }
    } else {
      int next = 1000;
#pragma unroll
      for (int r = kEW - 1; r >= kER; --r) {
        if ((cw[r >> 5] >> (r & 31)) & 1u) next = r;
        if (r < kER + kET) gup[r - kER][c] = (uint8_t)min(next - r, 255);
      }
    }
  }
  __syncthreads();
  // 3. row search for the tile pixels
  bool far = false;
#pragma unroll 2
  for (int q = 0; q < 16; ++q) {
    const int r = wid * 8 + (q >> 1), c = (q & 1) * 32 + lane;
    const int y = y0 + r, x = x0 + c;
    if (y >= h || x >= w) continue;
    const int wc = c + kER;
    const uint32_t g0 = min(gdn[r][wc], gup[r][wc]);
    uint32_t best;
    if (g0 == 0) {
      best = 0;
    } else {
      best = g0 == 255 ? 0xFFFFFFFFu : g0 * g0;
      for (uint32_t k = 1; k <= (uint32_t)kER && k * k < best; ++k) {
        const uint32_t gm = min(min(gdn[r][wc - k], gup[r][wc - k]),
                                min(gdn[r][wc + k], gup[r][wc + k]));
        if (gm != 255) best = min(best, k * k + gm * gm);
      }
      if (best > (uint32_t)(kER * kER)) far = true;
    }
    const int64_t i = (int64_t)y * w + x;
    if (dist2) dist2[i] = (int32_t)min(best, 0x7FFFFFFFu);
    const uint32_t v = best > (uint32_t)(kER * kER) ? 65534u : isqrt_small(16u * best);
    if (dq) dq[i] = (uint16_t)v;
    if (mk) mk[i] = (uint16_t)(v > (uint32_t)ws_h ? v - (uint32_t)ws_h : 0u);
  }
  if (__syncthreads_or(far) && tid == 0) *need_full = 1;
}

// ---- foreground list + bit plane (sparse path of the watershed) ----------------
// bits: one bit per pixel (raster order, 1 = foreground), with kBitPad zero
// words before and after so 64-bit windows never leave the allocation.  The
// list holds every foreground index, in raster order within a block.
// Each thread covers 16 consecutive pixels (one 16-byte load when aligned), so
// a block reserves list slots once per 4096 pixels.
__global__ void __launch_bounds__(256)
k_fg_list(const uint8_t* __restrict__ mask, int64_t n, uint32_t* __restrict__ bits,
          int32_t* __restrict__ list, int32_t* __restrict__ count) {
  pdl_enter();
  __shared__ int32_t sm[9];
  const bool vec = (reinterpret_cast<uintptr_t>(mask) & 15) == 0;
  for (int64_t b0 = (int64_t)blockIdx.x * 4096; b0 < n; b0 += (int64_t)gridDim.x * 4096) {
    const int64_t p0 = b0 + 16 * (int64_t)threadIdx.x;
    uint32_t m = 0;  // bit k: pixel p0 + k is foreground
    if (vec && p0 + 16 <= n) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(mask + p0));
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t z = ~__vcmpeq4(wv[q], 0u);  // 0xFF per foreground byte
        m |= (((z >> 7) & 1u) | ((z >> 14) & 2u) | ((z >> 21) & 4u) | ((z >> 28) & 8u)) << (4 * q);
      }
    } else {
      for (int k = 0; k < 16; ++k)
        if (p0 + k < n && mask[p0 + k]) m |= 1u << k;
    }
    // 32-pixel words: even lane = low half, odd lane = high half
    const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, m, 1);
    if (!(threadIdx.x & 1) && p0 < n) bits[p0 >> 5] = m | (other << 16);
    int32_t slot = block_reserve(__popc(m), count, sm);
    for (uint32_t r = m; r; r &= r - 1) list[slot++] = (int32_t)(p0 + __ffs(r) - 1);
  }
}

// Distance from column x to the nearest background pixel of the row starting
// at bit `rb`, within +-32 columns; 255 if none.
__device__ __forceinline__ uint32_t row_nearest_bg(const uint32_t* __restrict__ bits, int32_t rb,
                                                   int x, int w) {
  const int32_t c = rb + x;
  const int32_t wa = c >> 5, wb = (c - 32) >> 5;  // arithmetic shift: -1 for the first word
  const uint32_t sa = (uint32_t)c & 31u;
  const uint32_t hi = __funnelshift_r(bits[wa], bits[wa + 1], sa);   // columns x .. x+31
  const uint32_t lo = __funnelshift_r(bits[wb], bits[wb + 1], sa);   // columns x-32 .. x-1
  const int right_valid = w - x;   // columns x .. w-1
  const uint32_t mh = right_valid >= 32 ? 0xFFFFFFFFu : ((1u << right_valid) - 1u);
  const uint32_t ml = x >= 32 ? 0xFFFFFFFFu : ~((1u << (32 - x)) - 1u);
  const uint32_t bh = ~hi & mh, bl = ~lo & ml;
  const uint32_t dr = bh ? (uint32_t)(__ffs(bh) - 1) : 255u;
  const uint32_t dl = bl ? (uint32_t)(__clz(bl) + 1) : 255u;
  return min(dr, dl);
}

// Separable exact EDT over the foreground list.  Pass 1: every listed pixel's
// distance to the nearest background pixel of its own row (within +-32
// columns, 255 beyond), from two funnel-shifted words of the 1-bit plane.
__global__ void __launch_bounds__(256)
k_edt_rowdist(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
              const uint32_t* __restrict__ bits, FastDiv dw, uint8_t* __restrict__ hd, int h,
              uint8_t* __restrict__ nbm) {
  pdl_enter();
  const int w = (int)dw.d;
  const int n = *count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t p = list[k];
    const int y = fdiv(p, dw), x = p - y * w;
    hd[p] = (uint8_t)row_nearest_bg(bits, y * w, x, w);
    if (nbm) nbm[k] = (uint8_t)fg_nbrs(h, w, bits, p, y, x);
  }
}

// Pass 2: d2 = min over rows y +- dy of dy^2 + hd^2 (background pixels have
// hd = 0; the 1-bit plane tells them apart), scanned outwards until dy^2 >=
// best.  Exact while the result is <= 32^2 (every background pixel within
// Chebyshev distance 32 is seen); beyond that need_full is raised and the
// whole-tile pass runs.
template <bool kBgZero>
__global__ void __launch_bounds__(256)
k_edt_list(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
           const uint32_t* __restrict__ bits, const uint8_t* __restrict__ hd, int h, FastDiv dw,
           int32_t* __restrict__ dist2, uint16_t* __restrict__ dq,
           int32_t* __restrict__ need_full) {
  pdl_enter();
  constexpr uint32_t kR = 32;
  const int w = (int)dw.d;
  const int n = *count;
  bool far = false;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t p = list[k];
    const int y = fdiv(p, dw);
    const uint32_t d0 = hd[p];
    uint32_t best = d0 == 255u ? 0xFFFFFFFFu : d0 * d0;
    // rows are visited in batches of kB with every load of the batch in
    // flight together (mask and hd bytes unconditionally, selected after):
    // rows past the stopping point only add candidates >= dy^2 >= best, so
    // the result is the same as the row-by-row scan
    constexpr uint32_t kB = 4;
    // a row without background within range has hd = 255: its candidate is
    // >= 255^2 > kR^2, which ends in the need_full branch exactly as a
    // skipped row would, so no test is needed; pixels >= kR rows from both
    // image edges (nearly all) skip the bounds tests too
    auto scan = [&](auto checked) {
      for (uint32_t dy0 = 1; dy0 <= kR && dy0 * dy0 < best; dy0 += kB) {
        uint32_t mu[kB], hu[kB], md[kB], hdn[kB];
#pragma unroll
        for (uint32_t j = 0; j < kB; ++j) {
          const uint32_t dy = dy0 + j;
          const bool vu = !checked.value || y >= (int)dy, vd = !checked.value || y + (int)dy < h;
          const int32_t qu = p - (int32_t)dy * w, qd = p + (int32_t)dy * w;
          // kBgZero: the hd plane holds 0 at background pixels (the joint
          // fill/area stage wrote the mask bytes there), no bit tests
          mu[j] = kBgZero ? 1u : vu ? (bits[qu >> 5] >> (qu & 31)) & 1u : 1u;
          hu[j] = vu ? hd[qu] : 255u;
          md[j] = kBgZero ? 1u : vd ? (bits[qd >> 5] >> (qd & 31)) & 1u : 1u;
          hdn[j] = vd ? hd[qd] : 255u;
        }
#pragma unroll
        for (uint32_t j = 0; j < kB; ++j) {
          const uint32_t dy = dy0 + j;
          const uint32_t dm = min(mu[j] ? hu[j] : 0u, md[j] ? hdn[j] : 0u);
          best = min(best, dy * dy + dm * dm);
        }
      }
    };
    if (y >= (int)kR && y + (int)kR < h) scan(std::false_type{});
    else scan(std::true_type{});
    if (best > kR * kR) {
      far = true;
      continue;
    }
    if (dist2) dist2[p] = (int32_t)best;
    dq[p] = (uint16_t)isqrt_small(16u * best);
  }
  if (__any_sync(0xFFFFFFFFu, far) && (threadIdx.x & 31) == 0) *need_full = 1;
}

}  // namespace

int edt(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w,
        int32_t* dist2, uint16_t* dq, uint16_t* mk, int32_t ws_h) {
  const int nseg = (int)ceil_div(h, kSeg);
  uint16_t* seg = reinterpret_cast<uint16_t*>(ctx->seg_summary);
  uint16_t* g = ctx->u16c;
  int32_t* any_zero = ctx->misc + 2;
  int32_t* need_full = ctx->misc + 3;
  int32_t* row_flag = ctx->misc + 64;  // h entries
  RTG_TRY(zero_async(ctx, ZeroList{{any_zero}, {2 * sizeof(int32_t)}, 1}));  // + need_full
  const dim3 tiles((unsigned)ceil_div(w, kET), (unsigned)ceil_div(h, kET));
  RTG_CUDA(launch_k(ctx, k_edt_tile, tiles, 256, 0, mask, (int)h, (int)w, dist2, dq, mk, ws_h,
                                             need_full));
  RTG_LAUNCH("k_edt_tile");
  // exact whole-tile pass, gated on need_full (empty launches otherwise)
  const int64_t gblk = ceil_div(w, 128) * nseg;
  const unsigned gs = (unsigned)(gblk < ctx->num_sms * 4 ? gblk : ctx->num_sms * 4);
  RTG_CUDA(launch_k(ctx, k_edt_seg<ByteFg>, gs, 128, 0, ByteFg{mask}, (int)h, (int)w, seg,
                    any_zero, (const int32_t*)need_full));
  RTG_LAUNCH("k_edt_seg");
  RTG_CUDA(launch_k(ctx, k_edt_col<ByteFg>, gs, 128, 0, ByteFg{mask}, (int)h, (int)w,
                    (const uint16_t*)seg, g, (const int32_t*)need_full));
  RTG_LAUNCH("k_edt_col");
  const size_t smem = sizeof(uint16_t) * (size_t)w;
  const unsigned grows = (unsigned)(h < ctx->num_sms * 4 ? h : ctx->num_sms * 4);
  RTG_CUDA(launch_k(ctx, k_edt_row, grows, 256, smem, g, (int)h, (int)w, any_zero, dist2,
                                                      dq, mk, ws_h, row_flag, need_full));
  RTG_LAUNCH("k_edt_row");
  RTG_CUDA(launch_k(ctx, k_edt_row_exact, (unsigned)ceil_div(h, 128), 128, 0, 
      g, (int)h, (int)w, row_flag, ctx->i32b, ctx->i32c, dist2, dq, mk, ws_h, ctx->status,
      need_full));
  RTG_LAUNCH("k_edt_row_exact");
  return RTG_OK;
}

}  // namespace rtg

namespace rtg {

int fg_list(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w, int32_t* list,
            int32_t* count, uint32_t* bits_base) {
  const int64_t n = h * w;
  // count + pads (the words past the image end are partly written by the ballots)
  RTG_TRY(zero_async(ctx, ZeroList{{count, bits_base, bits_base + kBitPad + n / 32},
                                    {sizeof(int32_t), sizeof(uint32_t) * kBitPad,
                                     sizeof(uint32_t) * (kBitPad + 1)},
                                    3}));
  int blocks = (int)ceil_div(n, 4096);
  if (blocks > ctx->num_sms * 8) blocks = ctx->num_sms * 8;
  RTG_CUDA(launch_k(ctx, k_fg_list, blocks, 256, 0, mask, n, bits_base + kBitPad, list, count));
  RTG_LAUNCH("k_fg_list");
  return RTG_OK;
}

int edt_list(rtg_ctx* ctx, int64_t h, int64_t w, const int32_t* list,
             const int32_t* count, const uint32_t* bits_base, uint16_t* dq, uint8_t* nbm,
             uint8_t* hd_mask) {
  const int nseg = (int)ceil_div(h, kSeg);
  uint16_t* seg = reinterpret_cast<uint16_t*>(ctx->seg_summary);
  uint16_t* g = ctx->u16c;
  int32_t* any_zero = ctx->misc + 2;
  int32_t* need_full = ctx->misc + 3;
  int32_t* row_flag = ctx->misc + 64;
  // any_zero / need_full were zeroed by the caller (watershed)
  // row distances: into the mask bytes themselves when given (background
  // stays 0, foreground becomes its distance >= 1), else into m2
  uint8_t* hd = hd_mask ? hd_mask : ctx->m2;
  const FastDiv dwv = make_div((uint32_t)w);
  RTG_CUDA(launch_k(ctx, k_edt_rowdist, ctx->num_sms * 8, 256, 0, list, count, bits_base + kBitPad, dwv,
                                                           hd, (int)h, nbm));
  RTG_LAUNCH("k_edt_rowdist");
  const uint32_t* bits = bits_base + kBitPad;
  RTG_CUDA(launch_k(ctx, hd_mask ? k_edt_list<true> : k_edt_list<false>, ctx->num_sms * 8, 256, 0,
                    list, count, bits, (const uint8_t*)hd, (int)h, dwv,
                                                        nullptr, dq, need_full));
  RTG_LAUNCH("k_edt_list");
  // the exact whole-tile pass, gated on need_full, as one cooperative launch
  (void)nseg;
  const size_t smem = sizeof(uint16_t) * (size_t)w;
  static int occ_dev[64] = {0};  // co-resident CTAs per SM (per device)
  int& occ = occ_dev[ctx->device & 63];
  if (!occ) {
    int o = 0;
    RTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_edt_fallback<BitFg>, 256, smem));
    if (o < 1) return fail(RTG_ERR_INTERNAL, "k_edt_fallback does not fit on an SM");
    occ = o > 2 ? 2 : o;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(ctx->num_sms * occ));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RTG_CUDA(cudaLaunchKernelEx(&cfg, k_edt_fallback<BitFg>, BitFg{bits}, (int)h, (int)w, seg, g,
                              any_zero, dq, row_flag, ctx->i32b, ctx->i32c, ctx->status,
                              (const int32_t*)need_full));
  RTG_LAUNCH("k_edt_fallback");
  return RTG_OK;
}

}  // namespace rtg
