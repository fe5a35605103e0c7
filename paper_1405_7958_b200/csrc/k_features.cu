// o9 per-object features, the paper's two-step scheme:
// step 1 reduces pixels into fixed-size per-object intermediates (moments,
// intensity and gradient sums, perimeter edges, bbox, min/max), step 2 runs
// one thread per object to turn them into the feature row.
//
// Step 1 is a two-level reduction: vertical runs accumulated in registers
// into a per-block shared-memory table, flushed once per (object, 64x64
// block).  All
// intermediates are integers, so step 1 is order-independent and exact; step
// 2 is fp64 with FMA contraction disabled (--fmad=false), matching the oracle.
//
// Roofline: HBM/L2 bound; algorithmic bytes labels 4 B + intensity 1 B per px.
#include "common.cuh"

namespace rtg {
namespace {

__global__ void k_feat_clear(const int32_t* __restrict__ d_n, FeatureAcc acc) {
  pdl_enter();
  const int n = min(*d_n, acc.cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
    for (int f = 0; f < kSumFields; ++f) acc.sums[(int64_t)f * acc.cap + i] = 0ull;
#pragma unroll
    for (int f = 0; f < kMinFields; ++f) acc.mins[(int64_t)f * acc.cap + i] = INT32_MAX;
#pragma unroll
    for (int f = 0; f < kMaxFields; ++f) acc.maxs[(int64_t)f * acc.cap + i] = -1;
  }
}

// Step 1, one CTA per 64x64 block: every lane walks 16 rows down one column
// and accumulates the vertical run of the current label in registers (x is
// constant along a column, so the x moments follow from n and sum y); a run
// ends at a label change and is added into a per-block table in shared memory
// keyed by label (open addressing), in block-local coordinates so the sums
// fit 32 bits (except sum g^2).  The table is flushed with one set of global
// atomics per (object, block).  A run whose label finds the table full goes
// straight to the global accumulators.  Labels and intensities of the block
// (+ halo) are staged in shared memory first with coalesced loads.
constexpr int kFB = 64;        // block edge
constexpr int kStrip = 16;     // rows per lane walk (4 strips x 2 column halves = 8 warps)
constexpr int kSlots = 256;    // table entries per block
constexpr int kHalo = kFB + 2; // staged block + 1-pixel halo
enum { kTA = 0, kTY, kTX, kTYY, kTXX, kTXY, kTI, kTII, kTG, kTP, kTFields };

struct FeatTable {
  int32_t key[kSlots];
  uint32_t s[kTFields][kSlots];
  unsigned long long gg[kSlots];
  int32_t mn[kMinFields][kSlots];
  int32_t mx[kMaxFields][kSlots];
};

__device__ __forceinline__ int table_slot(FeatTable& T, int32_t l) {
  int s = (int)((uint32_t)l * 2654435761u >> 24);  // 8-bit hash
  for (int probe = 0; probe < kSlots; ++probe, s = (s + 1) & (kSlots - 1)) {
    const int32_t k = T.key[s];
    if (k == l) return s;
    if (k == 0) {
      const int32_t old = atomicCAS(&T.key[s], 0, l);
      if (old == 0 || old == l) return s;
    }
  }
  return -1;
}

// One vertical run (block-local coordinates; xl fixed).
struct ColRun {
  uint32_t n, sy, syy, si, sii, sg, sp, mni, mxi, y0, y1;
  unsigned long long sgg;
};

__device__ __forceinline__ void run_flush(FeatTable& T, const FeatureAcc& acc, int32_t l,
                                          const ColRun& a, uint32_t xl, int by0, int bx0) {
  const int s = table_slot(T, l);
  if (s >= 0) {
    atomicAdd(&T.s[kTA][s], a.n);
    atomicAdd(&T.s[kTY][s], a.sy);
    atomicAdd(&T.s[kTX][s], a.n * xl);
    atomicAdd(&T.s[kTYY][s], a.syy);
    atomicAdd(&T.s[kTXX][s], a.n * xl * xl);
    atomicAdd(&T.s[kTXY][s], a.sy * xl);
    atomicAdd(&T.s[kTI][s], a.si);
    atomicAdd(&T.s[kTII][s], a.sii);
    atomicAdd(&T.s[kTG][s], a.sg);
    atomicAdd(&T.s[kTP][s], a.sp);
    atomicAdd(&T.gg[s], a.sgg);
    atomicMin(&T.mn[kMinI][s], (int32_t)a.mni);
    atomicMin(&T.mn[kMinY][s], (int32_t)a.y0);
    atomicMin(&T.mn[kMinX][s], (int32_t)xl);
    atomicMax(&T.mx[kMaxI][s], (int32_t)a.mxi);
    atomicMax(&T.mx[kMaxY][s], (int32_t)a.y1);
    atomicMax(&T.mx[kMaxX][s], (int32_t)xl);
    return;
  }
  // table full: global accumulators directly (global coordinates)
  const int64_t c = acc.cap, k = l - 1;
  const unsigned long long n = a.n, Y = by0, X = (unsigned long long)bx0 + xl;
  unsigned long long* S = acc.sums;
  atomicAdd(&S[kSumArea * c + k], n);
  atomicAdd(&S[kSumY * c + k], a.sy + n * Y);
  atomicAdd(&S[kSumX * c + k], n * X);
  atomicAdd(&S[kSumYY * c + k], a.syy + 2 * Y * a.sy + n * Y * Y);
  atomicAdd(&S[kSumXX * c + k], n * X * X);
  atomicAdd(&S[kSumXY * c + k], X * (a.sy + n * Y));
  atomicAdd(&S[kSumI * c + k], (unsigned long long)a.si);
  atomicAdd(&S[kSumII * c + k], (unsigned long long)a.sii);
  atomicAdd(&S[kSumG * c + k], (unsigned long long)a.sg);
  atomicAdd(&S[kSumGG * c + k], a.sgg);
  atomicAdd(&S[kSumPerim * c + k], (unsigned long long)a.sp);
  atomicMin(&acc.mins[kMinI * c + k], (int32_t)a.mni);
  atomicMin(&acc.mins[kMinY * c + k], by0 + (int32_t)a.y0);
  atomicMin(&acc.mins[kMinX * c + k], (int32_t)X);
  atomicMax(&acc.maxs[kMaxI * c + k], (int32_t)a.mxi);
  atomicMax(&acc.maxs[kMaxY * c + k], by0 + (int32_t)a.y1);
  atomicMax(&acc.maxs[kMaxX * c + k], (int32_t)X);
}

__device__ __forceinline__ uint32_t isqrt_small(uint32_t v) {  // v < 2^26
  uint32_t r = (uint32_t)__fsqrt_rn((float)v);
  if (r * r > v) --r;
  if ((r + 1) * (r + 1) <= v) ++r;
  return r;
}

__global__ void __launch_bounds__(256)
k_feat_accum(const int32_t* __restrict__ labels, const uint8_t* __restrict__ I,
             int h, int w, const int32_t* __restrict__ d_n, FeatureAcc acc) {
  pdl_enter();
  __shared__ FeatTable T;
  __shared__ int32_t SL[kHalo][kHalo];
  __shared__ uint8_t SI[kHalo][kHalo + 2];
  const int nobj = min(*d_n, acc.cap);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int bx0 = blockIdx.x * kFB, by0 = blockIdx.y * kFB;
  for (int k = threadIdx.x; k < kSlots; k += blockDim.x) {
    T.key[k] = 0;
#pragma unroll
    for (int f = 0; f < kTFields; ++f) T.s[f][k] = 0;
    T.gg[k] = 0;
#pragma unroll
    for (int f = 0; f < kMinFields; ++f) T.mn[f][k] = INT32_MAX;
#pragma unroll
    for (int f = 0; f < kMaxFields; ++f) T.mx[f][k] = -1;
  }
  __syncthreads();
  // stage labels (invalid -> 0, outside -> 0) and intensities (clamped, the
  // Sobel border rule) of the block plus a 1-pixel halo
  for (int k = threadIdx.x; k < kHalo * kHalo; k += blockDim.x) {
    const int yy = k / kHalo, xx = k - yy * kHalo;
    const int y = by0 - 1 + yy, x = bx0 - 1 + xx;
    int32_t l = 0;
    if (y >= 0 && y < h && x >= 0 && x < w) {
      l = labels[(int64_t)y * w + x];
      l = l > 0 && l <= nobj ? l : 0;
    }
    const int yc = min(max(y, 0), h - 1), xc = min(max(x, 0), w - 1);
    SL[yy][xx] = l;
    SI[yy][xx] = I[(int64_t)yc * w + xc];
  }
  __syncthreads();
  const uint32_t xl = (uint32_t)((wid & 1) * 32 + lane);
  const int x = bx0 + (int)xl;
  const int rs = (wid >> 1) * kStrip;
  if (x < w) {
    const int cx = (int)xl + 1;  // staged column
    int32_t cur = 0;
    ColRun a{};
#pragma unroll 4
    for (int r = rs; r < rs + kStrip; ++r) {
      const int y = by0 + r;
      if (y >= h) break;
      const int32_t l = SL[r + 1][cx];
      if (l != cur) {
        if (cur) run_flush(T, acc, cur, a, xl, by0, bx0);
        cur = l;
        a = ColRun{};
        a.mni = 0xFFFFFFFFu;
        a.y0 = (uint32_t)r;
      }
      if (l) {
        const int t0 = SI[r][cx - 1], t1 = SI[r][cx], t2 = SI[r][cx + 1];
        const int m0 = SI[r + 1][cx - 1], m2 = SI[r + 1][cx + 1];
        const int b0 = SI[r + 2][cx - 1], b1 = SI[r + 2][cx], b2 = SI[r + 2][cx + 1];
        const int gx = (t2 + 2 * m2 + b2) - (t0 + 2 * m0 + b0);
        const int gy = (b0 + 2 * b1 + b2) - (t0 + 2 * t1 + t2);
        const uint32_t gq = isqrt_small(16u * (uint32_t)(gx * gx + gy * gy));
        const uint32_t v = SI[r + 1][cx], yl = (uint32_t)r;
        const uint32_t per = (SL[r][cx] != l) + (SL[r + 2][cx] != l) + (SL[r + 1][cx - 1] != l) +
                             (SL[r + 1][cx + 1] != l);
        a.n += 1;
        a.sy += yl;
        a.syy += yl * yl;
        a.si += v;
        a.sii += v * v;
        a.sg += gq;
        a.sgg += (unsigned long long)(gq * gq);
        a.sp += per;
        a.mni = min(a.mni, v);
        a.mxi = max(a.mxi, v);
        a.y1 = yl;
      }
    }
    if (cur) run_flush(T, acc, cur, a, xl, by0, bx0);
  }
  __syncthreads();
  // flush: block-local moments -> global coordinates (exact u64 arithmetic)
  const int64_t c = acc.cap;
  for (int s = threadIdx.x; s < kSlots; s += blockDim.x) {
    const int32_t l = T.key[s];
    if (l == 0) continue;
    const int64_t k = l - 1;
    const unsigned long long n = T.s[kTA][s], Y = by0, X = bx0;
    const unsigned long long sy = T.s[kTY][s], sx = T.s[kTX][s];
    unsigned long long* S = acc.sums;
    atomicAdd(&S[kSumArea * c + k], n);
    atomicAdd(&S[kSumY * c + k], sy + n * Y);
    atomicAdd(&S[kSumX * c + k], sx + n * X);
    atomicAdd(&S[kSumYY * c + k], T.s[kTYY][s] + 2 * Y * sy + n * Y * Y);
    atomicAdd(&S[kSumXX * c + k], T.s[kTXX][s] + 2 * X * sx + n * X * X);
    atomicAdd(&S[kSumXY * c + k], T.s[kTXY][s] + X * sy + Y * sx + n * X * Y);
    atomicAdd(&S[kSumI * c + k], (unsigned long long)T.s[kTI][s]);
    atomicAdd(&S[kSumII * c + k], (unsigned long long)T.s[kTII][s]);
    atomicAdd(&S[kSumG * c + k], (unsigned long long)T.s[kTG][s]);
    atomicAdd(&S[kSumGG * c + k], T.gg[s]);
    atomicAdd(&S[kSumPerim * c + k], (unsigned long long)T.s[kTP][s]);
    atomicMin(&acc.mins[kMinI * c + k], T.mn[kMinI][s]);
    atomicMin(&acc.mins[kMinY * c + k], by0 + T.mn[kMinY][s]);
    atomicMin(&acc.mins[kMinX * c + k], bx0 + T.mn[kMinX][s]);
    atomicMax(&acc.maxs[kMaxI * c + k], T.mx[kMaxI][s]);
    atomicMax(&acc.maxs[kMaxY * c + k], by0 + T.mx[kMaxY][s]);
    atomicMax(&acc.maxs[kMaxX * c + k], bx0 + T.mx[kMaxX][s]);
  }
}

// Step 1 over a foreground list (the sparse path: a superset of the labelled
// pixels, raster-ordered within blocks).  A warp takes 32 consecutive list
// entries; consecutive lanes of one label on one row form a run, reduced with
// a segmented shuffle reduction (runs are contiguous in lane order, so no
// match/collective loops); the run head issues one set of global atomics.
// y is constant along a run, so the y moments follow from n and sum x.
__global__ void __launch_bounds__(256)
k_feat_list(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
            const int32_t* __restrict__ labels, const uint8_t* __restrict__ I, int h, FastDiv dw,
            const int32_t* __restrict__ d_n, FeatureAcc acc) {
  pdl_enter();
  const unsigned full = 0xFFFFFFFFu;
  const int w = (int)dw.d;
  const int nobj = min(*d_n, acc.cap);
  const int n = *count;
  const int lane = threadIdx.x & 31;
  const int64_t c = acc.cap;
  for (int k0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; k0 < n;
       k0 += gridDim.x * blockDim.x) {
    const int k = k0 + lane;
    int32_t p = 0, l = 0;
    if (k < n) {
      p = list[k];
      l = labels[p];
    }
    if (!(l > 0 && l <= nobj)) l = 0;
    if (!__any_sync(full, l != 0)) continue;
    const int y = fdiv(p, dw), x = p - y * w;
    uint32_t v = 0, gq = 0, per = 0;
    if (l) {
      const int ym = y > 0 ? y - 1 : 0, yp = y + 1 < h ? y + 1 : h - 1;
      const int xm = x > 0 ? x - 1 : 0, xp = x + 1 < w ? x + 1 : w - 1;
      const uint8_t* rm = I + (int64_t)ym * w;
      const uint8_t* r0 = I + (int64_t)y * w;
      const uint8_t* rp = I + (int64_t)yp * w;
      const int gx = ((int)rm[xp] + 2 * (int)r0[xp] + (int)rp[xp]) -
                     ((int)rm[xm] + 2 * (int)r0[xm] + (int)rp[xm]);
      const int gy = ((int)rp[xm] + 2 * (int)rp[x] + (int)rp[xp]) -
                     ((int)rm[xm] + 2 * (int)rm[x] + (int)rm[xp]);
      gq = isqrt_small(16u * (uint32_t)(gx * gx + gy * gy));
      v = r0[x];
      per = (y == 0 || labels[p - w] != l) + (y == h - 1 || labels[p + w] != l) +
            (x == 0 || labels[p - 1] != l) + (x == w - 1 || labels[p + 1] != l);
    }
    // runs: a lane starts one unless its left lane has the same label and row
    const int32_t l_prev = __shfl_up_sync(full, l, 1);
    const int y_prev = __shfl_up_sync(full, y, 1);
    const unsigned heads = __ballot_sync(full, lane == 0 || l != l_prev || y != y_prev);
    // segmented reduction towards the run head: lanes (lane, lane + off] must
    // hold no head
    uint32_t sx = l ? (uint32_t)x : 0u, sxx = sx * sx, si = v, sii = v * v, sg = gq,
             sgg = gq * gq, sp = per, mni = l ? v : 0xFFFFFFFFu, mxi = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t ox = __shfl_down_sync(full, sx, off);
      const uint32_t oxx = __shfl_down_sync(full, sxx, off);
      const uint32_t oi = __shfl_down_sync(full, si, off);
      const uint32_t oii = __shfl_down_sync(full, sii, off);
      const uint32_t og = __shfl_down_sync(full, sg, off);
      const uint32_t ogg = __shfl_down_sync(full, sgg, off);
      const uint32_t op = __shfl_down_sync(full, sp, off);
      const uint32_t omn = __shfl_down_sync(full, mni, off);
      const uint32_t omx = __shfl_down_sync(full, mxi, off);
      const uint32_t span = ((heads >> 1) >> lane) & ((1u << off) - 1u);  // heads in (lane, lane+off]
      if (lane + off < 32 && span == 0) {
        sx += ox;
        sxx += oxx;
        si += oi;
        sii += oii;
        sg += og;
        sgg += ogg;
        sp += op;
        mni = min(mni, omn);
        mxi = max(mxi, omx);
      }
    }
    // run = lanes [lane, end] for a head lane; its last pixel has the largest x
    const unsigned after = (heads >> 1) >> lane;  // heads strictly after this lane
    const int end = after ? lane + __ffs(after) - 1 : 31;
    const int x_end = __shfl_sync(full, x, end);
    if (!l || !((heads >> lane) & 1u)) continue;
    const int64_t o = l - 1;
    const unsigned long long nn = (unsigned long long)(end - lane + 1), Y = (unsigned long long)y;
    unsigned long long* S = acc.sums;
    atomicAdd(&S[kSumArea * c + o], nn);
    atomicAdd(&S[kSumY * c + o], nn * Y);
    atomicAdd(&S[kSumX * c + o], (unsigned long long)sx);
    atomicAdd(&S[kSumYY * c + o], nn * Y * Y);
    atomicAdd(&S[kSumXX * c + o], (unsigned long long)sxx);
    atomicAdd(&S[kSumXY * c + o], Y * sx);
    atomicAdd(&S[kSumI * c + o], (unsigned long long)si);
    atomicAdd(&S[kSumII * c + o], (unsigned long long)sii);
    atomicAdd(&S[kSumG * c + o], (unsigned long long)sg);
    atomicAdd(&S[kSumGG * c + o], (unsigned long long)sgg);
    atomicAdd(&S[kSumPerim * c + o], (unsigned long long)sp);
    atomicMin(&acc.mins[kMinI * c + o], (int32_t)mni);
    atomicMin(&acc.mins[kMinY * c + o], y);
    atomicMin(&acc.mins[kMinX * c + o], x);
    atomicMax(&acc.maxs[kMaxI * c + o], (int32_t)mxi);
    atomicMax(&acc.maxs[kMaxY * c + o], y);
    atomicMax(&acc.maxs[kMaxX * c + o], x_end);
  }
}

// Step 1, one warp per 32x32 tile, no per-pixel atomics: the tile's labels
// and intensities (+ 1-pixel halo) are staged in shared memory; lane r owns
// row r.  The warp walks the tile's objects one at a time (the label of the
// first unvisited pixel of the lowest row holding one): every lane builds the
// 32-bit mask of that object's pixels in its row, derives the shape moments,
// bbox and perimeter from the masks (the rows above and below by shuffles,
// the halo at the tile edges), loops over the mask bits for the intensity
// and Sobel sums, and the warp reduces each field once; lane j then issues
// the global atomic of field j.  One set of atomics per (object, tile) -
// about 40k per 4096^2 tile instead of one per row run (7.3M with the list
// kernel).  Moments are tile-local (small integers) until the flush.
constexpr int kFT = 32;        // tile edge
constexpr int kLS = 35;        // staged label row stride (34 used; 35: conflict-free columns)
constexpr int kIS8 = 36;       // staged intensity row stride in bytes

struct FeatTileSmem {
  int32_t L[kFT + 2][kLS];
  uint8_t I[kFT + 2][kIS8];
};

__global__ void __launch_bounds__(128)
k_feat_tiles(const int32_t* __restrict__ labels, const uint8_t* __restrict__ I, int h, int w,
             int tiles_x, int ntiles, const int32_t* __restrict__ d_n, FeatureAcc acc) {
  pdl_enter();
  __shared__ FeatTileSmem S4[4];
  const unsigned full = 0xFFFFFFFFu;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * 4 + wid;
  if (tile >= ntiles) return;  // warps work independently (no block barrier)
  FeatTileSmem& S = S4[wid];
  const int nobj = min(*d_n, acc.cap);
  const int x0 = (tile % tiles_x) * kFT, y0 = (tile / tiles_x) * kFT;
  auto lab = [&](int y, int x) -> int32_t {
    if (y < 0 || y >= h || x < 0 || x >= w) return 0;
    const int32_t l = labels[(int64_t)y * w + x];
    return l > 0 && l <= nobj ? l : 0;
  };
  // 1. stage: row r of the tile is staged row r + 1, column c is c + 1
  const int y = y0 + lane;
  uint32_t rowbits = 0;  // this lane's labelled pixels
  if (y < h && x0 + kFT <= w && (w & 3) == 0) {
    const int4* src = reinterpret_cast<const int4*>(labels + (int64_t)y * w + x0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int4 v = __ldg(src + q);
      const int32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int32_t l = e[j] > 0 && e[j] <= nobj ? e[j] : 0;
        S.L[lane + 1][4 * q + j + 1] = l;
        rowbits |= (l ? 1u : 0u) << (4 * q + j);
      }
    }
  } else {
    for (int c = 0; c < kFT; ++c) {
      const int32_t l = lab(y, x0 + c);
      S.L[lane + 1][c + 1] = l;
      rowbits |= (l ? 1u : 0u) << c;
    }
  }
  if (!__any_sync(full, rowbits != 0)) return;  // no object in this tile
  S.L[lane + 1][0] = lab(y, x0 - 1);
  S.L[lane + 1][kFT + 1] = lab(y, x0 + kFT);
  for (int c = lane; c < kFT + 2; c += 32) {
    S.L[0][c] = lab(y0 - 1, x0 - 1 + c);
    S.L[kFT + 1][c] = lab(y0 + kFT, x0 - 1 + c);
  }
  // intensities with the Sobel border rule (replicated edges)
  for (int k = lane; k < (kFT + 2) * (kFT + 2); k += 32) {
    const int r = k / (kFT + 2), c = k - r * (kFT + 2);
    const int yy = min(max(y0 - 1 + r, 0), h - 1), xx = min(max(x0 - 1 + c, 0), w - 1);
    S.I[r][c] = I[(int64_t)yy * w + xx];
  }
  __syncwarp();
  // 2. one object at a time
  uint32_t rem = rowbits;
  const uint32_t yl = (uint32_t)lane;  // tile-local row
  while (true) {
    const unsigned has = __ballot_sync(full, rem != 0);
    if (!has) break;
    const int src = __ffs(has) - 1;
    int32_t pick = 0;
    if (lane == src) pick = S.L[lane + 1][__ffs(rem)];
    const int32_t L = __shfl_sync(full, pick, src);
    uint32_t m = 0;
    for (uint32_t q = rem; q; q &= q - 1) {
      const int c = __ffs(q) - 1;
      if (S.L[lane + 1][c + 1] == L) m |= 1u << c;
    }
    rem &= ~m;
    // masks of L in the rows above / below (tile rows by shuffle, halo rows
    // from shared memory) and left / right of the tile
    uint32_t up = __shfl_up_sync(full, m, 1), dn = __shfl_down_sync(full, m, 1);
    if (lane == 0 || lane == 31) {
      const int hr = lane == 0 ? 0 : kFT + 1;
      uint32_t hm = 0;
      for (int c = 0; c < kFT; ++c) hm |= (S.L[hr][c + 1] == L ? 1u : 0u) << c;
      if (lane == 0) up = hm;
      else dn = hm;
    }
    const uint32_t lb = S.L[lane + 1][0] == L ? 1u : 0u;
    const uint32_t rb = S.L[lane + 1][kFT + 1] == L ? 0x80000000u : 0u;
    const uint32_t n = __popc(m);
    uint32_t per = __popc(m & ~up) + __popc(m & ~dn) + __popc(m & ~((m << 1) | lb)) +
                   __popc(m & ~((m >> 1) | rb));
    uint32_t sx = 0, sxx = 0, si = 0, sii = 0, sg = 0, mni = 0xFFFFFFFFu, mxi = 0;
    unsigned long long sgg = 0;
    for (uint32_t q = m; q; q &= q - 1) {
      const int c = __ffs(q) - 1;
      const uint8_t* r0 = &S.I[lane][c];
      const uint8_t* r1 = &S.I[lane + 1][c];
      const uint8_t* r2 = &S.I[lane + 2][c];
      const int gx = ((int)r0[2] + 2 * (int)r1[2] + (int)r2[2]) -
                     ((int)r0[0] + 2 * (int)r1[0] + (int)r2[0]);
      const int gy = ((int)r2[0] + 2 * (int)r2[1] + (int)r2[2]) -
                     ((int)r0[0] + 2 * (int)r0[1] + (int)r0[2]);
      const uint32_t gq = isqrt_small(16u * (uint32_t)(gx * gx + gy * gy));
      const uint32_t v = r1[1];
      sx += (uint32_t)c;
      sxx += (uint32_t)(c * c);
      si += v;
      sii += v * v;
      sg += gq;
      sgg += (unsigned long long)(gq * gq);
      mni = min(mni, v);
      mxi = max(mxi, v);
    }
    // 3. warp reductions (tile-local coordinates: every u32 sum fits)
    const uint32_t tn = __reduce_add_sync(full, n);
    const uint32_t ty = __reduce_add_sync(full, n * yl);
    const uint32_t tyy = __reduce_add_sync(full, n * yl * yl);
    const uint32_t tx = __reduce_add_sync(full, sx);
    const uint32_t txx = __reduce_add_sync(full, sxx);
    const uint32_t txy = __reduce_add_sync(full, sx * yl);
    const uint32_t ti = __reduce_add_sync(full, si);
    const uint32_t tii = __reduce_add_sync(full, sii);
    const uint32_t tg = __reduce_add_sync(full, sg);
    const uint32_t tp = __reduce_add_sync(full, per);
    unsigned long long tgg = sgg;
#pragma unroll
    for (int off = 16; off; off >>= 1) tgg += __shfl_xor_sync(full, tgg, off);
    const uint32_t tmni = __reduce_min_sync(full, mni);
    const uint32_t tmxi = __reduce_max_sync(full, mxi);
    const uint32_t tminy = __reduce_min_sync(full, m ? yl : 0xFFFFFFFFu);
    const uint32_t tmaxy = __reduce_max_sync(full, m ? yl : 0u);
    const uint32_t tminx = __reduce_min_sync(full, m ? (uint32_t)(__ffs(m) - 1) : 0xFFFFFFFFu);
    const uint32_t tmaxx = __reduce_max_sync(full, m ? (uint32_t)(31 - __clz(m)) : 0u);
    // 4. lane j flushes field j (global coordinates, exact u64 arithmetic)
    const int64_t c = acc.cap, k = L - 1;
    const unsigned long long N = tn, Y = (unsigned long long)y0, X = (unsigned long long)x0;
    unsigned long long* Sm = acc.sums;
    switch (lane) {
      case 0: atomicAdd(&Sm[kSumArea * c + k], N); break;
      case 1: atomicAdd(&Sm[kSumY * c + k], ty + N * Y); break;
      case 2: atomicAdd(&Sm[kSumX * c + k], tx + N * X); break;
      case 3: atomicAdd(&Sm[kSumYY * c + k], tyy + 2 * Y * ty + N * Y * Y); break;
      case 4: atomicAdd(&Sm[kSumXX * c + k], txx + 2 * X * tx + N * X * X); break;
      case 5: atomicAdd(&Sm[kSumXY * c + k], txy + X * ty + Y * tx + N * X * Y); break;
      case 6: atomicAdd(&Sm[kSumI * c + k], (unsigned long long)ti); break;
      case 7: atomicAdd(&Sm[kSumII * c + k], (unsigned long long)tii); break;
      case 8: atomicAdd(&Sm[kSumG * c + k], (unsigned long long)tg); break;
      case 9: atomicAdd(&Sm[kSumGG * c + k], tgg); break;
      case 10: atomicAdd(&Sm[kSumPerim * c + k], (unsigned long long)tp); break;
      case 11: atomicMin(&acc.mins[kMinI * c + k], (int32_t)tmni); break;
      case 12: atomicMin(&acc.mins[kMinY * c + k], y0 + (int32_t)tminy); break;
      case 13: atomicMin(&acc.mins[kMinX * c + k], x0 + (int32_t)tminx); break;
      case 14: atomicMax(&acc.maxs[kMaxI * c + k], (int32_t)tmxi); break;
      case 15: atomicMax(&acc.maxs[kMaxY * c + k], y0 + (int32_t)tmaxy); break;
      case 16: atomicMax(&acc.maxs[kMaxX * c + k], x0 + (int32_t)tmaxx); break;
      default: break;
    }
  }
}

// Step 2: one thread per object.  Expression order mirrors the oracle
// (oracle/rtg_oracle.c orc_features) term by term.
__global__ void k_feat_finalize(const int32_t* __restrict__ d_n, FeatureAcc acc,
                                float* __restrict__ out, uint32_t* __restrict__ status) {
  pdl_enter();
  const int n_all = *d_n;
  if (n_all > acc.cap && blockIdx.x == 0 && threadIdx.x == 0)
    atomicOr(status, kStatusObjectOverflow);
  const int n = min(n_all, acc.cap);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int64_t c = acc.cap;
    const unsigned long long* S = acc.sums;
    float* f = out + (int64_t)k * RTG_NUM_FEATURES;
    const unsigned long long area = S[kSumArea * c + k];
    if (area == 0) {
      for (int j = 0; j < RTG_NUM_FEATURES; ++j) f[j] = 0.f;
      continue;
    }
    const double A = (double)area;
    const double cy = (double)(long long)S[kSumY * c + k] / A;
    const double cx = (double)(long long)S[kSumX * c + k] / A;
    const double mi = (double)(long long)S[kSumI * c + k] / A;
    const double vi = (double)(long long)S[kSumII * c + k] / A - mi * mi;
    const double mg = (double)(long long)S[kSumG * c + k] / (4.0 * A);
    const double vg = (double)(long long)S[kSumGG * c + k] / (16.0 * A) - mg * mg;
    const double mxx = (double)(long long)S[kSumXX * c + k] / A - cx * cx + 1.0 / 12.0;
    const double myy = (double)(long long)S[kSumYY * c + k] / A - cy * cy + 1.0 / 12.0;
    const double mxy = (double)(long long)S[kSumXY * c + k] / A - cx * cy;
    const double half = 0.5 * (mxx + myy);
    const double dd = 0.5 * (mxx - myy);
    const double root = sqrt(dd * dd + mxy * mxy);
    const double l1 = half + root;
    double l2 = half - root;
    if (l2 < 0.0) l2 = 0.0;
    const double P = (double)(long long)S[kSumPerim * c + k];
    const int32_t y0 = acc.mins[kMinY * c + k], x0 = acc.mins[kMinX * c + k];
    const int32_t y1 = acc.maxs[kMaxY * c + k], x1 = acc.maxs[kMaxX * c + k];
    f[RTG_F_AREA] = (float)A;
    f[RTG_F_PERIMETER] = (float)P;
    f[RTG_F_BBOX_Y0] = (float)y0;
    f[RTG_F_BBOX_X0] = (float)x0;
    f[RTG_F_BBOX_Y1] = (float)y1;
    f[RTG_F_BBOX_X1] = (float)x1;
    f[RTG_F_CENTROID_Y] = (float)cy;
    f[RTG_F_CENTROID_X] = (float)cx;
    f[RTG_F_MEAN_I] = (float)mi;
    f[RTG_F_STD_I] = (float)sqrt(vi > 0.0 ? vi : 0.0);
    f[RTG_F_MIN_I] = (float)acc.mins[kMinI * c + k];
    f[RTG_F_MAX_I] = (float)acc.maxs[kMaxI * c + k];
    f[RTG_F_MEAN_GRAD] = (float)mg;
    f[RTG_F_STD_GRAD] = (float)sqrt(vg > 0.0 ? vg : 0.0);
    f[RTG_F_MAJOR_AXIS] = (float)(4.0 * sqrt(l1));
    f[RTG_F_MINOR_AXIS] = (float)(4.0 * sqrt(l2));
    f[RTG_F_ECCENTRICITY] = (float)(l1 > 0.0 ? sqrt(1.0 - l2 / l1) : 0.0);
    f[RTG_F_ORIENTATION] = (float)(0.5 * atan2(2.0 * mxy, mxx - myy));
    f[RTG_F_CIRCULARITY] = (float)(4.0 * 3.14159265358979323846 * A / (P * P));
    f[RTG_F_EXTENT] = (float)(A / ((double)(y1 - y0 + 1) * (double)(x1 - x0 + 1)));
  }
}

}  // namespace

int features(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity,
             int64_t h, int64_t w, const int32_t* d_n, float* out, const int32_t* list,
             const int32_t* list_count, bool acc_cleared) {
  const int cap = ctx->acc.cap;
  const int gclear = (int)ceil_div(cap, 256);
  if (!acc_cleared) {
    RTG_CUDA(launch_k(ctx, k_feat_clear, gclear, 256, 0, d_n, ctx->acc));
    RTG_LAUNCH("k_feat_clear");
  }
  if (ctx->feat_impl == 0) {
    const int tiles_x = (int)ceil_div(w, kFT), ntiles = tiles_x * (int)ceil_div(h, kFT);
    RTG_CUDA(launch_k(ctx, k_feat_tiles, (unsigned)ceil_div(ntiles, 4), 128, 0, labels, intensity,
                      (int)h, (int)w, tiles_x, ntiles, d_n, ctx->acc));
    RTG_LAUNCH("k_feat_tiles");
  } else if (list && h <= 4096 && w <= 4096) {
    // the list kernel reduces global coordinates in 32 bits: tiles up to 4096^2
    RTG_CUDA(launch_k(ctx, k_feat_list, ctx->num_sms * 8, 256, 0, list, list_count, labels, intensity,
                                                           (int)h, make_div((uint32_t)w), d_n,
                                                           ctx->acc));
    RTG_LAUNCH("k_feat_list");
  } else {
    const dim3 grid((unsigned)ceil_div(w, kFB), (unsigned)ceil_div(h, kFB));
    RTG_CUDA(launch_k(ctx, k_feat_accum, grid, 256, 0, labels, intensity, (int)h, (int)w, d_n,
                                                ctx->acc));
    RTG_LAUNCH("k_feat_accum");
  }
  RTG_CUDA(launch_k(ctx, k_feat_finalize, gclear, 256, 0, d_n, ctx->acc, out, ctx->status));
  RTG_LAUNCH("k_feat_finalize");
  return RTG_OK;
}

}  // namespace rtg
