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
    // hold no head.  Nine fields travel in six shuffles: sum x (< 2^18, x <
    // 8192) with the perimeter count (<= 128), sum I (< 2^13) with sum of
    // gradients (< 2^18), and min I with 255 - max I as two 16-bit halves
    // combined by one 16x2 min; no packed field can carry into its neighbour.
    uint32_t A = (l ? (uint32_t)x : 0u) | (per << 18);
    uint32_t B = v | (gq << 13);
    uint32_t sxx = l ? (uint32_t)x * (uint32_t)x : 0u, sii = v * v, sgg = gq * gq;
    uint32_t M = l ? (v | ((255u - v) << 16)) : 0xFFFFFFFFu;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t oA = __shfl_down_sync(full, A, off);
      const uint32_t oB = __shfl_down_sync(full, B, off);
      const uint32_t oxx = __shfl_down_sync(full, sxx, off);
      const uint32_t oii = __shfl_down_sync(full, sii, off);
      const uint32_t ogg = __shfl_down_sync(full, sgg, off);
      const uint32_t oM = __shfl_down_sync(full, M, off);
      const uint32_t span = ((heads >> 1) >> lane) & ((1u << off) - 1u);  // heads in (lane, lane+off]
      if (lane + off < 32 && span == 0) {
        A += oA;
        B += oB;
        sxx += oxx;
        sii += oii;
        sgg += ogg;
        M = __vminu2(M, oM);  // one VIMNMX.U16x2 (the 8-bit form is emulated)
      }
    }
    const uint32_t sx = A & 0x3FFFFu, sp = A >> 18, si = B & 0x1FFFu, sg = B >> 13;
    const uint32_t mni = M & 0xFFFFu, mxi = 255u - (M >> 16);
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
  // the list kernel reduces global coordinates in 32 bits: tiles up to 4096^2
  if (list && h <= 4096 && w <= 4096) {
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
