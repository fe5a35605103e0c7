// o9 per-object features, the paper's two-step scheme:
// step 1 reduces pixels into fixed-size per-object intermediates (moments,
// intensity and gradient sums, perimeter edges, bbox, min/max), step 2 runs
// one thread per object to turn them into the feature row.
//
// Step 1 is a warp-level reduction: each warp covers 32 consecutive pixels,
// groups lanes of equal label with __match_any_sync, reduces every field with
// redux.sync (__reduce_{add,min,max}_sync) and lets one leader lane issue the
// global atomics, so atomics scale with object-runs, not pixels.  All
// intermediates are integers, so step 1 is order-independent and exact; step
// 2 is fp64 with FMA contraction disabled (--fmad=false), matching the oracle.
//
// Roofline: HBM/L2 bound; algorithmic bytes labels 4 B + intensity 1 B per px.
#include "common.cuh"

namespace rtg {
namespace {

__global__ void k_feat_clear(const int32_t* __restrict__ d_n, FeatureAcc acc) {
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

__device__ __forceinline__ uint32_t isqrt32(uint32_t v) {
  uint32_t r = (uint32_t)sqrt((double)v);
  while ((uint64_t)r * r > v) --r;
  while ((uint64_t)(r + 1) * (r + 1) <= v) ++r;
  return r;
}

__global__ void __launch_bounds__(256)
k_feat_accum(const int32_t* __restrict__ labels, const uint8_t* __restrict__ I,
             int h, int w, const int32_t* __restrict__ d_n, FeatureAcc acc) {
  const unsigned full = 0xFFFFFFFFu;
  const int nobj = min(*d_n, acc.cap);
  const int lane = threadIdx.x & 31;
  // 2-D grid-stride (rows x column chunks): a warp covers 32 consecutive
  // pixels of one row, no per-pixel division
  const int wpad = (w + 31) & ~31;
  for (int y = blockIdx.y; y < h; y += gridDim.y)
  for (int xb = blockIdx.x * blockDim.x; xb < wpad; xb += gridDim.x * blockDim.x) {
    const int x = xb + threadIdx.x;
    const int64_t i = (int64_t)y * w + x;
    const int32_t l = x < w ? labels[i] : 0;
    const bool on = l > 0 && l <= nobj;
    const unsigned act = __ballot_sync(full, on);
    if (!act) continue;
    if (!on) continue;
    const int ym = y > 0 ? y - 1 : 0, yp = y + 1 < h ? y + 1 : h - 1;
    const int xm = x > 0 ? x - 1 : 0, xp = x + 1 < w ? x + 1 : w - 1;
    const uint8_t* rm = I + (int64_t)ym * w;
    const uint8_t* r0 = I + (int64_t)y * w;
    const uint8_t* rp = I + (int64_t)yp * w;
    const int gx = ((int)rm[xp] + 2 * (int)r0[xp] + (int)rp[xp]) -
                   ((int)rm[xm] + 2 * (int)r0[xm] + (int)rp[xm]);
    const int gy = ((int)rp[xm] + 2 * (int)rp[x] + (int)rp[xp]) -
                   ((int)rm[xm] + 2 * (int)rm[x] + (int)rm[xp]);
    const uint32_t gq = isqrt32(16u * (uint32_t)(gx * gx + gy * gy));
    const uint32_t v = r0[x];
    uint32_t per = 0;
    per += (y == 0 || labels[i - w] != l);
    per += (y == h - 1 || labels[i + w] != l);
    per += (x == 0 || labels[i - 1] != l);
    per += (x == w - 1 || labels[i + 1] != l);

    const unsigned grp = __match_any_sync(act, l);
    const bool leader = lane == __ffs(grp) - 1;
    const uint32_t uy = (uint32_t)y, ux = (uint32_t)x;
    const uint32_t s_y = __reduce_add_sync(grp, uy);
    const uint32_t s_x = __reduce_add_sync(grp, ux);
    const uint32_t s_yy = __reduce_add_sync(grp, uy * uy);
    const uint32_t s_xx = __reduce_add_sync(grp, ux * ux);
    const uint32_t s_xy = __reduce_add_sync(grp, ux * uy);
    const uint32_t s_i = __reduce_add_sync(grp, v);
    const uint32_t s_ii = __reduce_add_sync(grp, v * v);
    const uint32_t s_g = __reduce_add_sync(grp, gq);
    const uint32_t s_gg = __reduce_add_sync(grp, gq * gq);
    const uint32_t s_p = __reduce_add_sync(grp, per);
    const uint32_t mn_i = __reduce_min_sync(grp, v);
    const uint32_t mx_i = __reduce_max_sync(grp, v);
    const uint32_t mn_y = __reduce_min_sync(grp, uy);
    const uint32_t mx_y = __reduce_max_sync(grp, uy);
    const uint32_t mn_x = __reduce_min_sync(grp, ux);
    const uint32_t mx_x = __reduce_max_sync(grp, ux);
    if (leader) {
      const int64_t k = l - 1;
      const int64_t c = acc.cap;
      unsigned long long* S = acc.sums;
      atomicAdd(&S[kSumArea * c + k], (unsigned long long)__popc(grp));
      atomicAdd(&S[kSumY * c + k], (unsigned long long)s_y);
      atomicAdd(&S[kSumX * c + k], (unsigned long long)s_x);
      atomicAdd(&S[kSumYY * c + k], (unsigned long long)s_yy);
      atomicAdd(&S[kSumXX * c + k], (unsigned long long)s_xx);
      atomicAdd(&S[kSumXY * c + k], (unsigned long long)s_xy);
      atomicAdd(&S[kSumI * c + k], (unsigned long long)s_i);
      atomicAdd(&S[kSumII * c + k], (unsigned long long)s_ii);
      atomicAdd(&S[kSumG * c + k], (unsigned long long)s_g);
      atomicAdd(&S[kSumGG * c + k], (unsigned long long)s_gg);
      atomicAdd(&S[kSumPerim * c + k], (unsigned long long)s_p);
      atomicMin(&acc.mins[kMinI * c + k], (int32_t)mn_i);
      atomicMin(&acc.mins[kMinY * c + k], (int32_t)mn_y);
      atomicMin(&acc.mins[kMinX * c + k], (int32_t)mn_x);
      atomicMax(&acc.maxs[kMaxI * c + k], (int32_t)mx_i);
      atomicMax(&acc.maxs[kMaxY * c + k], (int32_t)mx_y);
      atomicMax(&acc.maxs[kMaxX * c + k], (int32_t)mx_x);
    }
  }
}

// Step 2: one thread per object.  Expression order mirrors the oracle
// (oracle/rtg_oracle.c orc_features) term by term.
__global__ void k_feat_finalize(const int32_t* __restrict__ d_n, FeatureAcc acc,
                                float* __restrict__ out, uint32_t* __restrict__ status) {
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
             int64_t h, int64_t w, const int32_t* d_n, float* out) {
  const int cap = ctx->acc.cap;
  const int gclear = (int)ceil_div(cap, 256);
  k_feat_clear<<<gclear, 256, 0, ctx->stream>>>(d_n, ctx->acc);
  RTG_LAUNCH("k_feat_clear");
  const dim3 grid((unsigned)ceil_div(w, 256), (unsigned)(h < 1024 ? h : 1024));
  k_feat_accum<<<grid, 256, 0, ctx->stream>>>(labels, intensity, (int)h, (int)w, d_n, ctx->acc);
  RTG_LAUNCH("k_feat_accum");
  k_feat_finalize<<<gclear, 256, 0, ctx->stream>>>(d_n, ctx->acc, out, ctx->status);
  RTG_LAUNCH("k_feat_finalize");
  return RTG_OK;
}

}  // namespace rtg
