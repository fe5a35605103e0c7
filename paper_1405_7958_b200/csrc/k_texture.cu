// f4 texture features: per-nucleus
// "histograms and co-occurrence matrices", in the paper's two steps:
//   1. one warp per object bounding box accumulates the fixed-size integer
//      intermediates in shared memory — 16-bin intensity histogram, Canny
//      edge pixel count, 8x8
//      symmetric grey-level co-occurrence matrix over the offsets (0,1)
//      (1,0) (1,1) (1,-1) for pairs inside the object, and the intensity
//      moments sum v, v^2, v^3, v^4;
//   2. one thread per object turns them into the row (fp64, expression order
//      of oracle/rtg_oracle.c orc_texture_row, --fmad=false).
// Bounding boxes come from a dense min/max pass with warp-aggregated atomics
// (the rtg_texture_features entry points take labels alone).
//
// Roofline: labels 4 B + intensity 1 B per bbox pixel read (L2-resident
// bbox windows); the intermediates are 336 B per object.
#include "common.cuh"

namespace rtg {
namespace {

__global__ void k_tex_clear(const int32_t* __restrict__ d_n, int32_t cap, int32_t* __restrict__ bb,
                            uint32_t* __restrict__ hist, uint32_t* __restrict__ glcm,
                            unsigned long long* __restrict__ mom) {
  const int n = min(*d_n, cap);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    bb[4 * k + 0] = INT32_MAX;
    bb[4 * k + 1] = INT32_MAX;
    bb[4 * k + 2] = -1;
    bb[4 * k + 3] = -1;
  }
  (void)hist;
  (void)glcm;
  (void)mom;
}

// Bounding boxes: each warp covers 32 consecutive pixels of a row; lanes of
// one label are grouped with __match_any_sync and one leader updates.
__global__ void __launch_bounds__(256)
k_tex_bbox(const int32_t* __restrict__ labels, int h, int w, const int32_t* __restrict__ d_n,
           int32_t cap, int32_t* __restrict__ bb) {
  const unsigned full = 0xFFFFFFFFu;
  const int nobj = min(*d_n, cap);
  const int wpad = (w + 31) & ~31;
  for (int y = blockIdx.y; y < h; y += gridDim.y)
    for (int xb = blockIdx.x * blockDim.x; xb < wpad; xb += gridDim.x * blockDim.x) {
      const int x = xb + threadIdx.x;
      const int32_t l = x < w ? labels[(int64_t)y * w + x] : 0;
      const bool on = l > 0 && l <= nobj;
      const unsigned act = __ballot_sync(full, on);
      if (!act || !on) continue;
      const unsigned grp = __match_any_sync(act, l);
      const int xmin = __reduce_min_sync(grp, (unsigned)x), xmax = __reduce_max_sync(grp, (unsigned)x);
      if ((threadIdx.x & 31) != __ffs(grp) - 1) continue;
      int32_t* b = bb + 4 * (l - 1);
      atomicMin(b + 0, y);
      atomicMin(b + 1, xmin);
      atomicMax(b + 2, y);
      atomicMax(b + 3, xmax);
    }
}

// Step 1: one warp per object over its bounding box.
__global__ void __launch_bounds__(256)
k_tex_accum(const int32_t* __restrict__ labels, const uint8_t* __restrict__ I,
            const uint8_t* __restrict__ E, int h, int w,
            const int32_t* __restrict__ d_n, int32_t cap, const int32_t* __restrict__ bb,
            uint32_t* __restrict__ hist_out, uint32_t* __restrict__ glcm_out,
            unsigned long long* __restrict__ mom_out) {
  __shared__ uint32_t s_hist[8][17];  // 16 bins + Canny edge pixels
  __shared__ uint32_t s_glcm[8][64];
  const int nobj = min(*d_n, cap);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* hist = s_hist[wid];
  uint32_t* glcm = s_glcm[wid];
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int k = blockIdx.x * (blockDim.x >> 5) + wid; k < nobj; k += warps) {
    if (lane < 17) hist[lane] = 0;
    glcm[lane] = 0;
    glcm[lane + 32] = 0;
    __syncwarp();
    const int32_t y0 = bb[4 * k], x0 = bb[4 * k + 1], y1 = bb[4 * k + 2], x1 = bb[4 * k + 3];
    const int32_t l = k + 1;
    unsigned long long m1 = 0, m2 = 0, m3 = 0, m4 = 0;
    if (y1 >= 0) {
      for (int y = y0; y <= y1; ++y) {
        const int64_t rb = (int64_t)y * w;
        for (int x = x0 + lane; x <= x1; x += 32) {
          if (labels[rb + x] != l) continue;
          const uint32_t v = I[rb + x];
          atomicAdd(&hist[v >> 4], 1u);
          if (E[rb + x]) atomicAdd(&hist[16], 1u);
          const unsigned long long v2 = (unsigned long long)(v * v);
          m1 += v;
          m2 += v2;
          m3 += v2 * v;
          m4 += v2 * v2;
          const uint32_t q = v >> 5;
          // forward offsets: right, down, down-right, down-left
          if (x + 1 < w && labels[rb + x + 1] == l) {
            const uint32_t q2 = I[rb + x + 1] >> 5;
            atomicAdd(&glcm[q * 8 + q2], 1u);
            atomicAdd(&glcm[q2 * 8 + q], 1u);
          }
          if (y + 1 < h) {
            const int64_t nb = rb + w;
            if (labels[nb + x] == l) {
              const uint32_t q2 = I[nb + x] >> 5;
              atomicAdd(&glcm[q * 8 + q2], 1u);
              atomicAdd(&glcm[q2 * 8 + q], 1u);
            }
            if (x + 1 < w && labels[nb + x + 1] == l) {
              const uint32_t q2 = I[nb + x + 1] >> 5;
              atomicAdd(&glcm[q * 8 + q2], 1u);
              atomicAdd(&glcm[q2 * 8 + q], 1u);
            }
            if (x > 0 && labels[nb + x - 1] == l) {
              const uint32_t q2 = I[nb + x - 1] >> 5;
              atomicAdd(&glcm[q * 8 + q2], 1u);
              atomicAdd(&glcm[q2 * 8 + q], 1u);
            }
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m1 += __shfl_xor_sync(0xFFFFFFFFu, m1, o);
      m2 += __shfl_xor_sync(0xFFFFFFFFu, m2, o);
      m3 += __shfl_xor_sync(0xFFFFFFFFu, m3, o);
      m4 += __shfl_xor_sync(0xFFFFFFFFu, m4, o);
    }
    __syncwarp();
    if (lane < 17) hist_out[(int64_t)k * 17 + lane] = hist[lane];
    glcm_out[(int64_t)k * 64 + lane] = glcm[lane];
    glcm_out[(int64_t)k * 64 + lane + 32] = glcm[lane + 32];
    if (lane == 0) {
      mom_out[4 * (int64_t)k + 0] = m1;
      mom_out[4 * (int64_t)k + 1] = m2;
      mom_out[4 * (int64_t)k + 2] = m3;
      mom_out[4 * (int64_t)k + 3] = m4;
    }
    __syncwarp();
  }
}

// Step 2: one thread per object; term order of orc_texture_row.
__global__ void k_tex_finalize(const int32_t* __restrict__ d_n, int32_t cap,
                               const uint32_t* __restrict__ hist_in,
                               const uint32_t* __restrict__ glcm_in,
                               const unsigned long long* __restrict__ mom_in,
                               float* __restrict__ out) {
  const int n = min(*d_n, cap);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t* hist = hist_in + (int64_t)k * 17;
    const uint32_t* glcm = glcm_in + (int64_t)k * 64;
    const unsigned long long* mom = mom_in + 4 * (int64_t)k;
    float* o = out + (int64_t)k * RTG_NUM_TEXTURE;
    for (int j = 0; j < RTG_NUM_TEXTURE; ++j) o[j] = 0.f;
    long long nn = 0;
    for (int b = 0; b < 16; ++b) nn += hist[b];
    if (nn == 0) continue;
    const double N = (double)nn;
    double hent = 0.0, hen = 0.0;
    for (int b = 0; b < 16; ++b) {
      if (!hist[b]) continue;
      const double p = (double)hist[b] / N;
      hent -= p * log2(p);
      hen += p * p;
    }
    const double mu = (double)(long long)mom[0] / N, e2 = (double)(long long)mom[1] / N;
    const double e3 = (double)(long long)mom[2] / N, e4 = (double)(long long)mom[3] / N;
    const double var = e2 - mu * mu;
    double skew = 0.0, kurt = 0.0;
    if (var > 0.0) {
      const double sd = sqrt(var);
      skew = (e3 - 3.0 * mu * e2 + 2.0 * mu * mu * mu) / (var * sd);
      kurt = (e4 - 4.0 * mu * e3 + 6.0 * mu * mu * e2 - 3.0 * mu * mu * mu * mu) / (var * var) - 3.0;
    }
    o[RTG_T_HIST_ENTROPY] = (float)hent;
    o[RTG_T_HIST_ENERGY] = (float)hen;
    o[RTG_T_SKEWNESS] = (float)skew;
    o[RTG_T_KURTOSIS] = (float)kurt;
    o[RTG_T_EDGE_PIXELS] = (float)hist[16];
    o[RTG_T_EDGE_DENSITY] = (float)((double)hist[16] / N);
    long long tt = 0;
    for (int j = 0; j < 64; ++j) tt += glcm[j];
    if (tt == 0) continue;
    const double T = (double)tt;
    double asm_ = 0.0, con = 0.0, hom = 0.0, ent = 0.0, mui = 0.0, dis = 0.0, mx = 0.0;
    for (int i = 0; i < 8; ++i) {
      for (int j = 0; j < 8; ++j) {
        const uint32_t c = glcm[i * 8 + j];
        if (!c) continue;
        const double P = (double)c / T;
        const int d = i - j;
        asm_ += P * P;
        con += (double)(d * d) * P;
        hom += P / (1.0 + (double)(d * d));
        ent -= P * log2(P);
        mui += (double)i * P;
        dis += (double)(d < 0 ? -d : d) * P;
        if (P > mx) mx = P;
      }
    }
    double vari = 0.0, sij = 0.0, shade = 0.0;
    for (int i = 0; i < 8; ++i) {
      for (int j = 0; j < 8; ++j) {
        const uint32_t c = glcm[i * 8 + j];
        if (!c) continue;
        const double P = (double)c / T;
        const double di = (double)i - mui;
        const double t = (double)(i + j) - 2.0 * mui;
        vari += di * di * P;
        sij += (double)(i * j) * P;
        shade += t * t * t * P;
      }
    }
    o[RTG_T_GLCM_ASM] = (float)asm_;
    o[RTG_T_GLCM_CONTRAST] = (float)con;
    o[RTG_T_GLCM_HOMOGENEITY] = (float)hom;
    o[RTG_T_GLCM_ENTROPY] = (float)ent;
    o[RTG_T_GLCM_CORRELATION] = (float)(vari > 0.0 ? (sij - mui * mui) / vari : 0.0);
    o[RTG_T_GLCM_DISSIMILARITY] = (float)dis;
    o[RTG_T_GLCM_MAX_PROB] = (float)mx;
    o[RTG_T_GLCM_CLUSTER_SHADE] = (float)shade;
  }
}

// ---- Canny (rtg.h rtg_canny_dev) ------------------------------------------------
// One CTA per 32x32 tile: the intensity tile + a 4-pixel halo (clamped: the
// replicate border) is staged, smoothed (5x5 binomial) on the tile + 2 ring,
// Sobel magnitudes are taken on the tile + 1 ring (smoothed values at
// clamped coordinates; magnitudes outside the image are 0), and each tile
// pixel is classified after non-maximum suppression: 0 none, 1 weak, 2 strong.
// Hysteresis is the threshold decomposition again (components of {class >=
// 1} holding a class-2 pixel), on the CCL.
__global__ void __launch_bounds__(256)
k_canny_nms(const uint8_t* __restrict__ I, int h, int w, int32_t lo2, int32_t hi2,
            uint8_t* __restrict__ cls) {
  __shared__ uint8_t sI[40][41];
  __shared__ uint8_t sS[36][37];
  __shared__ int32_t sM[34][34];
  __shared__ int32_t sG[34][34];  // gx (high 16) | gy (low 16), tile + 1 ring
  const int y0 = blockIdx.y * 32, x0 = blockIdx.x * 32;
  const int tid = threadIdx.x;
  for (int k = tid; k < 40 * 40; k += 256) {
    const int yy = k / 40, xx = k - yy * 40;
    const int y = min(max(y0 - 4 + yy, 0), h - 1), x = min(max(x0 - 4 + xx, 0), w - 1);
    sI[yy][xx] = I[(int64_t)y * w + x];
  }
  __syncthreads();
  const int K[5] = {1, 4, 6, 4, 1};
  for (int k = tid; k < 36 * 36; k += 256) {
    const int yy = k / 36, xx = k - yy * 36;  // global (y0 - 2 + yy, x0 - 2 + xx)
    int32_t acc = 0;
#pragma unroll
    for (int dy = 0; dy < 5; ++dy)
#pragma unroll
      for (int dx = 0; dx < 5; ++dx) acc += K[dy] * K[dx] * sI[yy + dy][xx + dx];
    sS[yy][xx] = (uint8_t)((acc + 128) >> 8);
  }
  __syncthreads();
  // smoothed value at a clamped global position (inside the staged window)
  auto S = [&](int y, int x) -> int32_t {
    y = min(max(y, 0), h - 1);
    x = min(max(x, 0), w - 1);
    return sS[y - (y0 - 2)][x - (x0 - 2)];
  };
  for (int k = tid; k < 34 * 34; k += 256) {
    const int yy = k / 34, xx = k - yy * 34;
    const int y = y0 - 1 + yy, x = x0 - 1 + xx;
    int32_t m = 0, g = 0;
    if (y >= 0 && y < h && x >= 0 && x < w) {
      const int32_t gx = (S(y - 1, x + 1) + 2 * S(y, x + 1) + S(y + 1, x + 1)) -
                         (S(y - 1, x - 1) + 2 * S(y, x - 1) + S(y + 1, x - 1));
      const int32_t gy = (S(y + 1, x - 1) + 2 * S(y + 1, x) + S(y + 1, x + 1)) -
                         (S(y - 1, x - 1) + 2 * S(y - 1, x) + S(y - 1, x + 1));
      m = gx * gx + gy * gy;
      g = (int32_t)((uint32_t)(gx & 0xFFFF) << 16 | (uint32_t)(gy & 0xFFFF));
    }
    sM[yy][xx] = m;
    sG[yy][xx] = g;
  }
  __syncthreads();
  for (int k = tid; k < 32 * 32; k += 256) {
    const int r = k >> 5, c = k & 31;
    const int y = y0 + r, x = x0 + c;
    if (y >= h || x >= w) continue;
    const int32_t m = sM[r + 1][c + 1];
    const int32_t g = sG[r + 1][c + 1];
    const int32_t gx = (int32_t)(int16_t)(g >> 16), gy = (int32_t)(int16_t)(g & 0xFFFF);
    const int64_t ax = gx < 0 ? -gx : gx, ay = gy < 0 ? -gy : gy;
    const int64_t t22 = ax * 13573, ay15 = ay << 15;  // tan(22.5 deg) * 2^15
    int da_y, da_x;  // offset of the "previous" neighbour; the next one is its mirror
    if (ay15 < t22) { da_y = 0; da_x = -1; }
    else if (ay15 > t22 + (ax << 16)) { da_y = -1; da_x = 0; }
    else { const int s = ((gx ^ gy) < 0) ? -1 : 1; da_y = -1; da_x = -s; }
    const int32_t ma = sM[r + 1 + da_y][c + 1 + da_x], mb = sM[r + 1 - da_y][c + 1 - da_x];
    uint8_t out = 0;
    if (m > ma && m >= mb) out = m > hi2 ? 2 : (m > lo2 ? 1 : 0);
    cls[(int64_t)y * w + x] = out;
  }
}

}  // namespace

int canny(rtg_ctx* ctx, const uint8_t* intensity, int64_t h, int64_t w, int32_t low, int32_t high,
          uint8_t* edges) {
  uint8_t* cls = ctx->m1 == edges ? ctx->m2 : ctx->m1;
  const dim3 tiles((unsigned)ceil_div(w, 32), (unsigned)ceil_div(h, 32));
  k_canny_nms<<<tiles, 256, 0, ctx->stream>>>(intensity, (int)h, (int)w, low * low, high * high,
                                              cls);
  RTG_LAUNCH("k_canny_nms");
  // hysteresis: weak (1) pixels 8-connected to a strong (2) one
  return recon_threshold_uf(ctx, cls, cls, h, w, 1, 1, 8, nullptr, edges);
}

int texture(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity, int64_t h, int64_t w,
            const int32_t* d_n, float* out) {
  uint8_t* edges = ctx->m3;
  RTG_TRY(canny(ctx, intensity, h, w, RTG_CANNY_LOW, RTG_CANNY_HIGH, edges));
  const int32_t cap = ctx->max_objects;
  const int g = (int)ceil_div(cap, 256);
  k_tex_clear<<<g, 256, 0, ctx->stream>>>(d_n, cap, ctx->tex_bbox, ctx->tex_hist, ctx->tex_glcm,
                                          ctx->tex_mom);
  RTG_LAUNCH("k_tex_clear");
  const dim3 gb((unsigned)ceil_div(w, 256), (unsigned)(h < 1024 ? h : 1024));
  k_tex_bbox<<<gb, 256, 0, ctx->stream>>>(labels, (int)h, (int)w, d_n, cap, ctx->tex_bbox);
  RTG_LAUNCH("k_tex_bbox");
  k_tex_accum<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(labels, intensity, edges, (int)h,
                                                         (int)w, d_n, cap, ctx->tex_bbox,
                                                         ctx->tex_hist, ctx->tex_glcm,
                                                         ctx->tex_mom);
  RTG_LAUNCH("k_tex_accum");
  k_tex_finalize<<<g, 256, 0, ctx->stream>>>(d_n, cap, ctx->tex_hist, ctx->tex_glcm, ctx->tex_mom,
                                             out);
  RTG_LAUNCH("k_tex_finalize");
  return RTG_OK;
}

}  // namespace rtg
