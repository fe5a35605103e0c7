// f4 texture features: per-nucleus
// "histograms and co-occurrence matrices", in the paper's two steps:
//   1. one warp per object bounding box accumulates the fixed-size integer
//      intermediates in shared memory — 16-bin intensity histogram, 8x8
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
k_tex_accum(const int32_t* __restrict__ labels, const uint8_t* __restrict__ I, int h, int w,
            const int32_t* __restrict__ d_n, int32_t cap, const int32_t* __restrict__ bb,
            uint32_t* __restrict__ hist_out, uint32_t* __restrict__ glcm_out,
            unsigned long long* __restrict__ mom_out) {
  __shared__ uint32_t s_hist[8][16];
  __shared__ uint32_t s_glcm[8][64];
  const int nobj = min(*d_n, cap);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* hist = s_hist[wid];
  uint32_t* glcm = s_glcm[wid];
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int k = blockIdx.x * (blockDim.x >> 5) + wid; k < nobj; k += warps) {
    if (lane < 16) hist[lane] = 0;
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
    if (lane < 16) hist_out[(int64_t)k * 16 + lane] = hist[lane];
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
    const uint32_t* hist = hist_in + (int64_t)k * 16;
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

}  // namespace

int texture(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity, int64_t h, int64_t w,
            const int32_t* d_n, float* out) {
  const int32_t cap = ctx->max_objects;
  const int g = (int)ceil_div(cap, 256);
  k_tex_clear<<<g, 256, 0, ctx->stream>>>(d_n, cap, ctx->tex_bbox, ctx->tex_hist, ctx->tex_glcm,
                                          ctx->tex_mom);
  RTG_LAUNCH("k_tex_clear");
  const dim3 gb((unsigned)ceil_div(w, 256), (unsigned)(h < 1024 ? h : 1024));
  k_tex_bbox<<<gb, 256, 0, ctx->stream>>>(labels, (int)h, (int)w, d_n, cap, ctx->tex_bbox);
  RTG_LAUNCH("k_tex_bbox");
  k_tex_accum<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(labels, intensity, (int)h, (int)w, d_n,
                                                         cap, ctx->tex_bbox, ctx->tex_hist,
                                                         ctx->tex_glcm, ctx->tex_mom);
  RTG_LAUNCH("k_tex_accum");
  k_tex_finalize<<<g, 256, 0, ctx->stream>>>(d_n, cap, ctx->tex_hist, ctx->tex_glcm, ctx->tex_mom,
                                             out);
  RTG_LAUNCH("k_tex_finalize");
  return RTG_OK;
}

}  // namespace rtg
