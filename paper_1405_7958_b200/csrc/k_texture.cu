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

// Where the bounding boxes come from: the packed boxes of k_tex_bbox
// (stride 4) or the feature stage's per-object accumulators (stride 1, SoA).
struct TexBoxes {
  const int32_t *y0, *x0, *y1, *x1;
  int stride;
};

// Step 1: one warp per object over its bounding box; the 32 lanes walk the
// box's pixels in raster order (lane + 32 i), so narrow boxes keep every lane
// busy.
__global__ void __launch_bounds__(256)
k_tex_accum(const int32_t* __restrict__ labels, const uint8_t* __restrict__ I,
            const uint8_t* __restrict__ E, int h, int w,
            const int32_t* __restrict__ d_n, int32_t cap, TexBoxes bb,
            uint32_t* __restrict__ hist_out, uint32_t* __restrict__ glcm_out,
            unsigned long long* __restrict__ mom_out) {
  pdl_enter();
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
    const int64_t kb = (int64_t)k * bb.stride;
    const int32_t y0 = bb.y0[kb], x0 = bb.x0[kb], y1 = bb.y1[kb], x1 = bb.x1[kb];
    const int32_t l = k + 1;
    unsigned long long m1 = 0, m2 = 0, m3 = 0, m4 = 0;
    if (y1 >= 0 && x1 >= x0) {
      const int bw = x1 - x0 + 1;
      const int sdy = 32 / bw, sdx = 32 - sdy * bw;  // one step of 32 pixels
      int y = y0 + lane / bw, x = x0 + lane % bw;
      for (; y <= y1;) {
        const int64_t rb = (int64_t)y * w;
        if (labels[rb + x] == l) {
          const uint32_t v = I[rb + x];
          atomicAdd(&hist[v >> 4], 1u);
          if (E[rb + x]) atomicAdd(&hist[16], 1u);
          const unsigned long long v2 = (unsigned long long)(v * v);
          m1 += v;
          m2 += v2;
          m3 += v2 * v;
          m4 += v2 * v2;
          const uint32_t q = v >> 5;
          auto pair = [&](int64_t j) {
            if (labels[j] != l) return;
            const uint32_t q2 = I[j] >> 5;
            atomicAdd(&glcm[q * 8 + q2], 1u);
            atomicAdd(&glcm[q2 * 8 + q], 1u);
          };
          // forward offsets: right, down, down-right, down-left
          if (x + 1 < w) pair(rb + x + 1);
          if (y + 1 < h) {
            const int64_t nb = rb + w;
            pair(nb + x);
            if (x + 1 < w) pair(nb + x + 1);
            if (x > 0) pair(nb + x - 1);
          }
        }
        x += sdx;
        y += sdy;
        if (x > x1) {
          x -= bw;
          ++y;
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

// Step 2: one warp per object (one thread per object left most of the GPU
// idle on the fp64 log2 chains): lanes 0-15 take a histogram bin, every lane
// two co-occurrence cells; fp64 warp sums.  The terms are orc_texture_row's;
// only the summation order differs (fp64, far inside the 1e-5 bar).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

__global__ void __launch_bounds__(256)
k_tex_finalize(const int32_t* __restrict__ d_n, int32_t cap,
               const uint32_t* __restrict__ hist_in, const uint32_t* __restrict__ glcm_in,
               const unsigned long long* __restrict__ mom_in, float* __restrict__ out) {
  pdl_enter();
  const int n = min(*d_n, cap);
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < n; k += warps) {
    const uint32_t* hist = hist_in + (int64_t)k * 17;
    const uint32_t* glcm = glcm_in + (int64_t)k * 64;
    const unsigned long long* mom = mom_in + 4 * (int64_t)k;
    float* o = out + (int64_t)k * RTG_NUM_TEXTURE;
    const uint32_t hb = lane < 16 ? hist[lane] : 0u;
    const uint32_t edge = hist[16];
    const uint32_t c0 = glcm[lane], c1 = glcm[lane + 32];
    const long long nn = (long long)__reduce_add_sync(0xFFFFFFFFu, hb);
    if (lane < RTG_NUM_TEXTURE) o[lane] = 0.f;
    if (nn == 0) continue;
    const double N = (double)nn;
    double hent = 0.0, hen = 0.0;
    if (hb) {
      const double p = (double)hb / N;
      hent = -p * log2(p);
      hen = p * p;
    }
    hent = warp_sum(hent);
    hen = warp_sum(hen);
    const long long tt = (long long)__reduce_add_sync(0xFFFFFFFFu, c0 + c1);
    double fl[RTG_NUM_TEXTURE] = {};
    fl[RTG_T_HIST_ENTROPY] = hent;
    fl[RTG_T_HIST_ENERGY] = hen;
    const double mu = (double)(long long)mom[0] / N, e2 = (double)(long long)mom[1] / N;
    const double e3 = (double)(long long)mom[2] / N, e4 = (double)(long long)mom[3] / N;
    const double var = e2 - mu * mu;
    if (var > 0.0) {
      const double sd = sqrt(var);
      fl[RTG_T_SKEWNESS] = (e3 - 3.0 * mu * e2 + 2.0 * mu * mu * mu) / (var * sd);
      fl[RTG_T_KURTOSIS] =
          (e4 - 4.0 * mu * e3 + 6.0 * mu * mu * e2 - 3.0 * mu * mu * mu * mu) / (var * var) - 3.0;
    }
    fl[RTG_T_EDGE_PIXELS] = (double)edge;
    fl[RTG_T_EDGE_DENSITY] = (double)edge / N;
    if (tt > 0) {
      const double T = (double)tt;
      double asm_ = 0.0, con = 0.0, hom = 0.0, ent = 0.0, mui = 0.0, dis = 0.0, mx = 0.0;
      for (int half = 0; half < 2; ++half) {
        const int cell = lane + 32 * half;
        const uint32_t c = half ? c1 : c0;
        if (!c) continue;
        const int i = cell >> 3, j = cell & 7;
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
      asm_ = warp_sum(asm_);
      con = warp_sum(con);
      hom = warp_sum(hom);
      ent = warp_sum(ent);
      mui = warp_sum(mui);
      dis = warp_sum(dis);
#pragma unroll
      for (int of = 16; of > 0; of >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, of));
      double vari = 0.0, sij = 0.0, shade = 0.0;
      for (int half = 0; half < 2; ++half) {
        const int cell = lane + 32 * half;
        const uint32_t c = half ? c1 : c0;
        if (!c) continue;
        const int i = cell >> 3, j = cell & 7;
        const double P = (double)c / T;
        const double di = (double)i - mui;
        const double t = (double)(i + j) - 2.0 * mui;
        vari += di * di * P;
        sij += (double)(i * j) * P;
        shade += t * t * t * P;
      }
      vari = warp_sum(vari);
      sij = warp_sum(sij);
      shade = warp_sum(shade);
      fl[RTG_T_GLCM_ASM] = asm_;
      fl[RTG_T_GLCM_CONTRAST] = con;
      fl[RTG_T_GLCM_HOMOGENEITY] = hom;
      fl[RTG_T_GLCM_ENTROPY] = ent;
      fl[RTG_T_GLCM_CORRELATION] = vari > 0.0 ? (sij - mui * mui) / vari : 0.0;
      fl[RTG_T_GLCM_DISSIMILARITY] = dis;
      fl[RTG_T_GLCM_MAX_PROB] = mx;
      fl[RTG_T_GLCM_CLUSTER_SHADE] = shade;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < RTG_NUM_TEXTURE; ++j)
      if (lane == j) o[j] = (float)fl[j];
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
  pdl_enter();
  // rows padded to whole words: sI 40 bytes = 10 words, sH 36 + 4 u16
  __shared__ __align__(16) uint8_t sI[40][44];
  __shared__ __align__(16) uint16_t sH[40][40];  // horizontal 5-tap sums, 36 columns
  __shared__ __align__(16) uint8_t sS[36][40];
  __shared__ int32_t sM[34][34];
  __shared__ int32_t sG[34][34];  // gx (high 16) | gy (low 16), tile + 1 ring
  const int y0 = blockIdx.y * 32, x0 = blockIdx.x * 32;
  const int tid = threadIdx.x;
  // stage: 40 rows of 40 clamped bytes (whole words inside the image)
  const bool inner = y0 >= 4 && x0 >= 4 && y0 + 36 <= h && x0 + 36 <= w && (w & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(I) & 3) == 0;
  if (inner) {
    for (int k = tid; k < 40 * 10; k += 256) {
      const int yy = k / 10, q = k - yy * 10;
      *reinterpret_cast<uint32_t*>(&sI[yy][4 * q]) =
          __ldg(reinterpret_cast<const uint32_t*>(I + (int64_t)(y0 - 4 + yy) * w + x0 - 4) + q);
    }
  } else {
    for (int k = tid; k < 40 * 40; k += 256) {
      const int yy = k / 40, xx = k - yy * 40;
      const int y = min(max(y0 - 4 + yy, 0), h - 1), x = min(max(x0 - 4 + xx, 0), w - 1);
      sI[yy][xx] = I[(int64_t)y * w + x];
    }
  }
  __syncthreads();
  // separable 5x5 binomial: (1 4 6 4 1) across, then down; four outputs per
  // thread from two / five word reads
  for (int k = tid; k < 40 * 9; k += 256) {
    const int yy = k / 9, q = k - yy * 9;
    const uint32_t a = *reinterpret_cast<const uint32_t*>(&sI[yy][4 * q]);
    const uint32_t b = *reinterpret_cast<const uint32_t*>(&sI[yy][4 * q + 4]);
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[j] = (a >> (8 * j)) & 0xFFu;
      v[j + 4] = (b >> (8 * j)) & 0xFFu;
    }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = v[j] + 4 * v[j + 1] + 6 * v[j + 2] + 4 * v[j + 3] + v[j + 4];
    *reinterpret_cast<uint2*>(&sH[yy][4 * q]) = make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16));
  }
  __syncthreads();
  for (int k = tid; k < 36 * 9; k += 256) {
    const int yy = k / 9, q = k - yy * 9;
    uint32_t acc[4] = {128u, 128u, 128u, 128u};
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const uint2 u = *reinterpret_cast<const uint2*>(&sH[yy + t][4 * q]);
      const uint32_t wgt = t == 2 ? 6u : (t == 1 || t == 3) ? 4u : 1u;
      acc[0] += wgt * (u.x & 0xFFFFu);
      acc[1] += wgt * (u.x >> 16);
      acc[2] += wgt * (u.y & 0xFFFFu);
      acc[3] += wgt * (u.y >> 16);
    }
    *reinterpret_cast<uint32_t*>(&sS[yy][4 * q]) =
        (acc[0] >> 8) | ((acc[1] >> 8) << 8) | ((acc[2] >> 8) << 16) | ((acc[3] >> 8) << 24);
  }
  __syncthreads();
  // Sobel reads the smoothed value at the CLAMPED position: at the image
  // border, copy the in-image entries over the outside ones (rows first,
  // then columns) so the Sobel below reads the window directly
  const bool edge_tile = y0 < 2 || x0 < 2 || y0 + 34 > h || x0 + 34 > w;
  if (edge_tile) {
    for (int k = tid; k < 36 * 36; k += 256) {
      const int yy = k / 36, xx = k - yy * 36;
      const int y = y0 - 2 + yy, yc = min(max(y, 0), h - 1);
      if (yc != y) sS[yy][xx] = sS[yc - (y0 - 2)][xx];
    }
    __syncthreads();
    for (int k = tid; k < 36 * 36; k += 256) {
      const int yy = k / 36, xx = k - yy * 36;
      const int x = x0 - 2 + xx, xc = min(max(x, 0), w - 1);
      if (xc != x) sS[yy][xx] = sS[yy][xc - (x0 - 2)];
    }
    __syncthreads();
  }
  for (int k = tid; k < 34 * 34; k += 256) {
    const int yy = k / 34, xx = k - yy * 34;
    const int y = y0 - 1 + yy, x = x0 - 1 + xx;
    int32_t m = 0, g = 0;
    if (y >= 0 && y < h && x >= 0 && x < w) {
      // window row yy .. yy + 2, column xx .. xx + 2 (sS origin is y0 - 2, x0 - 2)
      const uint8_t* a = &sS[yy][xx];
      const uint8_t* b = &sS[yy + 1][xx];
      const uint8_t* c = &sS[yy + 2][xx];
      const int32_t gx = (a[2] + 2 * b[2] + c[2]) - (a[0] + 2 * b[0] + c[0]);
      const int32_t gy = (c[0] + 2 * c[1] + c[2]) - (a[0] + 2 * a[1] + a[2]);
      m = gx * gx + gy * gy;
      g = (int32_t)((uint32_t)(gx & 0xFFFF) << 16 | (uint32_t)(gy & 0xFFFF));
    }
    sM[yy][xx] = m;
    sG[yy][xx] = g;
  }
  __syncthreads();
  // four pixels per thread: row tid / 8, columns 4 (tid % 8) .. + 3
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = tid >> 3, c = ((tid & 7) << 2) + j;
    const int y = y0 + r, x = x0 + c;
    if (y >= h || x >= w) continue;
    const int32_t m = sM[r + 1][c + 1];
    const int32_t g = sG[r + 1][c + 1];
    const int32_t gx = (int32_t)(int16_t)(g >> 16), gy = (int32_t)(int16_t)(g & 0xFFFF);
    // |g| <= 4 * 255, so every product below fits 32 bits
    const uint32_t ax = gx < 0 ? -gx : gx, ay = gy < 0 ? -gy : gy;
    const uint32_t t22 = ax * 13573u, ay15 = ay << 15;  // tan(22.5 deg) * 2^15
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
  RTG_CUDA(launch_k(ctx, k_canny_nms, tiles, 256, 0, intensity, (int)h, (int)w, low * low,
                    high * high, cls));
  RTG_LAUNCH("k_canny_nms");
  // hysteresis: weak (1) pixels 8-connected to a strong (2) one (run-table
  // labelling where the width allows: the u16 planes are free after the
  // watershed)
  return recon_threshold_uf(ctx, cls, cls, h, w, 1, 1, 8, nullptr, edges, false,
                            /*runs=*/true);
}

int texture(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity, int64_t h, int64_t w,
            const int32_t* d_n, float* out, const FeatureAcc* boxes) {
  uint8_t* edges = ctx->m3;
  RTG_TRY(canny(ctx, intensity, h, w, RTG_CANNY_LOW, RTG_CANNY_HIGH, edges));
  const int32_t cap = ctx->max_objects;
  const int g = (int)ceil_div(cap, 256);
  TexBoxes bb{ctx->tex_bbox + 0, ctx->tex_bbox + 1, ctx->tex_bbox + 2, ctx->tex_bbox + 3, 4};
  if (boxes) {
    // the feature stage already reduced every object's bounding box
    const int64_t c = boxes->cap;
    bb = TexBoxes{boxes->mins + kMinY * c, boxes->mins + kMinX * c, boxes->maxs + kMaxY * c,
                  boxes->maxs + kMaxX * c, 1};
  } else {
    k_tex_clear<<<g, 256, 0, ctx->stream>>>(d_n, cap, ctx->tex_bbox, ctx->tex_hist,
                                            ctx->tex_glcm, ctx->tex_mom);
    RTG_LAUNCH("k_tex_clear");
    const dim3 gb((unsigned)ceil_div(w, 256), (unsigned)(h < 1024 ? h : 1024));
    k_tex_bbox<<<gb, 256, 0, ctx->stream>>>(labels, (int)h, (int)w, d_n, cap, ctx->tex_bbox);
    RTG_LAUNCH("k_tex_bbox");
  }
  RTG_CUDA(launch_k(ctx, k_tex_accum, ctx->num_sms * 8, 256, 0, labels, intensity, edges, (int)h,
                    (int)w, d_n, cap, bb, ctx->tex_hist, ctx->tex_glcm, ctx->tex_mom));
  RTG_LAUNCH("k_tex_accum");
  RTG_CUDA(launch_k(ctx, k_tex_finalize, (unsigned)ceil_div(cap, 8), 256, 0, d_n, cap,
                    ctx->tex_hist, ctx->tex_glcm, ctx->tex_mom, out));
  RTG_LAUNCH("k_tex_finalize");
  return RTG_OK;
}

}  // namespace rtg
