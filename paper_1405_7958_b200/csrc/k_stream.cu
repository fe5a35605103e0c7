// o1 + o2: fused colour deconvolution and thresholds (PAPER.md:1133-1135,
// 1592) as a 128-bit streaming kernel, plus the small elementwise kernels of
// the pipeline.
//
// Roofline: HBM-bound.  Algorithmic bytes per pixel:
// RGB in 3 B + hematoxylin 1 B + HMAX marker 1 B + tissue 1 B = 6 B/px.
// Each thread moves 16 pixels: 3 x LDG.128 in, 3 x STG.128 out.
#include "common.cuh"

namespace rtg {
namespace {

struct CdParams {
  HemaLut lut;
  int32_t bg, rg10, rb10, recon_h;
};

__device__ __forceinline__ void cd_pixel(const int32_t (*lut)[256],
                                         const CdParams& p, uint32_t r,
                                         uint32_t g, uint32_t b, uint32_t& hv,
                                         uint32_t& mk, uint32_t& tis) {
  const int32_t s = lut[0][r] + lut[1][g] + lut[2][b];
  int32_t v = 0;
  if (s > 0) {
    v = (s + 32768) >> 16;
    v = v > 255 ? 255 : v;
  }
  hv = (uint32_t)v;
  mk = (uint32_t)(v > p.recon_h ? v - p.recon_h : 0);
  const bool bg = (int)r > p.bg && (int)g > p.bg && (int)b > p.bg;
  const bool rbc = 10 * (int)r > p.rg10 * (int)g && 10 * (int)r > p.rb10 * (int)b;
  tis = (!bg && !rbc) ? 1u : 0u;
}

// Flat path: rgb is h*w*3 contiguous, 16-byte aligned; 16 px per thread.
__global__ void __launch_bounds__(256)
k_colordeconv_vec(const uint4* __restrict__ rgb, int64_t ngroups,
                  const __grid_constant__ CdParams p, uint4* __restrict__ hema,
                  uint4* __restrict__ marker, uint4* __restrict__ tissue) {
  pdl_enter();
  __shared__ int32_t lut[3][256];
  for (int i = threadIdx.x; i < 768; i += blockDim.x)
    lut[i >> 8][i & 255] = p.lut.v[i >> 8][i & 255];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups;
       g += stride) {
    uint32_t wv[12];
    {
      const uint4 a = __ldcs(rgb + 3 * g);
      const uint4 b = __ldcs(rgb + 3 * g + 1);
      const uint4 c = __ldcs(rgb + 3 * g + 2);
      wv[0] = a.x; wv[1] = a.y; wv[2] = a.z; wv[3] = a.w;
      wv[4] = b.x; wv[5] = b.y; wv[6] = b.z; wv[7] = b.w;
      wv[8] = c.x; wv[9] = c.y; wv[10] = c.z; wv[11] = c.w;
    }
    uint32_t ho[4] = {0, 0, 0, 0}, mo[4] = {0, 0, 0, 0}, to[4] = {0, 0, 0, 0};
#pragma unroll
    for (int px = 0; px < 16; ++px) {
      const int b0 = 3 * px, b1 = 3 * px + 1, b2 = 3 * px + 2;
      const uint32_t r = (wv[b0 >> 2] >> (8 * (b0 & 3))) & 0xFFu;
      const uint32_t gg = (wv[b1 >> 2] >> (8 * (b1 & 3))) & 0xFFu;
      const uint32_t bb = (wv[b2 >> 2] >> (8 * (b2 & 3))) & 0xFFu;
      uint32_t hv, mk, tis;
      cd_pixel(lut, p, r, gg, bb, hv, mk, tis);
      ho[px >> 2] |= hv << (8 * (px & 3));
      mo[px >> 2] |= mk << (8 * (px & 3));
      to[px >> 2] |= tis << (8 * (px & 3));
    }
    if (hema) hema[g] = make_uint4(ho[0], ho[1], ho[2], ho[3]);
    if (marker) marker[g] = make_uint4(mo[0], mo[1], mo[2], mo[3]);
    if (tissue) tissue[g] = make_uint4(to[0], to[1], to[2], to[3]);
  }
}

// General path: arbitrary pitch / alignment / tail, one pixel per thread.
__global__ void __launch_bounds__(256)
k_colordeconv_px(const uint8_t* __restrict__ rgb, int64_t h, int64_t w,
                 int64_t pitch, int64_t first, const __grid_constant__ CdParams p,
                 uint8_t* __restrict__ hema, uint8_t* __restrict__ marker,
                 uint8_t* __restrict__ tissue) {
  pdl_enter();
  __shared__ int32_t lut[3][256];
  for (int i = threadIdx.x; i < 768; i += blockDim.x)
    lut[i >> 8][i & 255] = p.lut.v[i >> 8][i & 255];
  __syncthreads();
  const int64_t n = h * w;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = first + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       i < n; i += stride) {
    const int64_t y = i / w, x = i - y * w;
    const uint8_t* px = rgb + y * pitch + 3 * x;
    uint32_t hv, mk, tis;
    cd_pixel(lut, p, px[0], px[1], px[2], hv, mk, tis);
    if (hema) hema[i] = (uint8_t)hv;
    if (marker) marker[i] = (uint8_t)mk;
    if (tissue) tissue[i] = (uint8_t)tis;
  }
}

// candidate = recon >= thresh && tissue, 16 px per thread.
__global__ void __launch_bounds__(256)
k_candidate(const uint4* __restrict__ recon, const uint4* __restrict__ tissue,
            int64_t ngroups, uint32_t thresh, uint4* __restrict__ out) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups;
       g += stride) {
    const uint4 r = recon[g], t = tissue[g];
    const uint32_t rv[4] = {r.x, r.y, r.z, r.w};
    const uint32_t tv[4] = {t.x, t.y, t.z, t.w};
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // per-byte (recon >= thresh) via SIMD compare: __vcmpgeu4 -> 0xFF lanes
      const uint32_t ge = __vcmpgeu4(rv[k], thresh * 0x01010101u);
      o[k] = ge & tv[k] & 0x01010101u;
    }
    out[g] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void k_candidate_tail(const uint8_t* recon, const uint8_t* tissue,
                                 int64_t first, int64_t n, int32_t thresh,
                                 uint8_t* out) {
  pdl_enter();
  const int64_t i = first + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint8_t)(recon[i] >= thresh && tissue[i]);
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// Up to four regions zeroed by one PDL-launched kernel (a cudaMemsetAsync
// node would cut the programmatic overlap of the kernel chain).
__global__ void __launch_bounds__(256) k_zero(ZeroList z) {
  pdl_enter();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < z.count; ++r) {
    uint8_t* p = static_cast<uint8_t*>(z.ptr[r]);
    const int64_t n = (int64_t)z.bytes[r];
    int64_t done = 0;
    if (((uintptr_t)p & 15u) == 0) {
      const int64_t n16 = n / 16;
      uint4* q = reinterpret_cast<uint4*>(p);
      for (int64_t i = tid; i < n16; i += nth) q[i] = make_uint4(0, 0, 0, 0);
      done = n16 * 16;
    }
    for (int64_t i = done + tid; i < n; i += nth) p[i] = 0;
  }
}

}  // namespace

void hema_lut(const rtg_params* p, HemaLut* lut) {
  // identical expression to the oracle (oracle/rtg_oracle.c orc_hema_lut):
  // llround(coef * od * (255 / h_scale) * 65536), od = -log10((v+1)/256).
  const double scale255 = 255.0 / p->h_scale;
  for (int c = 0; c < 3; ++c) {
    for (int v = 0; v < 256; ++v) {
      const double od = -log10((double)(v + 1) / 256.0);
      lut->v[c][v] = (int32_t)llround(p->h_coef[c] * od * scale255 * 65536.0);
    }
  }
}

int launch_colordeconv(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w,
                       int64_t pitch, const rtg_params* p, uint8_t* hema,
                       uint8_t* marker, uint8_t* tissue) {
  CdParams cp;
  hema_lut(p, &cp.lut);
  cp.bg = p->bg_thresh;
  cp.rg10 = p->rbc_rg10;
  cp.rb10 = p->rbc_rb10;
  cp.recon_h = p->recon_h;
  const int64_t n = h * w;
  const bool flat = pitch == 3 * w && aligned16(rgb) &&
                    (!hema || aligned16(hema)) && (!marker || aligned16(marker)) &&
                    (!tissue || aligned16(tissue));
  int64_t done = 0;
  if (flat) {
    const int64_t ngroups = n / 16;
    if (ngroups > 0) {
      const int64_t want = ceil_div(ngroups, 256);
      const int blocks = (int)(want < (int64_t)ctx->num_sms * 8 ? want : (int64_t)ctx->num_sms * 8);
      RTG_CUDA(launch_k(ctx, k_colordeconv_vec, blocks, 256, 0, 
          reinterpret_cast<const uint4*>(rgb), ngroups, cp,
          reinterpret_cast<uint4*>(hema), reinterpret_cast<uint4*>(marker),
          reinterpret_cast<uint4*>(tissue)));
      RTG_LAUNCH("k_colordeconv_vec");
    }
    done = ngroups * 16;
  }
  if (done < n) {
    const int64_t rem = n - done;
    const int64_t want = ceil_div(rem, 256);
    const int blocks = (int)(want < (int64_t)ctx->num_sms * 16 ? want : (int64_t)ctx->num_sms * 16);
    RTG_CUDA(launch_k(ctx, k_colordeconv_px, blocks, 256, 0, rgb, h, w, pitch, done, cp,
                                                      hema, marker, tissue));
    RTG_LAUNCH("k_colordeconv_px");
  }
  return RTG_OK;
}

int zero_async(rtg_ctx* ctx, const ZeroList& z) {
  int64_t big = 0;
  for (int r = 0; r < z.count; ++r) big = big > (int64_t)z.bytes[r] ? big : (int64_t)z.bytes[r];
  int64_t blocks = ceil_div(big / 16 + 1, 256);
  if (blocks > ctx->num_sms * 4) blocks = ctx->num_sms * 4;
  RTG_CUDA(launch_k(ctx, k_zero, dim3((unsigned)blocks), dim3(256), 0, z));
  RTG_LAUNCH("k_zero");
  return RTG_OK;
}

int launch_candidate(rtg_ctx* ctx, const uint8_t* recon, const uint8_t* tissue,
                     int64_t n, int32_t thresh, uint8_t* out) {
  int64_t done = 0;
  if (aligned16(recon) && aligned16(tissue) && aligned16(out)) {
    const int64_t ngroups = n / 16;
    if (ngroups > 0) {
      const int64_t want = ceil_div(ngroups, 256);
      const int blocks = (int)(want < (int64_t)ctx->num_sms * 8 ? want : (int64_t)ctx->num_sms * 8);
      const uint32_t t = thresh < 0 ? 0u : thresh > 255 ? 256u : (uint32_t)thresh;
      if (t <= 255) {
        RTG_CUDA(launch_k(ctx, k_candidate, blocks, 256, 0, 
            reinterpret_cast<const uint4*>(recon),
            reinterpret_cast<const uint4*>(tissue), ngroups, t,
            reinterpret_cast<uint4*>(out)));
        RTG_LAUNCH("k_candidate");
        done = ngroups * 16;
      }
    }
  }
  if (done < n) {
    RTG_CUDA(launch_k(ctx, k_candidate_tail, (unsigned)ceil_div(n - done, 256), 256, 0, 
        recon, tissue, done, n, thresh, out));
    RTG_LAUNCH("k_candidate_tail");
  }
  return RTG_OK;
}

}  // namespace rtg
