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

// Optional 1-bit outputs of the vector kernels (uint16 pieces, one per
// 16-pixel group): ReconToNuclei's foreground (H >= t) and seed (H >= t + h)
// planes and the tissue plane.  fg == nullptr: none.
struct CdBits {
  uint16_t* fg = nullptr;
  uint16_t* sd = nullptr;
  uint16_t* ts = nullptr;
  uint32_t t4 = 0, s4 = 0;  // 256 - threshold, replicated into the four bytes
  int fg_on = 0, sd_on = 0;  // 0: threshold above 255, no pixel qualifies
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

// Flat path: rgb is h*w*3 contiguous, 16-byte aligned; 16 px per group.
// Each thread owns `iters` groups strided by the grid and prefetches group
// k+1 (3 x LDG.128, evict-first) before it computes group k; the first group
// is in flight while the block stages the LUTs.  The three 16.16 LUTs (the
// rounding constant folded into lut[0]) are replicated once per lane
// (word v*32 + lane, 96 KB per CTA): every LDS of a warp hits 32 distinct
// banks whatever the pixel values, where a shared 1 KB table averaged two
// wavefronts per gather (profiles/r1_colordeconv_*).  Per pixel: 3 PRMT
// byte extracts, 3 LEA + 3 LDS, one IADD3, the shift, and a saturating pack
// (cvt.pack.sat) of 2 pixels per instruction; the tissue test is integer
// min/max arithmetic on the same bytes (~22 instructions/px, was ~45).
// Streaming 16-byte load: evict-first in L1/L2, 256-byte L2 prefetch (a
// warp's three loads cover 1.5 KB of contiguous RGB).
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t pack_sat_u8(int32_t v0, int32_t v1, int32_t v2,
                                                int32_t v3) {
  uint32_t hi, d;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(v3), "r"(v2));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(v1), "r"(v0), "r"(hi));
  return d;
}

// byte MSBs (0xFF / 0x00 lanes of a SIMD compare) -> 4-bit mask, and bit 0
// of each byte (0 / 1 bytes) -> 4-bit mask: one multiply gathers the four
// bits without carries.
__device__ __forceinline__ uint32_t msb_nib(uint32_t v) {
  return ((v & 0x80808080u) * 0x00204081u) >> 28;
}
__device__ __forceinline__ uint32_t lsb_nib(uint32_t v) {
  return (((v & 0x01010101u) * 0x00204081u) >> 21) & 0xFu;
}
// Byte-wise x >= t as byte MSBs, tc = (256 - t) in every byte (1 <= t <=
// 255): bit 7 of each byte of x + tc carried out iff x >= t.  The low seven
// bits add without crossing bytes; the carry out of bit 7 is the majority of
// the two bit-7 inputs and the carry into it (three logic ops; the
// __vcmpgeu4 intrinsic is emulated in ~7).
__device__ __forceinline__ uint32_t ge_msbs(uint32_t x, uint32_t tc) {
  const uint32_t lo = (x & 0x7F7F7F7Fu) + (tc & 0x7F7F7F7Fu);
  return ((x & tc) | (x & lo) | (tc & lo)) & 0x80808080u;
}

// 16 pixels (48 interleaved RGB bytes in wv) -> 16 hematoxylin, tissue (and
// marker) bytes with the lane-replicated LUTs; with bits.fg also the
// ReconToNuclei threshold planes as 16-bit pieces of 1-bit planes (group g
// = bits 16g .. 16g+15): H >= t, (H >= t + h) && H >= t, tissue.
template <bool kMarker>
__device__ __forceinline__ void cd_group(const uint32_t (&wv)[12], const int32_t* l0,
                                         const int32_t* l1, const int32_t* l2, int32_t bgt,
                                         int32_t rg10, int32_t rb10, int32_t rh, uint4* hema,
                                         uint4* marker, uint4* tissue, uint32_t g,
                                         const CdBits& bits) {
  uint32_t ho[4], to[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int32_t hv[4], tv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int px = 4 * k + q;
      const int i0 = 3 * px, i1 = 3 * px + 1, i2 = 3 * px + 2;
      const int32_t r = (int32_t)__byte_perm(wv[i0 >> 2], 0, 0x4440 | (i0 & 3));
      const int32_t gg = (int32_t)__byte_perm(wv[i1 >> 2], 0, 0x4440 | (i1 & 3));
      const int32_t bb = (int32_t)__byte_perm(wv[i2 >> 2], 0, 0x4440 | (i2 & 3));
      hv[q] = (l0[r * 32] + l1[gg * 32] + l2[bb * 32]) >> 16;
      // tissue = !(min(r,g,b) > bg) && !(10r > rg10*g && 10r > rb10*b)
      //        = min(bg - min(r,g,b), max(rg10*g, rb10*b) - 10r) >= 0
      const int32_t nb = bgt - min(min(r, gg), bb);
      const int32_t nr = max(rg10 * gg, rb10 * bb) - 10 * r;
      tv[q] = (int32_t)((~(uint32_t)(nb | nr)) >> 31);
    }
    ho[k] = pack_sat_u8(hv[0], hv[1], hv[2], hv[3]);
    to[k] = pack_sat_u8(tv[0], tv[1], tv[2], tv[3]);
  }
  hema[g] = make_uint4(ho[0], ho[1], ho[2], ho[3]);
  if (tissue) tissue[g] = make_uint4(to[0], to[1], to[2], to[3]);
  if (bits.fg) {
    uint32_t f = 0, sd = 0, t = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (bits.fg_on) f |= msb_nib(ge_msbs(ho[k], bits.t4)) << (4 * k);
      if (bits.sd_on) sd |= msb_nib(ge_msbs(ho[k], bits.s4)) << (4 * k);
      t |= lsb_nib(to[k]) << (4 * k);
    }
    bits.fg[g] = (uint16_t)f;
    bits.sd[g] = (uint16_t)(sd & f);
    bits.ts[g] = (uint16_t)t;
  }
  if (kMarker) {
    // max(H - recon_h, 0) per byte (H in [0,255], recon_h >= 0)
    uint32_t mo[4];
    const uint32_t hrep = (uint32_t)(rh > 255 ? 255 : rh) * 0x01010101u;
#pragma unroll
    for (int k = 0; k < 4; ++k) mo[k] = __vsubus4(ho[k], hrep);
    marker[g] = make_uint4(mo[0], mo[1], mo[2], mo[3]);
  }
}

// The three LUTs into shared memory: lsmall [3][256] (+32768 rounding in
// lut[0]) and the lane-replicated copy lrep [3][256][32].
__device__ __forceinline__ void cd_stage_luts(const CdParams& p, int32_t* lrep, int32_t* lsmall) {
  // 192 x 16-byte constant-bank reads (divergent LDC replays once per
  // distinct address, so wide reads keep the staging short) ...
  const int4* src = reinterpret_cast<const int4*>(&p.lut.v[0][0]);
  int4* dst = reinterpret_cast<int4*>(lsmall);
  for (int i = threadIdx.x; i < 192; i += blockDim.x) {
    int4 v = src[i];
    if (i < 64) {  // lut[0] carries the +32768 of the rounding shift
      v.x += 32768; v.y += 32768; v.z += 32768; v.w += 32768;
    }
    dst[i] = v;
  }
  __syncthreads();
  // ... then 32 lane copies of each entry, 16 bytes per store
  int4* rep = reinterpret_cast<int4*>(lrep);
  for (int i = threadIdx.x; i < 3 * 256 * 8; i += blockDim.x) {
    const int32_t v = lsmall[i >> 3];
    rep[i] = make_int4(v, v, v, v);
  }
  __syncthreads();
}

constexpr int kCdThreads = 512;
constexpr int kCdBlocksPerSm = 2;
constexpr size_t kCdSmem = 3 * 256 * 32 * sizeof(int32_t) + 3 * 256 * sizeof(int32_t);

template <bool kMarker>
__global__ void __launch_bounds__(kCdThreads, kCdBlocksPerSm)
k_colordeconv_vec(const uint4* __restrict__ rgb, uint32_t ngroups, int iters,
                  const __grid_constant__ CdParams p, uint4* __restrict__ hema,
                  uint4* __restrict__ marker, uint4* __restrict__ tissue, const ClearList clear,
                  const CdBits bits) {
  pdl_enter();
  if (blockIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < 6; ++r)  // constant indices: the list stays in parameter space
      if (r < clear.count)
        for (int i = threadIdx.x; i < clear.n[r]; i += blockDim.x) clear.p[r][i] = 0;
  }
  extern __shared__ __align__(16) int32_t cd_smem[];
  int32_t* lrep = cd_smem;                   // [3][256][32]
  int32_t* lsmall = cd_smem + 3 * 256 * 32;  // [3][256]
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  uint4 a = make_uint4(0, 0, 0, 0), b = a, c = a;
  if (g < ngroups) {
    a = ld_stream(rgb + 3 * g);
    b = ld_stream(rgb + 3 * g + 1);
    c = ld_stream(rgb + 3 * g + 2);
  }
  cd_stage_luts(p, lrep, lsmall);
  const int lane = threadIdx.x & 31;
  const int32_t* l0 = lrep + lane;
  const int32_t* l1 = lrep + 256 * 32 + lane;
  const int32_t* l2 = lrep + 2 * 256 * 32 + lane;
  const int32_t bgt = p.bg, rg10 = p.rg10, rb10 = p.rb10, rh = p.recon_h;
  for (int it = 0; it < iters && g < ngroups; ++it, g += stride) {
    const uint32_t wv[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
    const uint32_t gn = g + stride;
    if (it + 1 < iters && gn < ngroups) {
      a = ld_stream(rgb + 3 * gn);
      b = ld_stream(rgb + 3 * gn + 1);
      c = ld_stream(rgb + 3 * gn + 2);
    }
    cd_group<kMarker>(wv, l0, l1, l2, bgt, rg10, rb10, rh, hema, marker, tissue, g, bits);
  }
}


// TMA-staged variant (RTG_OPT_STREAM_IMPL = 1): one CTA per SM streams
// chunks of 512 x 16 px (24 KB of RGB) through a 4-stage shared-memory ring
// filled by 1-D bulk async copies (cp.async.bulk, completion on an mbarrier);
// thread 0 refills a stage as soon as every thread has read it, so four
// chunks are in flight per SM without any load instruction in the consumer
// warps (their 48 bytes come from three conflict-free LDS.128).  Same
// per-pixel arithmetic as k_colordeconv_vec (cd_group).
constexpr int kTmaThreads = 512;
constexpr int kTmaStages = 4;
constexpr uint32_t kTmaChunk = kTmaThreads * 48u;  // bytes of RGB per stage
constexpr size_t kTmaSmem = kCdSmem + kTmaStages * (size_t)kTmaChunk + kTmaStages * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <bool kMarker>
__global__ void __launch_bounds__(kTmaThreads, 1)
k_colordeconv_tma(const uint8_t* __restrict__ rgb, uint32_t ngroups,
                  const __grid_constant__ CdParams p, uint4* __restrict__ hema,
                  uint4* __restrict__ marker, uint4* __restrict__ tissue, const ClearList clear,
                  const CdBits bits) {
  pdl_enter();
  if (blockIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < 6; ++r)
      if (r < clear.count)
        for (int i = threadIdx.x; i < clear.n[r]; i += blockDim.x) clear.p[r][i] = 0;
  }
  extern __shared__ __align__(16) int32_t cd_smem[];
  int32_t* lrep = cd_smem;
  int32_t* lsmall = cd_smem + 3 * 256 * 32;
  uint8_t* ring = reinterpret_cast<uint8_t*>(cd_smem) + kCdSmem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kTmaStages * (size_t)kTmaChunk);
  const uint32_t nchunks = (ngroups + kTmaThreads - 1) / kTmaThreads;
  const uint64_t total = (uint64_t)ngroups * 48u;
  auto chunk_bytes = [&](uint32_t c) -> uint32_t {
    const uint64_t off = (uint64_t)c * kTmaChunk;
    const uint64_t left = total - off;
    return left < kTmaChunk ? (uint32_t)left : kTmaChunk;
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < kTmaStages; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the first chunks are in flight while the LUTs are staged
    for (int st = 0; st < kTmaStages; ++st) {
      const uint32_t c = blockIdx.x + (uint32_t)st * gridDim.x;
      if (c < nchunks) {
        mbar_expect_tx(&bars[st], chunk_bytes(c));
        bulk_load(ring + st * (size_t)kTmaChunk, rgb + (uint64_t)c * kTmaChunk, chunk_bytes(c),
                  &bars[st]);
      }
    }
  }
  cd_stage_luts(p, lrep, lsmall);  // ends with __syncthreads (barrier init visible)
  const int lane = threadIdx.x & 31;
  const int32_t* l0 = lrep + lane;
  const int32_t* l1 = lrep + 256 * 32 + lane;
  const int32_t* l2 = lrep + 2 * 256 * 32 + lane;
  const int32_t bgt = p.bg, rg10 = p.rg10, rb10 = p.rb10, rh = p.recon_h;
  uint32_t it = 0;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const int st = (int)(it % kTmaStages);
    mbar_wait(&bars[st], (it / kTmaStages) & 1u);
    const uint32_t g = c * kTmaThreads + threadIdx.x;
    uint32_t wv[12];
    if (g < ngroups) {
      const uint4* src = reinterpret_cast<const uint4*>(ring + st * (size_t)kTmaChunk) + 3 * threadIdx.x;
      const uint4 a = src[0], b = src[1], d = src[2];
      wv[0] = a.x; wv[1] = a.y; wv[2] = a.z; wv[3] = a.w;
      wv[4] = b.x; wv[5] = b.y; wv[6] = b.z; wv[7] = b.w;
      wv[8] = d.x; wv[9] = d.y; wv[10] = d.z; wv[11] = d.w;
    }
    __syncthreads();  // every thread has its bytes: the stage may be refilled
    if (threadIdx.x == 0) {
      const uint32_t cn = c + (uint32_t)kTmaStages * gridDim.x;
      if (cn < nchunks) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[st], chunk_bytes(cn));
        bulk_load(ring + st * (size_t)kTmaChunk, rgb + (uint64_t)cn * kTmaChunk, chunk_bytes(cn),
                  &bars[st]);
      }
    }
    if (g < ngroups)
      cd_group<kMarker>(wv, l0, l1, l2, bgt, rg10, rb10, rh, hema, marker, tissue, g, bits);
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
                       uint8_t* marker, uint8_t* tissue, const ClearList* clear,
                       uint32_t* const* recon_bits, bool* bits_written) {
  ClearList cl{};
  if (clear) cl = *clear;
  CdParams cp;
  hema_lut(p, &cp.lut);
  cp.bg = p->bg_thresh;
  cp.rg10 = p->rbc_rg10;
  cp.rb10 = p->rbc_rb10;
  cp.recon_h = p->recon_h;
  const int64_t n = h * w;
  const bool flat = pitch == 3 * w && aligned16(rgb) && hema && aligned16(hema) &&
                    (tissue || recon_bits) && (!tissue || aligned16(tissue)) &&
                    (!marker || aligned16(marker)) && n % 16 == 0;
  CdBits bits;
  if (bits_written) *bits_written = false;
  if (recon_bits && flat) {
    // recon_bits = {fg, seed, tissue} planes; thresholds as FgThresh
    const int64_t t = p->nuc_thresh, ts = (int64_t)p->nuc_thresh + p->recon_h;
    bits.fg = reinterpret_cast<uint16_t*>(recon_bits[0]);
    bits.sd = reinterpret_cast<uint16_t*>(recon_bits[1]);
    bits.ts = reinterpret_cast<uint16_t*>(recon_bits[2]);
    bits.fg_on = t <= 255;
    bits.sd_on = ts <= 255;
    // (256 - t) per byte for ge_msbs; t >= 1 here (nuc_thresh > 0, recon_h >= 0)
    bits.t4 = 0x01010101u * (uint32_t)(t >= 1 && t <= 255 ? 256 - t : 0);
    bits.s4 = 0x01010101u * (uint32_t)(ts >= 1 && ts <= 255 ? 256 - ts : 0);
    if (t < 1) return fail(RTG_ERR_INTERNAL, "threshold planes need nuc_thresh >= 1");
    if (bits_written) *bits_written = true;
    tissue = nullptr;  // the tissue plane goes out as bits only
  } else if (!tissue) {
    return fail(RTG_ERR_INTERNAL, "colour deconvolution without a tissue output");
  }
  int64_t done = 0;
  if (flat) {
    const int64_t ngroups = n / 16 < INT32_MAX ? n / 16 : 0;
    if (ngroups > 0) {
      // all groups in one resident wave: iters per thread, then as few
      // blocks as cover ngroups at that depth
      if (ctx->stream_impl == 1) {
        RTG_SMEM_OPTIN(k_colordeconv_tma<true>, kTmaSmem);
        RTG_SMEM_OPTIN(k_colordeconv_tma<false>, kTmaSmem);
        auto kern = marker ? k_colordeconv_tma<true> : k_colordeconv_tma<false>;
        const uint32_t nchunks = (uint32_t)ceil_div(ngroups, kTmaThreads);
        const int blocks = (int)(nchunks < (uint32_t)ctx->num_sms ? nchunks : ctx->num_sms);
        RTG_CUDA(launch_k(ctx, kern, blocks, kTmaThreads, kTmaSmem, rgb, (uint32_t)ngroups, cp,
                          reinterpret_cast<uint4*>(hema), reinterpret_cast<uint4*>(marker),
                          reinterpret_cast<uint4*>(tissue), cl, bits));
        cl.count = 0;
        RTG_LAUNCH("k_colordeconv_tma");
      } else {
        RTG_SMEM_OPTIN(k_colordeconv_vec<true>, kCdSmem);
        RTG_SMEM_OPTIN(k_colordeconv_vec<false>, kCdSmem);
        const int64_t slots = (int64_t)ctx->num_sms * kCdBlocksPerSm * kCdThreads;
        const int iters = (int)ceil_div(ngroups, slots);
        const int blocks = (int)ceil_div(ngroups, (int64_t)kCdThreads * iters);
        auto kern = marker ? k_colordeconv_vec<true> : k_colordeconv_vec<false>;
        RTG_CUDA(launch_k(ctx, kern, blocks, kCdThreads, kCdSmem,
                          reinterpret_cast<const uint4*>(rgb), (uint32_t)ngroups, iters, cp,
                          reinterpret_cast<uint4*>(hema), reinterpret_cast<uint4*>(marker),
                          reinterpret_cast<uint4*>(tissue), cl, bits));
        cl.count = 0;
        RTG_LAUNCH("k_colordeconv_vec");
      }
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
  if (cl.count) {  // no vector launch: a separate zeroing launch
    ZeroList z{};
    for (int r = 0; r < cl.count; ++r) {
      z.ptr[r] = cl.p[r];
      z.bytes[r] = sizeof(int32_t) * (uint64_t)cl.n[r];
    }
    z.count = cl.count;
    RTG_TRY(zero_async(ctx, z));
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
