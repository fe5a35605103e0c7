// Device rasteriser of the synthetic H&E tiles.  Consumes the shape list
// generated on the host by rtg_synth_shapes (synth.c) and reproduces
// rtg_synth_raster_host byte for byte: per-pixel winner = max shape key
// (atomicMax, order-independent), colour = base + tint + hash noise.
#include <vector>

#include "common.cuh"
#include "synth.h"

extern "C" int64_t rtg_synth_shapes(uint64_t tile_seed, int64_t h, int64_t w,
                                    rtg_shape* out);
extern "C" int64_t rtg_synth_max_shapes(int64_t h, int64_t w);

namespace rtg {
namespace {

__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__global__ void k_synth_stamp(const rtg_shape* __restrict__ shapes, int h, int w,
                              uint32_t* __restrict__ key) {
  const rtg_shape s = shapes[blockIdx.x];
  const int y0 = max(s.y0, 0), y1 = min(s.y1, h - 1);
  const int x0 = max(s.x0, 0), x1 = min(s.x1, w - 1);
  if (y0 > y1 || x0 > x1) return;
  const int bw = x1 - x0 + 1;
  const int cnt = (y1 - y0 + 1) * bw;
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
    const int y = y0 + k / bw, x = x0 + k % bw;
    const int64_t dy = y - s.cy, dx = x - s.cx;
    if (s.A * dx * dx + s.B * dx * dy + s.C * dy * dy <= s.K)
      atomicMax(&key[(int64_t)y * w + x], s.key);
  }
}

__constant__ unsigned char c_base[4][3] = {
    {230, 160, 200}, {242, 238, 242}, {205, 70, 80}, {95, 70, 155}};

__global__ void k_synth_colour(const rtg_shape* __restrict__ shapes, uint64_t seed,
                               int64_t n, const uint32_t* __restrict__ key,
                               uint8_t* __restrict__ rgb) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = key[p];
    const int cls = k ? (int)(k >> 24) : 0;
    const int tint = k ? shapes[k & 0xFFFFFFu].tint : 0;
    const uint64_t z = splitmix64_d(seed ^ 0xd1b54a32d192ed03ULL ^ (uint64_t)p);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int a = (int)((z >> (16 * c)) & 0xFF);
      const int b = (int)((z >> (16 * c + 8)) & 0xFF);
      int v = c_base[cls][c] + tint + ((a + b) >> 4) - 16;
      rgb[3 * p + c] = (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
    }
  }
}

}  // namespace

int synth_dev(rtg_ctx* ctx, uint64_t global_seed, int64_t tile_row,
              int64_t tile_col, int64_t h, int64_t w, uint8_t* d_rgb) {
  const uint64_t seed = rtg_tile_seed(global_seed, tile_row, tile_col);
  std::vector<rtg_shape> shapes((size_t)rtg_synth_max_shapes(h, w));
  const int64_t ns = rtg_synth_shapes(seed, h, w, shapes.data());
  rtg_shape* d_shapes = nullptr;
  RTG_CUDA(cudaMallocAsync((void**)&d_shapes, sizeof(rtg_shape) * (size_t)(ns > 0 ? ns : 1),
                           ctx->stream));
  if (ns > 0)
    RTG_CUDA(cudaMemcpyAsync(d_shapes, shapes.data(), sizeof(rtg_shape) * (size_t)ns,
                             cudaMemcpyHostToDevice, ctx->stream));
  uint32_t* key = reinterpret_cast<uint32_t*>(ctx->i32a);
  RTG_CUDA(cudaMemsetAsync(key, 0, sizeof(uint32_t) * (size_t)(h * w), ctx->stream));
  if (ns > 0) {
    k_synth_stamp<<<(unsigned)ns, 128, 0, ctx->stream>>>(d_shapes, (int)h, (int)w, key);
    RTG_LAUNCH("k_synth_stamp");
  }
  const int64_t n = h * w;
  k_synth_colour<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(d_shapes, seed, n, key, d_rgb);
  RTG_LAUNCH("k_synth_colour");
  RTG_CUDA(cudaFreeAsync(d_shapes, ctx->stream));
  // the host vector must outlive the async copy of pageable memory: a
  // pageable cudaMemcpyAsync is staged before it returns, so this is safe.
  return RTG_OK;
}

}  // namespace rtg
