// o6 PreWatershed + o7 Watershed.
//
// Markers: F = HMAX_ws_h(dq) by IWPP reconstruction, Fw = fg ? F + 1 : 0,
// regional maxima = Fw > recon(Fw - 1, Fw) (a second IWPP pass).
// Watershed: the arrowing ("tobogganing") formulation of the Koerbes et al.
// GPU watershed the paper uses: every foreground pixel points to its steepest
// ascending 8-neighbour (max Fw, ties -> minimum linear index); pixels of
// non-maximal plateaus point down the BFS distance to the plateau exits
// (ties -> minimum index); regional-maximum pixels are roots.  Following the
// arrows gives each pixel its marker.  Every rule is local and
// order-independent, so the labelling is unique (bit-exact vs the CPU
// oracle).  Separation lines: drop pixels having an 8-neighbour with a higher
// basin id.
//
// Roofline: HBM/L2 bound; algorithmic bytes mask 1 B in + sep 1 B + basin 4 B
// out (dq/markers/Fw are internal planes).
#include "common.cuh"

namespace rtg {
namespace {

constexpr int32_t kInfD = 1 << 30;

__global__ void k_ws_prep(int64_t n, const uint8_t* __restrict__ mask,
                          const uint16_t* __restrict__ F, uint16_t* __restrict__ Fw) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    Fw[i] = (uint16_t)(mask[i] ? (uint32_t)F[i] + 1u : 0u);
}

// Arrows / plateau list.  ptr: steepest ascent for pixels with a higher
// neighbour (delta 0); every other foreground pixel goes on the plateau list
// (delta INF): the plateau BFS either reaches it (non-maximal plateau) or not
// — then it is a regional maximum, i.e. Fw > recon(Fw - 1, Fw), because its
// plateau has no pixel with a higher neighbour.  ptr / delta are written for
// foreground pixels only; rm is cleared everywhere (the BFS sets markers).
__global__ void __launch_bounds__(256)
k_ws_arrows(int h, int w, const uint16_t* __restrict__ Fw, uint8_t* __restrict__ rm,
            int32_t* __restrict__ ptr, int32_t* __restrict__ delta,
            int32_t* __restrict__ flat_list, int32_t* __restrict__ flat_count) {
  for (int y = blockIdx.y; y < h; y += gridDim.y)
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < w; x += gridDim.x * blockDim.x) {
    const int64_t i = (int64_t)y * w + x;
    const uint32_t f = Fw[i];
    const uint8_t is_rm = 0;
    int32_t p = -1, d = -1;
    if (f) {
      {
        uint32_t best = f;
        int32_t arg = -1;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
          for (int dx = -1; dx <= 1; ++dx) {
            if (dy == 0 && dx == 0) continue;
            const int yy = y + dy, xx = x + dx;
            if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
            const int32_t j = yy * w + xx;
            const uint32_t fj = Fw[j];
            if (fj > best) { best = fj; arg = j; }  // row-major order: first max = min index
          }
        }
        if (arg >= 0) {
          p = arg;
          d = 0;
        } else {
          p = -2;
          d = kInfD;
          const int slot = atomicAdd(flat_count, 1);
          flat_list[slot] = (int32_t)i;
        }
      }
    }
    rm[i] = is_rm;
    if (f) {
      ptr[i] = p;
      delta[i] = d;
    }
  }
}

// One grid-wide relaxation pass over the plateau list (chaotic Bellman-Ford:
// values only decrease and always equal the length of some real path, so
// passes in any order converge to the unique fixed point).  A few of these
// resolve almost every plateau before the single-CTA pass below, which owns
// the convergence test, has to iterate.
// Relaxes plateau pixel i once; returns true when its distance dropped.
// Branch-free neighbour gathers (out-of-tile neighbours alias i), so the 16
// loads of a pixel are issued back to back.
__device__ __forceinline__ bool relax_plateau_px(int h, int w, const uint16_t* __restrict__ Fw,
                                                 int32_t i, int32_t* delta) {
  const int y = i / w, x = i - y * w;
  const uint32_t f = Fw[i];
  const int32_t cur = __ldcg(&delta[i]);
  int32_t best = cur;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      if (dy == 0 && dx == 0) continue;
      const int yy = y + dy, xx = x + dx;
      const bool in = yy >= 0 && yy < h && xx >= 0 && xx < w;
      const int32_t j = in ? yy * w + xx : i;
      const uint32_t fj = Fw[j];
      const int32_t dj = __ldcg(&delta[j]);
      const int32_t cand = (in && fj == f && dj >= 0 && dj < kInfD) ? dj + 1 : kInfD;
      best = min(best, cand);
    }
  }
  if (best < cur) {
    __stcg(&delta[i], best);
    return true;
  }
  return false;
}

// Software grid barrier (sense by generation).  Only used by kernels launched
// with cudaLaunchCooperativeKernel, which guarantees co-residency.
__device__ __forceinline__ void grid_barrier(unsigned* arrive, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = atomicAdd(gen, 0u);
    __threadfence();
    if (atomicAdd(arrive, 1u) == gridDim.x - 1) {
      atomicExch(arrive, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (atomicAdd(gen, 0u) == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Plateau distances and arrows in one cooperative launch: rounds of
// grid-wide chaotic Bellman-Ford over the plateau list until a round changes
// nothing (values only decrease and always equal some real path length, so
// the fixed point is the BFS distance), then every plateau pixel points at the
// same-level neighbour at distance delta-1 with the minimum linear index.
// flags[0..1] and bar[0..1] must be zero on entry.
__global__ void __launch_bounds__(256)
k_ws_plateau(int h, int w, const uint16_t* __restrict__ Fw,
             const int32_t* __restrict__ flat_list, const int32_t* __restrict__ flat_count,
             int32_t* delta, int32_t* __restrict__ ptr, uint8_t* __restrict__ rm,
             int32_t* flags, unsigned* bar) {
  const int n = *flat_count;
  if (n == 0) return;
  for (int round = 0; round <= n + 1; ++round) {
    bool any = false;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
      any |= relax_plateau_px(h, w, Fw, flat_list[k], delta);
    if (__syncthreads_or(any) && threadIdx.x == 0) atomicExch(&flags[round & 1], 1);
    grid_barrier(bar, bar + 1);
    const int changed = *(volatile int32_t*)&flags[round & 1];
    grid_barrier(bar, bar + 1);  // everyone has read the flag
    if (blockIdx.x == 0 && threadIdx.x == 0) flags[round & 1] = 0;  // reused two rounds later
    if (!changed) break;
  }
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t i = flat_list[k];
    const int32_t di = __ldcg(&delta[i]);
    if (di >= kInfD) {  // unreachable: a regional-maximum (marker) pixel
      rm[i] = 1;
      ptr[i] = i;
      continue;
    }
    const int y = i / w, x = i - y * w;
    const uint32_t f = Fw[i];
    int32_t arg = -2;
    for (int dy = -1; dy <= 1 && arg < 0; ++dy) {
      for (int dx = -1; dx <= 1; ++dx) {
        if (dy == 0 && dx == 0) continue;
        const int yy = y + dy, xx = x + dx;
        if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
        const int32_t j = yy * w + xx;
        if (Fw[j] == f && __ldcg(&delta[j]) == di - 1) { arg = j; break; }
      }
    }
    ptr[i] = arg;
  }
}

__global__ void k_ws_resolve(int64_t n, const uint8_t* __restrict__ mask,
                             const int32_t* __restrict__ ptr,
                             const int32_t* __restrict__ mroots,
                             int32_t* __restrict__ basin) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t b = 0;
    if (mask[i]) {
      int32_t q = (int32_t)i;
      int32_t nx = ptr[q];
      while (nx >= 0 && nx != q) {
        q = nx;
        nx = ptr[q];
      }
      b = nx == q ? root_of(mroots, q) + 1 : 0;
    }
    basin[i] = b;
  }
}

__global__ void k_ws_separate(int h, int w, const int32_t* __restrict__ basin,
                              uint8_t* __restrict__ sep) {
  for (int y = blockIdx.y; y < h; y += gridDim.y)
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < w; x += gridDim.x * blockDim.x) {
    const int64_t i = (int64_t)y * w + x;
    const int32_t b = basin[i];
    uint8_t keep = b > 0;
    if (keep) {
      for (int dy = -1; dy <= 1 && keep; ++dy) {
        for (int dx = -1; dx <= 1; ++dx) {
          const int yy = y + dy, xx = x + dx;
          if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
          if (basin[(int64_t)yy * w + xx] > b) { keep = 0; break; }
        }
      }
    }
    sep[i] = keep;
  }
}

int grid_for(rtg_ctx* ctx, int64_t n) {
  const int64_t want = ceil_div(n, 256);
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  return (int)(want < cap ? want : cap);
}

}  // namespace

int watershed(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w,
              int32_t ws_h, uint8_t* sep, int32_t* basin) {
  const int64_t n = h * w;
  uint16_t* dq = ctx->u16a;
  uint16_t* F = ctx->u16b;
  prof_mark(ctx, RTG_STAGE_EDT);
  RTG_TRY(edt(ctx, mask, h, w, nullptr, dq, F, ws_h));
  prof_mark(ctx, RTG_STAGE_MARKERS);
  RTG_TRY(iwpp_recon_u16(ctx, F, dq, h, w, 8));  // HMAX
  uint16_t* Fw = ctx->u16a;                       // dq is dead now
  k_ws_prep<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, mask, F, Fw);
  RTG_LAUNCH("k_ws_prep");
  prof_mark(ctx, RTG_STAGE_WATERSHED);
  int32_t* ptr = ctx->i32a;
  int32_t* delta = ctx->i32b;
  int32_t* flat_count = ctx->misc + 1;
  RTG_CUDA(cudaMemsetAsync(flat_count, 0, sizeof(int32_t), ctx->stream));
  const dim3 grid2d((unsigned)ceil_div(w, 256), (unsigned)(h < 1024 ? h : 1024));
  k_ws_arrows<<<grid2d, 256, 0, ctx->stream>>>((int)h, (int)w, Fw, ctx->rm, ptr, delta,
                                               ctx->flat_list, flat_count);
  RTG_LAUNCH("k_ws_arrows");
  {
    // plateau BFS; unreached plateau pixels become the markers (rm)
    int32_t* flags = ctx->misc + 16;                              // 2 round flags
    unsigned* bar = reinterpret_cast<unsigned*>(ctx->misc + 20);  // barrier arrive/gen
    RTG_CUDA(cudaMemsetAsync(ctx->misc + 16, 0, sizeof(int32_t) * 8, ctx->stream));
    int hh = (int)h, ww = (int)w;
    const int32_t* flat = ctx->flat_list;
    uint8_t* rm = ctx->rm;
    void* args[] = {&hh, &ww, &Fw, &flat, &flat_count, &delta, &ptr, &rm, &flags, &bar};
    // one 256-thread CTA per SM: co-resident by construction, and guaranteed
    // so by the cooperative launch
    RTG_CUDA(cudaLaunchCooperativeKernel((const void*)k_ws_plateau, dim3(ctx->num_sms),
                                         dim3(256), args, 0, ctx->stream));
    RTG_LAUNCH("k_ws_plateau");
  }
  int32_t* mroots = ctx->i32c;
  RTG_TRY(ccl_roots(ctx, ctx->rm, h, w, 8, mroots));
  k_ws_resolve<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, mask, ptr, mroots, basin);
  RTG_LAUNCH("k_ws_resolve");
  k_ws_separate<<<grid2d, 256, 0, ctx->stream>>>((int)h, (int)w, basin, sep);
  RTG_LAUNCH("k_ws_separate");
  return RTG_OK;
}

}  // namespace rtg
