// o6 PreWatershed + o7 Watershed.
//
// Markers: F = HMAX_ws_h(dq) by IWPP reconstruction, Fw = fg ? F + 1 : 0;
// the markers are the regional maxima of Fw.
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
// Plateaus without a grid-wide BFS: "flat" pixels (no higher neighbour) form
// plateau components — adjacent flat pixels always share a level, since a
// flat pixel has no higher neighbour — which are labelled by union-find.  A
// component is a regional maximum (a marker, labelled by its minimum index,
// which is what a CCL of the marker mask would give) iff none of its pixels
// touches a same-level non-flat pixel ("seed", distance 1).  Only the other
// components need distances; each is small and is solved by one warp.
//
// Roofline: HBM/L2 bound; algorithmic bytes mask 1 B in + sep 1 B + basin 4 B
// out (dq/markers/Fw are internal planes).
#include "common.cuh"

namespace rtg {
namespace {

constexpr int32_t kInfD = 1 << 30;
constexpr int32_t kSeeded = 1 << 30;  // plateau root flag in the count word
constexpr int32_t kCountMask = kSeeded - 1;

__global__ void k_ws_prep(int64_t n, const uint8_t* __restrict__ mask,
                          const uint16_t* __restrict__ F, uint16_t* __restrict__ Fw) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    Fw[i] = (uint16_t)(mask[i] ? (uint32_t)F[i] + 1u : 0u);
}

// Arrows, one CTA per 32x32 tile with a 2-pixel halo of Fw in shared memory.
// Non-flat pixels: steepest ascent (par = -1).  Flat pixels: par = self,
// cnt = 0, appended to the flat list; a flat pixel with a same-level non-flat
// neighbour is a seed (distance 1) and points at the first such neighbour in
// row-major order (the minimum index), every other flat pixel gets ptr = -2.
// rm is cleared everywhere (markers are set by k_ws_classify).
__global__ void __launch_bounds__(256)
k_ws_arrows(int h, int w, const uint16_t* __restrict__ Fw, uint8_t* __restrict__ rm,
            int32_t* __restrict__ ptr, int32_t* __restrict__ par, int32_t* __restrict__ cnt,
            int32_t* __restrict__ flat_list, int32_t* __restrict__ flat_count) {
  __shared__ uint16_t sf[36][36];
  __shared__ uint8_t shi[34][36];
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int tid = threadIdx.x;
  const int lane = tid & 31, wr = tid >> 5;
  // stage rows of 32 (+4) contiguous values per warp: no index division
  {
    // all loads first (independent, in flight together), then the stores
    uint16_t va[5], vb[5];
    const int x = x0 - 2 + lane, x2 = x0 + 30 + lane;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int yy = wr + 8 * j, y = y0 - 2 + yy;
      const bool yin = yy < 36 && y >= 0 && y < h;
      const int64_t rb = (int64_t)y * w;
      va[j] = (yin && x >= 0 && x < w) ? __ldg(Fw + rb + x) : (uint16_t)0;
      vb[j] = (yin && lane < 4 && x2 < w) ? __ldg(Fw + rb + x2) : (uint16_t)0;
    }
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int yy = wr + 8 * j;
      if (yy < 36) {
        sf[yy][lane] = va[j];
        if (lane < 4) sf[yy][32 + lane] = vb[j];
      }
    }
  }
  __syncthreads();
  // "has a higher neighbour" for the tile and its 1-pixel ring (foreground
  // only: background never matches a foreground level)
  auto hi_at = [&](int yy, int xx) -> uint8_t {
    const uint32_t f = sf[yy][xx];
    if (!f) return 0;
    return sf[yy - 1][xx - 1] > f || sf[yy - 1][xx] > f || sf[yy - 1][xx + 1] > f ||
           sf[yy][xx - 1] > f || sf[yy][xx + 1] > f || sf[yy + 1][xx - 1] > f ||
           sf[yy + 1][xx] > f || sf[yy + 1][xx + 1] > f;
  };
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const int yy = 1 + wr + 8 * j;
    if (yy <= 34) {
      shi[yy - 1][lane] = hi_at(yy, lane + 1);
      if (lane < 2) shi[yy - 1][32 + lane] = hi_at(yy, 33 + lane);
    }
  }
  __syncthreads();
  const int c = lane;
  int32_t mine[4];
  int nmine = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = wr + 8 * q;
    const int y = y0 + r, x = x0 + c;
    if (y < h && x < w) {
      const int64_t i = (int64_t)y * w + x;
      const uint32_t f = sf[r + 2][c + 2];
      rm[i] = 0;
      if (f) {
        int32_t p = -2;
        if (shi[r + 1][c + 1]) {
          uint32_t best = f;
          int arg = 0;
#pragma unroll
          for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx) {
              const uint32_t fj = sf[r + 2 + dy][c + 2 + dx];
              if (fj > best) { best = fj; arg = dy * w + dx; }  // first max = min index
            }
          p = (int32_t)(i + arg);
          par[i] = -1;
        } else {
#pragma unroll
          for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx)
              if (p == -2 && sf[r + 2 + dy][c + 2 + dx] == f && shi[r + 1 + dy][c + 1 + dx])
                p = (int32_t)(i + dy * w + dx);
          par[i] = (int32_t)i;
          cnt[i] = 0;
          mine[nmine++] = (int32_t)i;
        }
        ptr[i] = p;
      }
    }
  }
  __shared__ int32_t sm[9];
  int32_t base = block_reserve(nmine, flat_count, sm);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (q < nmine) flat_list[base + q] = mine[q];
}

// Plateau components: union with the backward same-level flat neighbours
// (a neighbour is flat iff par >= 0).
__global__ void k_ws_union(int h, int w, const uint16_t* __restrict__ Fw,
                           const int32_t* __restrict__ flat_list,
                           const int32_t* __restrict__ flat_count, int32_t* par) {
  const int n = *flat_count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t i = flat_list[k];
    const int y = i / w, x = i - y * w;
    const uint16_t f = Fw[i];
    if (y > 0) {
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int xx = x + dx;
        if (xx < 0 || xx >= w) continue;
        const int32_t j = i - w + dx;
        if (Fw[j] == f && __ldcg(par + j) >= 0) uf_unite_g(par, i, j);
      }
    }
    if (x > 0 && Fw[i - 1] == f && __ldcg(par + i - 1) >= 0) uf_unite_g(par, i, i - 1);
  }
}

// Flattens every flat pixel onto its root, flags seeded roots and hands each
// pixel a slot in its component (slot stored in the delta plane).
__global__ void k_ws_roots(const int32_t* __restrict__ flat_list,
                           const int32_t* __restrict__ flat_count,
                           const int32_t* __restrict__ ptr, int32_t* par, int32_t* cnt,
                           int32_t* __restrict__ slot) {
  const int n = *flat_count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t i = flat_list[k];
    const int32_t r = uf_find_g(par, i);
    if (r != i) atomicMin(par + i, r);
    if (ptr && ptr[i] >= 0) atomicOr(cnt + r, kSeeded);
    slot[i] = atomicAdd(cnt + r, 1) & kCountMask;
  }
}

// Unseeded components are the markers (rm = 1, ptr = self; the root is the
// marker label).  Each seeded root reserves its members' range and enters the
// component list.  alloc = {member cursor, component count} as one u64.
__global__ void __launch_bounds__(256)
k_ws_classify(const int32_t* __restrict__ flat_list, const int32_t* __restrict__ flat_count,
              const int32_t* __restrict__ par, int32_t* cnt, int32_t* __restrict__ ptr,
              uint8_t* __restrict__ rm, unsigned long long* alloc,
              int32_t* __restrict__ comp_root, int32_t* __restrict__ comp_size) {
  __shared__ unsigned long long sm[9];
  const int n = *flat_count;
  for (int k0 = blockIdx.x * blockDim.x; k0 < n; k0 += gridDim.x * blockDim.x) {
    const int k = k0 + threadIdx.x;
    int32_t root = -1, sz = 0;
    if (k < n) {
      const int32_t i = flat_list[k];
      const int32_t r = __ldcg(par + i);
      const int32_t v = __ldcg(cnt + r);
      if (!(v & kSeeded)) {
        rm[i] = 1;
        ptr[i] = i;
      } else if (r == i) {
        root = i;
        sz = v & kCountMask;
      }
    }
    const unsigned long long slot = block_reserve2(root >= 0 ? 1u : 0u, (uint32_t)sz, alloc, sm);
    if (root >= 0) {
      const int32_t base = (int32_t)(slot & 0xFFFFFFFFull), c = (int32_t)(slot >> 32);
      __stcg(cnt + root, kSeeded | base);  // members still read the flag: it stays set
      comp_root[c] = root;
      comp_size[c] = sz;
    }
  }
}

__global__ void k_ws_scatter(const int32_t* __restrict__ flat_list,
                             const int32_t* __restrict__ flat_count,
                             const int32_t* __restrict__ par, const int32_t* __restrict__ cnt,
                             const int32_t* __restrict__ slot, int32_t* __restrict__ members) {
  const int n = *flat_count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t i = flat_list[k];
    const int32_t v = cnt[par[i]];
    if (v & kSeeded) members[(v & kCountMask) + slot[i]] = i;
  }
}

// Same-plateau neighbour mask of p (bit t = row-major neighbour t of 8).
__device__ __forceinline__ uint32_t plateau_nbrs(int h, int w, const uint16_t* __restrict__ Fw,
                                                 const int32_t* __restrict__ par, int32_t p,
                                                 uint16_t f, int32_t r) {
  const int y = p / w, x = p - y * w;
  uint32_t m = 0;
  int t = 0;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      if (dy == 0 && dx == 0) continue;
      const int yy = y + dy, xx = x + dx;
      if (yy >= 0 && yy < h && xx >= 0 && xx < w) {
        const int32_t j = p + dy * w + dx;
        if (Fw[j] == f && __ldcg(par + j) == r) m |= 1u << t;
      }
      ++t;
    }
  return m;
}

__device__ __forceinline__ int32_t nbr_index(int w, int32_t p, int t) {
  const int k = t < 4 ? t : t + 1;  // skip the centre
  return p + (k / 3 - 1) * w + (k % 3 - 1);
}

// Plateau distances and arrows, one warp per seeded component: chaotic
// Bellman-Ford over the members (values only decrease and always equal some
// real path length, so the fixed point is the BFS distance), then every
// non-seed member points at its first (minimum-index) same-plateau neighbour
// at distance d - 1.  Up to 32 * kPer members are kept in registers; larger
// components re-derive their neighbour masks every pass.
__global__ void __launch_bounds__(256)
k_ws_plateau(int h, int w, const uint16_t* __restrict__ Fw, const int32_t* __restrict__ par,
             const int32_t* __restrict__ cnt, const int32_t* __restrict__ members,
             const int32_t* __restrict__ comp_root, const int32_t* __restrict__ comp_size,
             const unsigned long long* __restrict__ alloc, int32_t* __restrict__ ptr,
             int32_t* delta) {
  constexpr int kPer = 4;
  const int ncomp = (int)(*alloc >> 32);
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  volatile int32_t* vd = delta;
  for (int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < ncomp; c += warps) {
    const int32_t r = comp_root[c], sz = comp_size[c];
    const int32_t* mem = members + (cnt[r] & kCountMask);
    const uint16_t f = Fw[r];
    if (sz <= 32 * kPer) {
      int32_t px[kPer], d[kPer];
      uint32_t nb[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int k = lane + 32 * q;
        px[q] = -1;
        d[q] = kInfD;
        nb[q] = 0;
        if (k < sz) {
          px[q] = mem[k];
          d[q] = ptr[px[q]] >= 0 ? 1 : kInfD;
          nb[q] = plateau_nbrs(h, w, Fw, par, px[q], f, r);
          vd[px[q]] = d[q];
        }
      }
      __syncwarp();
      while (true) {
        bool changed = false;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          if (px[q] < 0 || d[q] == 1) continue;
          int32_t best = d[q];
          for (uint32_t m = nb[q]; m; m &= m - 1)
            best = min(best, vd[nbr_index(w, px[q], __ffs(m) - 1)] + 1);
          if (best < d[q]) {
            d[q] = best;
            vd[px[q]] = best;
            changed = true;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, changed)) break;
      }
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        if (px[q] < 0 || d[q] == 1) continue;
        for (uint32_t m = nb[q]; m; m &= m - 1) {
          const int32_t j = nbr_index(w, px[q], __ffs(m) - 1);
          if (vd[j] == d[q] - 1) { ptr[px[q]] = j; break; }
        }
      }
    } else {
      for (int k = lane; k < sz; k += 32) vd[mem[k]] = ptr[mem[k]] >= 0 ? 1 : kInfD;
      __syncwarp();
      while (true) {
        bool changed = false;
        for (int k = lane; k < sz; k += 32) {
          const int32_t p = mem[k];
          const int32_t dp = vd[p];
          if (dp == 1) continue;
          int32_t best = dp;
          for (uint32_t m = plateau_nbrs(h, w, Fw, par, p, f, r); m; m &= m - 1)
            best = min(best, vd[nbr_index(w, p, __ffs(m) - 1)] + 1);
          if (best < dp) {
            vd[p] = best;
            changed = true;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, changed)) break;
      }
      for (int k = lane; k < sz; k += 32) {
        const int32_t p = mem[k];
        const int32_t dp = vd[p];
        if (dp == 1) continue;
        for (uint32_t m = plateau_nbrs(h, w, Fw, par, p, f, r); m; m &= m - 1) {
          const int32_t j = nbr_index(w, p, __ffs(m) - 1);
          if (vd[j] == dp - 1) { ptr[p] = j; break; }
        }
      }
    }
  }
}

// ---- HMAX by sparse components ------------------------------------------------
// F = recon(max(dq - h, 0), dq).  A foreground pixel p with an 8-neighbour q,
// dq(q) >= dq(p) + h, keeps F(p) = dq(p): q's marker reaches p through two
// pixels >= dq(p), and F <= dq.  The remaining foreground pixels ("suspects")
// form small 8-connected components; within one, F is the reconstruction of
// the marker under dq with the component's fixed neighbours (F = dq, or 0 on
// background) as boundary values, so each component is independent and one
// warp iterates it to its fixed point.  Output: Fw = fg ? F + 1 : 0.
__global__ void __launch_bounds__(256)
k_hmax_init(int h, int w, const uint16_t* __restrict__ dq, int32_t ws_h,
            uint16_t* __restrict__ Fw, uint8_t* __restrict__ sflag, int32_t* __restrict__ par,
            int32_t* __restrict__ cnt, int32_t* __restrict__ list, int32_t* __restrict__ count) {
  __shared__ uint16_t sd[34][36];
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int tid = threadIdx.x;
  {
    const int lane = tid & 31, wr = tid >> 5;
    uint16_t va[5], vb[5];
    const int x = x0 - 1 + lane, x2 = x0 + 31 + lane;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int yy = wr + 8 * j, y = y0 - 1 + yy;
      const bool yin = yy < 34 && y >= 0 && y < h;
      const int64_t rb = (int64_t)y * w;
      va[j] = (yin && x >= 0 && x < w) ? __ldg(dq + rb + x) : (uint16_t)0;
      vb[j] = (yin && lane < 2 && x2 < w) ? __ldg(dq + rb + x2) : (uint16_t)0;
    }
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int yy = wr + 8 * j;
      if (yy < 34) {
        sd[yy][lane] = va[j];
        if (lane < 2) sd[yy][32 + lane] = vb[j];
      }
    }
  }
  __syncthreads();
  const int c = tid & 31;
  int32_t mine[4];
  int nmine = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = (tid >> 5) + 8 * q;
    const int y = y0 + r, x = x0 + c;
    if (y < h && x < w) {
      const int64_t i = (int64_t)y * w + x;
      const int32_t v = sd[r + 1][c + 1];
      uint32_t fw = 0;
      bool sus = false;
      if (v) {
        int32_t mx = 0;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) mx = max(mx, (int32_t)sd[r + dy][c + dx]);
        if (mx >= v + ws_h) {
          fw = (uint32_t)v + 1u;
        } else {
          sus = true;
          fw = (uint32_t)(v > ws_h ? v - ws_h : 0) + 1u;
          par[i] = (int32_t)i;
          cnt[i] = 0;
          mine[nmine++] = (int32_t)i;
        }
      }
      Fw[i] = (uint16_t)fw;
      sflag[i] = sus;
    }
  }
  __shared__ int32_t sm[9];
  int32_t base = block_reserve(nmine, count, sm);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (q < nmine) list[base + q] = mine[q];
}

__global__ void k_hmax_union(int h, int w, const uint8_t* __restrict__ sflag,
                             const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                             int32_t* par) {
  const int n = *count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t i = list[k];
    const int y = i / w, x = i - y * w;
    if (y > 0) {
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int xx = x + dx;
        if (xx >= 0 && xx < w && sflag[i - w + dx]) uf_unite_g(par, i, i - w + dx);
      }
    }
    if (x > 0 && sflag[i - 1]) uf_unite_g(par, i, i - 1);
  }
}

// Every component root reserves its members' range (cnt[r] := kSeeded | base,
// the form k_ws_scatter reads) and enters the component list.
__global__ void __launch_bounds__(256)
k_hmax_alloc(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
             const int32_t* __restrict__ par, int32_t* cnt, unsigned long long* alloc,
             int32_t* __restrict__ comp_root, int32_t* __restrict__ comp_size) {
  __shared__ unsigned long long sm[9];
  const int n = *count;
  for (int k0 = blockIdx.x * blockDim.x; k0 < n; k0 += gridDim.x * blockDim.x) {
    const int k = k0 + threadIdx.x;
    int32_t i = -1, sz = 0;
    if (k < n) {
      i = list[k];
      if (__ldcg(par + i) == i) sz = __ldcg(cnt + i) & kCountMask;
      else i = -1;
    }
    const unsigned long long slot = block_reserve2(i >= 0 ? 1u : 0u, (uint32_t)sz, alloc, sm);
    if (i >= 0) {
      const int32_t base = (int32_t)(slot & 0xFFFFFFFFull), c = (int32_t)(slot >> 32);
      cnt[i] = kSeeded | base;
      comp_root[c] = i;
      comp_size[c] = sz;
    }
  }
}

// Neighbour summary of suspect p: bit t set = row-major neighbour t is a
// suspect (same component); fixed = max F over the other neighbours.
__device__ __forceinline__ uint32_t hmax_nbrs(int h, int w, const uint16_t* __restrict__ dq,
                                              const uint8_t* __restrict__ sflag, int32_t p,
                                              int32_t& fixed) {
  const int y = p / w, x = p - y * w;
  uint32_t m = 0;
  int t = 0;
  fixed = 0;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      if (dy == 0 && dx == 0) continue;
      const int yy = y + dy, xx = x + dx;
      if (yy >= 0 && yy < h && xx >= 0 && xx < w) {
        const int32_t j = p + dy * w + dx;
        if (sflag[j]) m |= 1u << t;
        else fixed = max(fixed, (int32_t)dq[j]);
      }
      ++t;
    }
  return m;
}

__global__ void __launch_bounds__(256)
k_hmax_solve(int h, int w, const uint16_t* __restrict__ dq, const uint8_t* __restrict__ sflag,
             int32_t ws_h, const int32_t* __restrict__ cnt, const int32_t* __restrict__ members,
             const int32_t* __restrict__ comp_root, const int32_t* __restrict__ comp_size,
             const unsigned long long* __restrict__ alloc, uint16_t* Fw) {
  constexpr int kPer = 4;
  const int ncomp = (int)(*alloc >> 32);
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  volatile uint16_t* vf = Fw;
  for (int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < ncomp; c += warps) {
    const int32_t r = comp_root[c], sz = comp_size[c];
    const int32_t* mem = members + (cnt[r] & kCountMask);
    if (sz <= 32 * kPer) {
      int32_t px[kPer], d[kPer], f[kPer];
      uint32_t nb[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int k = lane + 32 * q;
        px[q] = -1;
        d[q] = f[q] = 0;
        nb[q] = 0;
        if (k < sz) {
          px[q] = mem[k];
          d[q] = dq[px[q]];
          int32_t fixed;
          nb[q] = hmax_nbrs(h, w, dq, sflag, px[q], fixed);
          f[q] = min(d[q], max(d[q] > ws_h ? d[q] - ws_h : 0, fixed));
          vf[px[q]] = (uint16_t)(f[q] + 1);
        }
      }
      __syncwarp();
      while (true) {
        bool changed = false;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          if (px[q] < 0 || f[q] == d[q]) continue;
          int32_t best = f[q];
          for (uint32_t m = nb[q]; m; m &= m - 1)
            best = max(best, (int32_t)vf[nbr_index(w, px[q], __ffs(m) - 1)] - 1);
          best = min(best, d[q]);
          if (best > f[q]) {
            f[q] = best;
            vf[px[q]] = (uint16_t)(best + 1);
            changed = true;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, changed)) break;
      }
    } else {
      for (int k = lane; k < sz; k += 32) {
        const int32_t p = mem[k];
        const int32_t dp = dq[p];
        int32_t fixed;
        hmax_nbrs(h, w, dq, sflag, p, fixed);
        vf[p] = (uint16_t)(min(dp, max(dp > ws_h ? dp - ws_h : 0, fixed)) + 1);
      }
      __syncwarp();
      while (true) {
        bool changed = false;
        for (int k = lane; k < sz; k += 32) {
          const int32_t p = mem[k];
          const int32_t dp = dq[p], fp = (int32_t)vf[p] - 1;
          if (fp == dp) continue;
          int32_t fixed;
          int32_t best = fp;
          for (uint32_t m = hmax_nbrs(h, w, dq, sflag, p, fixed); m; m &= m - 1)
            best = max(best, (int32_t)vf[nbr_index(w, p, __ffs(m) - 1)] - 1);
          best = min(best, dp);
          if (best > fp) {
            vf[p] = (uint16_t)(best + 1);
            changed = true;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, changed)) break;
      }
    }
  }
}

// Basins + separation in one tiled pass: every pixel of the tile and its
// 1-pixel ring follows its arrows to the marker (basin = 1 + marker root),
// kept in shared memory; a pixel survives the separation unless an
// 8-neighbour has a higher basin id.  basin (optional) receives the ids.
__global__ void __launch_bounds__(256)
k_ws_basins(int h, int w, const uint8_t* __restrict__ mask, const int32_t* __restrict__ ptr,
            const int32_t* __restrict__ par, int32_t* __restrict__ basin,
            uint8_t* __restrict__ sep) {
  __shared__ int32_t sb[34][35];
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, wr = threadIdx.x >> 5;
  auto resolve = [&](int y, int x) -> int32_t {
    if (y < 0 || y >= h || x < 0 || x >= w) return 0;
    int32_t q = y * w + x;
    if (!mask[q]) return 0;
    int32_t nx = ptr[q];
    while (nx >= 0 && nx != q) {
      q = nx;
      nx = ptr[q];
    }
    return nx == q ? par[q] + 1 : 0;
  };
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const int yy = wr + 8 * j;
    if (yy < 34) {
      sb[yy][lane] = resolve(y0 - 1 + yy, x0 - 1 + lane);
      if (lane < 2) sb[yy][32 + lane] = resolve(y0 - 1 + yy, x0 + 31 + lane);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = wr + 8 * q;
    const int y = y0 + r, x = x0 + lane;
    if (y >= h || x >= w) continue;
    const int32_t b = sb[r + 1][lane + 1];
    const bool keep = b > 0 && sb[r][lane] <= b && sb[r][lane + 1] <= b && sb[r][lane + 2] <= b &&
                      sb[r + 1][lane] <= b && sb[r + 1][lane + 2] <= b &&
                      sb[r + 2][lane] <= b && sb[r + 2][lane + 1] <= b && sb[r + 2][lane + 2] <= b;
    const int64_t i = (int64_t)y * w + x;
    sep[i] = keep;
    if (basin) basin[i] = b;
  }
}

int grid_for(rtg_ctx* ctx, int64_t n) {
  const int64_t want = ceil_div(n, 256);
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  return (int)(want < cap ? want : cap);
}

}  // namespace

int watershed(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w,
              int32_t ws_h, uint8_t* sep, int32_t* basin, bool want_basin) {
  const int64_t n = h * w;
  uint16_t* dq = ctx->u16a;
  uint16_t* F = ctx->u16b;
  prof_mark(ctx, RTG_STAGE_EDT);
  const bool iwpp_hmax = ctx->hmax_impl == 1;
  RTG_TRY(edt(ctx, mask, h, w, nullptr, dq, iwpp_hmax ? F : nullptr, ws_h));
  prof_mark(ctx, RTG_STAGE_MARKERS);
  uint16_t* Fw;
  const int g = ctx->num_sms * 8;
  // component lists (root, size): the arena holds 16 B per pixel
  int32_t* comp_root = reinterpret_cast<int32_t*>(ctx->arena);
  int32_t* comp_size = comp_root + n;
  auto* alloc = reinterpret_cast<unsigned long long*>(ctx->misc + 16);
  if (iwpp_hmax) {
    RTG_TRY(iwpp_recon_u16(ctx, F, dq, h, w, 8));  // HMAX
    Fw = ctx->u16a;                                 // dq is dead now
    k_ws_prep<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, mask, F, Fw);
    RTG_LAUNCH("k_ws_prep");
  } else {
    Fw = F;
    int32_t* list = ctx->flat_list;
    int32_t* count = ctx->misc + 1;
    int32_t* par = ctx->i32c;
    int32_t* slot = ctx->i32b;
    uint8_t* sflag = ctx->m1;
    RTG_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), ctx->stream));
    RTG_CUDA(cudaMemsetAsync(alloc, 0, sizeof(unsigned long long), ctx->stream));
    const dim3 tiles((unsigned)ceil_div(w, 32), (unsigned)ceil_div(h, 32));
    k_hmax_init<<<tiles, 256, 0, ctx->stream>>>((int)h, (int)w, dq, ws_h, Fw, sflag, par, basin,
                                                list, count);
    RTG_LAUNCH("k_hmax_init");
    k_hmax_union<<<g, 256, 0, ctx->stream>>>((int)h, (int)w, sflag, list, count, par);
    RTG_LAUNCH("k_hmax_union");
    k_ws_roots<<<g, 256, 0, ctx->stream>>>(list, count, nullptr, par, basin, slot);
    RTG_LAUNCH("k_ws_roots");
    k_hmax_alloc<<<g, 256, 0, ctx->stream>>>(list, count, par, basin, alloc, comp_root,
                                             comp_size);
    RTG_LAUNCH("k_hmax_alloc");
    k_ws_scatter<<<g, 256, 0, ctx->stream>>>(list, count, par, basin, slot, ctx->lroots);
    RTG_LAUNCH("k_ws_scatter");
    k_hmax_solve<<<g, 256, 0, ctx->stream>>>((int)h, (int)w, dq, sflag, ws_h, basin,
                                             ctx->lroots, comp_root, comp_size, alloc, Fw);
    RTG_LAUNCH("k_hmax_solve");
  }
  prof_mark(ctx, RTG_STAGE_WATERSHED);
  int32_t* ptr = ctx->i32a;
  int32_t* delta = ctx->i32b;
  int32_t* par = ctx->i32c;
  int32_t* flat_count = ctx->misc + 1;
  RTG_CUDA(cudaMemsetAsync(flat_count, 0, sizeof(int32_t), ctx->stream));
  RTG_CUDA(cudaMemsetAsync(alloc, 0, sizeof(unsigned long long), ctx->stream));
  const dim3 tiles((unsigned)ceil_div(w, 32), (unsigned)ceil_div(h, 32));
  k_ws_arrows<<<tiles, 256, 0, ctx->stream>>>((int)h, (int)w, Fw, ctx->rm, ptr, par, basin,
                                              ctx->flat_list, flat_count);
  RTG_LAUNCH("k_ws_arrows");
  k_ws_union<<<g, 256, 0, ctx->stream>>>((int)h, (int)w, Fw, ctx->flat_list, flat_count, par);
  RTG_LAUNCH("k_ws_union");
  k_ws_roots<<<g, 256, 0, ctx->stream>>>(ctx->flat_list, flat_count, ptr, par, basin, delta);
  RTG_LAUNCH("k_ws_roots");
  k_ws_classify<<<g, 256, 0, ctx->stream>>>(ctx->flat_list, flat_count, par, basin, ptr, ctx->rm,
                                            alloc, comp_root, comp_size);
  RTG_LAUNCH("k_ws_classify");
  k_ws_scatter<<<g, 256, 0, ctx->stream>>>(ctx->flat_list, flat_count, par, basin, delta,
                                           ctx->lroots);
  RTG_LAUNCH("k_ws_scatter");
  k_ws_plateau<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>((int)h, (int)w, Fw, par, basin,
                                                          ctx->lroots, comp_root, comp_size,
                                                          alloc, ptr, delta);
  RTG_LAUNCH("k_ws_plateau");
  k_ws_basins<<<tiles, 256, 0, ctx->stream>>>((int)h, (int)w, mask, ptr, par,
                                              want_basin ? basin : nullptr, sep);
  RTG_LAUNCH("k_ws_basins");
  return RTG_OK;
}

}  // namespace rtg
