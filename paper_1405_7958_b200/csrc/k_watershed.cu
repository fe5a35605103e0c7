// o6 PreWatershed + o7 Watershed.
//
// Markers: F = HMAX_ws_h(dq), Fw = fg ? F + 1 : 0; the markers are the
// regional maxima of Fw.
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
// Sparse execution: only foreground pixels carry work (about 15% of a
// tissue tile), so every pass runs over the foreground list built from the
// mask (fg_list) instead of over the tile; neighbour reads are gated by the
// mask bytes, so planes are never cleared for background pixels.
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
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    Fw[i] = (uint16_t)(mask[i] ? (uint32_t)F[i] + 1u : 0u);
}

__device__ __forceinline__ int32_t nbr_index(int w, int32_t p, int t) {
  const int k = t < 4 ? t : t + 1;  // skip the centre
  return p + (k / 3 - 1) * w + (k % 3 - 1);
}

// Watershed arrows are stored as one byte per pixel: the code of the
// 8-neighbour it points to, (dy + 1) * 4 + (dx + 1), so a chain step is
// q + ((c >> 2) & 3) * w + (c & 3) - (w + 1); kDirSelf (the zero offset) = a
// marker pixel (root), kDirNone = no arrow yet.  A byte
// plane keeps the basin chains' gathers 4x denser than i32 indices.
constexpr uint8_t kDirSelf = 5;
constexpr uint8_t kDirNone = 0xF5;  // decodes, masked, to the zero offset too

__device__ __forceinline__ uint8_t dir_code(int t) {  // row-major neighbour t of 8
  return (uint8_t)((0xA9864210u >> (4 * t)) & 0xFu);
}

// The 8 neighbour values selected by mask m (others = fill), as unrolled
// predicated loads so all of them are in flight together (a loop over the
// set bits would serialise one memory latency per neighbour).
template <typename T, typename S>
__device__ __forceinline__ void gather8(const T* a, int w, int32_t p, uint32_t m, S fill,
                                        S (&v)[8]) {
#pragma unroll
  for (int t = 0; t < 8; ++t) v[t] = ((m >> t) & 1u) ? (S)a[nbr_index(w, p, t)] : fill;
}

// Backward unions (k_ws_union, k_hmax_union): p joins its backward
// 8-neighbours of the same component (above-left, above, above-right, left),
// skipping the ones a neighbour's own unions already imply: the left neighbour (when joined)
// has already joined the above-left and above pixels, and two horizontally
// adjacent same-component pixels above are joined with each other.  Every
// component stays connected; the number of union-find operations (and the
// chain lengths they build) drops from up to four per pixel to about one.

// Arrows over the foreground list.  Non-flat pixels: steepest ascent (flat
// byte 0).  Flat pixels: flat byte 1, appended to the flat list at slot k
// (fmap[p] = k, parK[k] = k, cntK[k] = 0); their seed arrow is set by
// k_ws_union.
__global__ void __launch_bounds__(256)
k_ws_arrows(int h, FastDiv dw, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
            const uint32_t* __restrict__ mask, const uint8_t* __restrict__ nbm,
            const uint16_t* __restrict__ Fw,
            uint8_t* __restrict__ dir, int32_t* __restrict__ fmap, int32_t* __restrict__ parK,
            int32_t* __restrict__ cntK, uint8_t* __restrict__ flat, int32_t* __restrict__ flat_list,
            int32_t* __restrict__ flat_count, uint8_t* __restrict__ eqm) {
  pdl_enter();
  const int w = (int)dw.d;
  __shared__ int32_t sm[9];
  const int n = *count;
  for (int k0 = blockIdx.x * blockDim.x; k0 < n; k0 += gridDim.x * blockDim.x) {
    const int k = k0 + threadIdx.x;
    bool is_flat = false;
    int32_t p = 0;
    uint32_t eq = 0;  // foreground neighbours at p's level
    if (k < n) {
      p = list[k];
      uint32_t fv[8];
      const uint32_t fm = list_nbrs(h, dw, mask, nbm, k, p);
      gather8(Fw, w, p, fm, 0u, fv);
      // steepest ascent as one max over keys value << 3 | (7 - t): the first
      // (row-major) maximum wins ties, and p's own key (f << 3 | 7) beats
      // every neighbour at its level or below
      const uint32_t self = (uint32_t)Fw[p] << 3 | 7u;
      uint32_t best = self;
#pragma unroll
      for (int t = 0; t < 8; ++t) best = max(best, fv[t] << 3 | (7u - t));
#pragma unroll
      for (int t = 0; t < 8; ++t) eq |= (((fm >> t) & 1u) && fv[t] == (self >> 3) ? 1u : 0u) << t;
      if (best != self) {
        dir[p] = dir_code(7 - (int)(best & 7u));
        flat[p] = 0;
      } else {
        dir[p] = kDirNone;
        flat[p] = 1;
        is_flat = true;
      }
    }
    const int32_t slot = block_reserve_flag(is_flat, flat_count, sm);
    if (is_flat) {
      // the plateau machinery runs on compact flat-pixel slots
      flat_list[slot] = p;
      fmap[p] = slot;
      parK[slot] = slot;
      cntK[slot] = 0;
      eqm[slot] = (uint8_t)eq;  // same-level neighbours: the plateau kernels' only gather
    }
  }
}

// Union-find over compact slots whose root is the slot of the smallest
// PIXEL index (keys = the flat list): a marker keeps the label a CCL of the
// marker mask would give it (its minimum pixel).  Roots are linked by CAS,
// larger key under smaller, so keys strictly decrease towards a root.
__device__ __forceinline__ int32_t ukey_find(int32_t* par, int32_t a) {
  int32_t p = __ldcg(par + a);
  while (p != a) {
    const int32_t gp = __ldcg(par + p);
    if (gp != p) par[a] = gp;  // halving: an ancestor replaces the parent
    a = p;
    p = gp;
  }
  return a;
}
__device__ __forceinline__ void ukey_unite(int32_t* par, const int32_t* __restrict__ key,
                                           int32_t a, int32_t b) {
  while (true) {
    a = ukey_find(par, a);
    b = ukey_find(par, b);
    if (a == b) return;
    if (__ldg(key + a) < __ldg(key + b)) { const int32_t t = a; a = b; b = t; }
    if (atomicCAS(par + a, a, b) == a) return;  // a was still a root
  }
}

// Flat pixels: the seed arrow (first row-major same-level non-flat
// neighbour: distance 1) and plateau unions with the backward same-level flat
// neighbours.
__global__ void k_ws_union(int w, const uint8_t* __restrict__ flat,
                           const int32_t* __restrict__ flat_list,
                           const int32_t* __restrict__ flat_count, uint8_t* __restrict__ dir,
                           const int32_t* __restrict__ fmap, int32_t* parK,
                           const uint8_t* __restrict__ eqm) {
  pdl_enter();
  const int n = *flat_count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t i = flat_list[k];
    int seed = -1;
    const uint32_t eq = eqm[k];  // same-level neighbours (k_ws_arrows)
    uint32_t fl[8];
    gather8(flat, w, i, eq, 1u, fl);
    uint32_t same = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (!((eq >> t) & 1u)) continue;
      if (!fl[t]) {
        if (seed < 0) seed = t;
      } else if (t < 4) {  // backward neighbour (above or left)
        same |= 1u << t;
      }
    }
    // unite_backward's skips, on compact slots (fmap: pixel -> slot)
    const bool ul = same & 1u, u = same & 2u, ur = same & 4u, l = same & 8u;
    if (l) {
      ukey_unite(parK, flat_list, k, __ldg(fmap + i - 1));
      if (ur && !u) ukey_unite(parK, flat_list, k, __ldg(fmap + i - w + 1));
    } else if (u) {
      ukey_unite(parK, flat_list, k, __ldg(fmap + i - w));
    } else {
      if (ul) ukey_unite(parK, flat_list, k, __ldg(fmap + i - w - 1));
      if (ur) ukey_unite(parK, flat_list, k, __ldg(fmap + i - w + 1));
    }
    if (seed >= 0) dir[i] = dir_code(seed);
  }
}

// Compact plateau roots: flatten, seeded flags, a slot per member.  The find
// is read-only: slots are not key-ordered, so a halving store (unlike the
// pixel forests' atomicMin) could overwrite an already flattened parent with
// a stale ancestor.
__global__ void k_ws_roots_c(const int32_t* __restrict__ flat_list,
                             const int32_t* __restrict__ flat_count,
                             const uint8_t* __restrict__ dir, int32_t* parK, int32_t* cntK,
                             int32_t* __restrict__ slot) {
  pdl_enter();
  const int n = *flat_count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    int32_t r = k, p = __ldcg(parK + k);
    while (p != r) {
      r = p;
      p = __ldcg(parK + p);
    }
    if (r != k) parK[k] = r;
    if (dir[flat_list[k]] != kDirNone) atomicOr(cntK + r, kSeeded);
    slot[k] = atomicAdd(cntK + r, 1) & kCountMask;
  }
}

// Unseeded components are the markers (arrow = kDirSelf; the root is the marker
// label).  Each seeded root reserves its members' range and enters the
// component list.  alloc = {member cursor, component count} as one u64.
__global__ void __launch_bounds__(256)
k_ws_classify(const int32_t* __restrict__ flat_list, const int32_t* __restrict__ flat_count,
              const int32_t* __restrict__ parK, int32_t* cntK, uint8_t* __restrict__ dir,
              int32_t* __restrict__ parP, unsigned long long* alloc) {
  pdl_enter();
  __shared__ unsigned long long sm[9];
  const int n = *flat_count;
  for (int k0 = blockIdx.x * blockDim.x; k0 < n; k0 += gridDim.x * blockDim.x) {
    const int k = k0 + threadIdx.x;
    int32_t root = -1, sz = 0;
    if (k < n) {
      const int32_t i = flat_list[k];
      const int32_t r = __ldcg(parK + k);
      const int32_t v = __ldcg(cntK + r);
      if (!(v & kSeeded)) {
        // a marker: its label is its root's pixel (the minimum), read by
        // k_ws_basins at the marker pixels
        dir[i] = kDirSelf;
        parP[i] = __ldg(flat_list + r);
      } else if (r == k) {
        root = k;
        sz = v & kCountMask;
      }
    }
    const unsigned long long slot = block_reserve2(root >= 0 ? 1u : 0u, (uint32_t)sz, alloc, sm);
    if (root >= 0) {
      const int32_t base = (int32_t)(slot & 0xFFFFFFFFull);
      __stcg(cntK + root, kSeeded | base);  // members still read the flag: it stays set
    }
  }
}

// Members of the seeded components, back to back by component (compact).
__global__ void k_ws_scatter_c(const int32_t* __restrict__ flat_list,
                               const int32_t* __restrict__ flat_count,
                               const int32_t* __restrict__ parK, const int32_t* __restrict__ cntK,
                               const int32_t* __restrict__ slot, int32_t* __restrict__ members) {
  pdl_enter();
  const int n = *flat_count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t v = cntK[parK[k]];
    if (v & kSeeded) {
      const int32_t sl = slot[k], i = flat_list[k];
      members[(v & kCountMask) + sl] = sl == 0 ? ~i : i;  // ~: first member of a component
    }
  }
}

// Same-plateau neighbour mask of p (bit t = row-major neighbour t of 8): the
// flat neighbours at p's level.  That is exactly its plateau component's
// neighbours, since k_ws_union unites every such pair.
__device__ __forceinline__ uint32_t plateau_nbrs(int w, const uint8_t* __restrict__ flat,
                                                 const int32_t* __restrict__ fmap,
                                                 const uint8_t* __restrict__ eqm, int32_t p) {
  const uint32_t eq = eqm[__ldg(fmap + p)];  // p's same-level neighbours (k_ws_arrows)
  uint32_t fl[8];
  gather8(flat, w, p, eq, 0u, fl);
  uint32_t cand = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (fl[t]) cand |= 1u << t;
  return cand;
}

// Components are laid out back to back in `members` (component order), each
// flagged at its first entry (~pixel).  Warp chunk [w0, w0 + 32) takes every
// component that STARTS in it — a whole number of small components per warp,
// so a warp-wide convergence test is exact and tiny components share a warp.
// Returns false when no component starts in the chunk; else [s0, e).
__device__ __forceinline__ bool packed_range(const int32_t* __restrict__ members, int nmem,
                                             int w0, int lane, int& s0, int& e) {
  const unsigned full = 0xFFFFFFFFu;
  const int k = w0 + lane;
  const unsigned st = __ballot_sync(full, k < nmem && members[k] < 0);
  if (!st) return false;
  s0 = w0 + __ffs(st) - 1;
  e = nmem;
  for (int b = w0 + 32; b < nmem; b += 32) {
    const int kk = b + lane;
    const unsigned nx = __ballot_sync(full, kk < nmem && members[kk] < 0);
    if (nx) {
      e = b + __ffs(nx) - 1;
      break;
    }
  }
  return true;
}

__device__ __forceinline__ int32_t member_px(int32_t m) { return m < 0 ? ~m : m; }

// Plateau distances and arrows over packed components: chaotic Bellman-Ford
// over the members (values only decrease and always equal some real path
// length, so the fixed point is the BFS distance), then every non-seed member
// points at its first (minimum-index) same-plateau neighbour at distance
// d - 1.  Up to 32 * kPer members per warp in registers; longer ranges
// re-derive their neighbour masks every pass.
__global__ void __launch_bounds__(256)
k_ws_plateau(int w, const uint8_t* __restrict__ flat, const int32_t* __restrict__ fmap,
             const uint8_t* __restrict__ eqm,
             const int32_t* __restrict__ members, const unsigned long long* __restrict__ alloc,
             uint8_t* __restrict__ dir, int32_t* delta, int2* __restrict__ scratch,
             uint8_t* slotmap) {
  pdl_enter();
  constexpr int kPer = 4;
  // small ranges relax in shared memory (distances by slot, neighbour slots)
  __shared__ int32_t s_val[8][32 * kPer];
  __shared__ uint8_t s_nbs[8][32 * kPer][8];
  const int nmem = (int)(*alloc & 0xFFFFFFFFull);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  volatile int32_t* vd = delta;
  volatile int32_t* sv = s_val[wl];
  for (int w0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < nmem;
       w0 += nwarps * 32) {
    int s0, e;
    if (!packed_range(members, nmem, w0, lane, s0, e)) continue;
    if (e - s0 <= 32 * kPer) {
      int32_t px[kPer], d[kPer];
      uint32_t nb[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int k = s0 + lane + 32 * q;
        px[q] = -1;
        d[q] = kInfD;
        nb[q] = 0;
        if (k < e) {
          px[q] = member_px(members[k]);
          d[q] = dir[px[q]] != kDirNone ? 1 : kInfD;
          nb[q] = plateau_nbrs(w, flat, fmap, eqm, px[q]);
          sv[lane + 32 * q] = d[q];
          slotmap[px[q]] = (uint8_t)(lane + 32 * q);
        }
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        if (px[q] < 0) continue;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if ((nb[q] >> t) & 1u) s_nbs[wl][lane + 32 * q][t] = slotmap[nbr_index(w, px[q], t)];
      }
      __syncwarp();
      while (true) {
        bool changed = false;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          if (px[q] < 0 || d[q] == 1) continue;
          const uint8_t* ns = s_nbs[wl][lane + 32 * q];
          int32_t best = d[q];
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if ((nb[q] >> t) & 1u) best = min(best, sv[ns[t]] + 1);
          if (best < d[q]) {
            d[q] = best;
            sv[lane + 32 * q] = best;
            changed = true;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, changed)) break;
      }
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        if (px[q] < 0 || d[q] == 1) continue;
        const uint8_t* ns = s_nbs[wl][lane + 32 * q];
#pragma unroll
        for (int t = 7; t >= 0; --t)  // the first (minimum-index) match wins
          if (((nb[q] >> t) & 1u) && sv[ns[t]] == d[q] - 1) dir[px[q]] = dir_code(t);
      }
      __syncwarp();
    } else {
      // long range: per-member (pixel, neighbour mask) cached in scratch
      for (int k = s0 + lane; k < e; k += 32) {
        const int32_t p = member_px(members[k]);
        vd[p] = dir[p] != kDirNone ? 1 : kInfD;
        scratch[k] = make_int2(p, (int32_t)plateau_nbrs(w, flat, fmap, eqm, p));
      }
      __syncwarp();
      while (true) {
        bool changed = false;
        for (int k = s0 + lane; k < e; k += 32) {
          const int2 pm = scratch[k];
          const int32_t dp = vd[pm.x];
          if (dp == 1) continue;
          int32_t dv[8];
          gather8(vd, w, pm.x, (uint32_t)pm.y, kInfD, dv);
          int32_t best = dp;
#pragma unroll
          for (int t = 0; t < 8; ++t) best = min(best, dv[t] + 1);
          if (best < dp) {
            vd[pm.x] = best;
            changed = true;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, changed)) break;
      }
      for (int k = s0 + lane; k < e; k += 32) {
        const int2 pm = scratch[k];
        const int32_t dp = vd[pm.x];
        if (dp == 1) continue;
        int32_t dv[8];
        gather8(vd, w, pm.x, (uint32_t)pm.y, kInfD, dv);
#pragma unroll
        for (int t = 7; t >= 0; --t)
          if (dv[t] == dp - 1) dir[pm.x] = dir_code(t);
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
k_hmax_init(int h, FastDiv dw, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
            const uint32_t* __restrict__ mask, const uint8_t* __restrict__ nbm,
            const uint16_t* __restrict__ dq, int32_t ws_h,
            uint16_t* __restrict__ Fw, uint8_t* __restrict__ sflag, int32_t* __restrict__ par,
            int32_t* __restrict__ cnt, int32_t* __restrict__ slist,
            int32_t* __restrict__ scount, int32_t* __restrict__ smap,
            uint8_t* __restrict__ smask) {
  pdl_enter();
  const int w = (int)dw.d;
  __shared__ int32_t sm[9];
  const int n = *count;
  for (int k0 = blockIdx.x * blockDim.x; k0 < n; k0 += gridDim.x * blockDim.x) {
    const int k = k0 + threadIdx.x;
    bool sus = false;
    int32_t p = 0;
    uint32_t fm = 0;
    if (k < n) {
      p = list[k];
      const int32_t v = dq[p];
      int32_t dv[8];
      fm = list_nbrs(h, dw, mask, nbm, k, p);
      gather8(dq, w, p, fm, 0, dv);
      int32_t mx = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) mx = max(mx, dv[t]);
      if (mx >= v + ws_h) {
        Fw[p] = (uint16_t)(v + 1);
        sflag[p] = 0;
      } else {
        sus = true;
        Fw[p] = (uint16_t)((v > ws_h ? v - ws_h : 0) + 1);
        sflag[p] = 1;
      }
    }
    const int32_t slot = block_reserve_flag(sus, scount, sm);
    if (sus) {
      // the component machinery runs on compact suspect indices (slot k):
      // its forest and counters stay a few hundred KB, L2-resident
      slist[slot] = p;
      smap[p] = slot;
      par[slot] = slot;
      cnt[slot] = 0;
      smask[slot] = (uint8_t)fm;  // foreground neighbours: no bit-plane tests downstream
    }
  }
}

__global__ void k_hmax_union(int w, const uint8_t* __restrict__ sflag,
                             const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                             const int32_t* __restrict__ smap, int32_t* par,
                             const uint8_t* __restrict__ smask) {
  pdl_enter();
  const int n = *count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t i = list[k];
    // backward neighbours only (bits 0..3: above row and left)
    uint32_t sv[8];
    gather8(sflag, w, i, smask[k] & 0xFu, 0u, sv);
    // unite_backward's skips, on compact indices (smap: pixel -> suspect slot)
    const bool ul = sv[0], u = sv[1], ur = sv[2], l = sv[3];
    if (l) {
      uf_unite_g(par, k, __ldg(smap + i - 1));
      if (ur && !u) uf_unite_g(par, k, __ldg(smap + i - w + 1));
    } else if (u) {
      uf_unite_g(par, k, __ldg(smap + i - w));
    } else {
      if (ul) uf_unite_g(par, k, __ldg(smap + i - w - 1));
      if (ur) uf_unite_g(par, k, __ldg(smap + i - w + 1));
    }
  }
}

// Roots / slots / member placement of the compact suspect forest (the HMAX
// counterparts of k_ws_roots_c / k_ws_scatter_c, indexed by suspect slot).
__global__ void k_hmax_roots(const int32_t* __restrict__ count, int32_t* par, int32_t* cnt,
                             int32_t* __restrict__ slot) {
  pdl_enter();
  const int n = *count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t r = uf_find_g(par, k);
    if (r != k) atomicMin(par + k, r);
    slot[k] = atomicAdd(cnt + r, 1) & kCountMask;
  }
}

__global__ void k_hmax_scatter(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                               const int32_t* __restrict__ par, const int32_t* __restrict__ cnt,
                               const int32_t* __restrict__ slot, int32_t* __restrict__ members) {
  pdl_enter();
  const int n = *count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t v = cnt[par[k]];
    const int32_t sl = slot[k], i = list[k];
    members[(v & kCountMask) + sl] = sl == 0 ? ~i : i;  // ~: first member of a component
  }
}

// Every component root reserves its members' range (cnt[r] := kSeeded | base,
// the form k_ws_scatter_c reads) and enters the component list.
__global__ void __launch_bounds__(256)
k_hmax_alloc(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
             const int32_t* __restrict__ par, int32_t* cnt, unsigned long long* alloc) {
  pdl_enter();
  __shared__ unsigned long long sm[9];
  const int n = *count;
  for (int k0 = blockIdx.x * blockDim.x; k0 < n; k0 += gridDim.x * blockDim.x) {
    const int k = k0 + threadIdx.x;
    int32_t i = -1, sz = 0;  // compact: i = suspect slot k when it is a root
    if (k < n && __ldcg(par + k) == k) {
      i = k;
      sz = __ldcg(cnt + k) & kCountMask;
    }
    const unsigned long long slot = block_reserve2(i >= 0 ? 1u : 0u, (uint32_t)sz, alloc, sm);
    if (i >= 0) {
      const int32_t base = (int32_t)(slot & 0xFFFFFFFFull);
      cnt[i] = kSeeded | base;
    }
  }
}

// Neighbour summary of suspect p: bit t set = row-major neighbour t is a
// suspect (same component); fixed = max F over the other neighbours.
__device__ __forceinline__ uint32_t hmax_nbrs(int w, const int32_t* __restrict__ smap,
                                              const uint8_t* __restrict__ smask,
                                              const uint16_t* __restrict__ dq,
                                              const uint8_t* __restrict__ sflag, int32_t p,
                                              int32_t& fixed) {
  const uint32_t fm = smask[__ldg(smap + p)];  // k_hmax_init's foreground-neighbour mask
  uint32_t sv[8];
  int32_t dv[8];
  gather8(sflag, w, p, fm, 0u, sv);
  gather8(dq, w, p, fm, 0, dv);
  uint32_t m = 0;
  fixed = 0;  // background neighbours: F = 0
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (sv[t]) m |= 1u << t;
    else fixed = max(fixed, dv[t]);
  }
  return m;
}

__global__ void __launch_bounds__(256)
k_hmax_solve(int w, const int32_t* __restrict__ smap, const uint8_t* __restrict__ smask,
             const uint16_t* __restrict__ dq, const uint8_t* __restrict__ sflag, int32_t ws_h,
             const int32_t* __restrict__ members, const unsigned long long* __restrict__ alloc,
             uint16_t* Fw, int2* __restrict__ scratch, uint8_t* slotmap) {
  pdl_enter();
  constexpr int kPer = 4;
  // small ranges iterate in shared memory: member values by slot (index in
  // the warp's range) and each member's neighbour slots, so a relaxation
  // sweep costs shared-memory latency instead of an L2 round trip
  __shared__ int32_t s_val[8][32 * kPer];
  __shared__ uint8_t s_nbs[8][32 * kPer][8];
  const int nmem = (int)(*alloc & 0xFFFFFFFFull);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  volatile uint16_t* vf = Fw;
  volatile int32_t* sv = s_val[wl];
  for (int w0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < nmem;
       w0 += nwarps * 32) {
    int s0, e;
    if (!packed_range(members, nmem, w0, lane, s0, e)) continue;
    if (e - s0 <= 32 * kPer) {
      int32_t px[kPer], d[kPer], f[kPer];
      uint32_t nb[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int k = s0 + lane + 32 * q;
        px[q] = -1;
        d[q] = f[q] = 0;
        nb[q] = 0;
        if (k < e) {
          px[q] = member_px(members[k]);
          d[q] = dq[px[q]];
          int32_t fixed;
          nb[q] = hmax_nbrs(w, smap, smask, dq, sflag, px[q], fixed);
          f[q] = min(d[q], max(d[q] > ws_h ? d[q] - ws_h : 0, fixed));
          sv[lane + 32 * q] = f[q];
          slotmap[px[q]] = (uint8_t)(lane + 32 * q);
        }
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        if (px[q] < 0) continue;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if ((nb[q] >> t) & 1u) s_nbs[wl][lane + 32 * q][t] = slotmap[nbr_index(w, px[q], t)];
      }
      __syncwarp();
      while (true) {
        bool changed = false;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          if (px[q] < 0 || f[q] == d[q]) continue;
          int32_t best = f[q];
          const uint8_t* ns = s_nbs[wl][lane + 32 * q];
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if ((nb[q] >> t) & 1u) best = max(best, sv[ns[t]]);  // s_val holds F (not F + 1)
          best = min(best, d[q]);
          if (best > f[q]) {
            f[q] = best;
            sv[lane + 32 * q] = best;
            changed = true;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, changed)) break;
      }
#pragma unroll
      for (int q = 0; q < kPer; ++q)
        if (px[q] >= 0) Fw[px[q]] = (uint16_t)(f[q] + 1);
      __syncwarp();
    } else {
      // long range: per-member (pixel, neighbour mask | dq << 8) cached in scratch
      for (int k = s0 + lane; k < e; k += 32) {
        const int32_t p = member_px(members[k]);
        const int32_t dp = dq[p];
        int32_t fixed;
        const uint32_t nbm = hmax_nbrs(w, smap, smask, dq, sflag, p, fixed);
        vf[p] = (uint16_t)(min(dp, max(dp > ws_h ? dp - ws_h : 0, fixed)) + 1);
        scratch[k] = make_int2(p, (int32_t)(nbm | ((uint32_t)dp << 8)));
      }
      __syncwarp();
      while (true) {
        bool changed = false;
        for (int k = s0 + lane; k < e; k += 32) {
          const int2 pm = scratch[k];
          const int32_t dp = (int32_t)((uint32_t)pm.y >> 8), fp = (int32_t)vf[pm.x] - 1;
          if (fp == dp) continue;
          int32_t fv[8];
          gather8(vf, w, pm.x, (uint32_t)pm.y & 0xFFu, 0, fv);
          int32_t best = fp;
#pragma unroll
          for (int t = 0; t < 8; ++t) best = max(best, fv[t] - 1);
          best = min(best, dp);
          if (best > fp) {
            vf[pm.x] = (uint16_t)(best + 1);
            changed = true;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, changed)) break;
      }
    }
  }
}

// Basin of every listed pixel: follow the arrows to the marker (basin = 1 +
// marker root).
// Four chains per thread followed in lockstep, so four dependent loads are
// in flight per step instead of one (the kernel is latency-bound: every
// step of an arrow chain is a dependent L2 load).
__global__ void __launch_bounds__(256)
k_ws_basins(int w, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
            const uint8_t* __restrict__ dir, const int32_t* __restrict__ par,
            int32_t* __restrict__ basin) {
  pdl_enter();
  constexpr int kC = 4;
  // the step of every code (index c & 15): one shared load per step instead
  // of the decode arithmetic
  __shared__ int32_t s_off[16];
  if (threadIdx.x < 16) {
    const int c = (int)threadIdx.x;
    s_off[c] = ((c >> 2) & 3) * w + (c & 3) - (w + 1);
  }
  __syncthreads();
  const int n = *count;
  const int span = gridDim.x * blockDim.x * kC;
  for (int k0 = blockIdx.x * blockDim.x * kC + threadIdx.x; k0 < n; k0 += span) {
    int32_t p[kC], q[kC];
    uint32_t d[kC];
#pragma unroll
    for (int j = 0; j < kC; ++j) {
      const int k = k0 + j * (int)blockDim.x;
      p[j] = k < n ? list[k] : -1;
    }
#pragma unroll
    for (int j = 0; j < kC; ++j) {
      q[j] = p[j] >= 0 ? p[j] : p[0];  // a spare slot walks a real chain
      d[j] = dir[q[j]];
    }
    // Codes decode with (c >> 2) & 3, under which kDirSelf and kDirNone are
    // both the zero offset: a finished chain stays put, so the chains take
    // kSteps steps between convergence tests with no per-step predicate.
    constexpr int kSteps = 4;
    auto moving = [](uint32_t c) { return c != kDirSelf && c != kDirNone; };
    while (true) {
      bool any = false;
#pragma unroll
      for (int j = 0; j < kC; ++j) any |= moving(d[j]);
      if (!any) break;
#pragma unroll
      for (int s = 0; s < kSteps; ++s) {
#pragma unroll
        for (int j = 0; j < kC; ++j) {
          q[j] += s_off[d[j] & 15u];
          d[j] = dir[q[j]];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kC; ++j)
      if (p[j] >= 0) basin[p[j]] = d[j] == kDirSelf ? par[q[j]] + 1 : 0;
  }
}

// Separation: a listed pixel survives unless an 8-neighbour has a higher
// basin id (background pixels of sep are cleared beforehand).  With
// sep_bits (cleared by the joint fill/area stage) the result goes into that
// 1-bit plane instead: the lanes of a warp that share a word OR their bits
// together and one of them issues the atomic (the list is row-ordered, so a
// warp touches one or two words).
__global__ void k_ws_separate(int h, FastDiv dw, const int32_t* __restrict__ list,
                              const int32_t* __restrict__ count,
                              const uint32_t* __restrict__ mask, const uint8_t* __restrict__ nbm,
                              const int32_t* __restrict__ basin, uint8_t* __restrict__ sep,
                              uint32_t* __restrict__ sep_bits) {
  pdl_enter();
  const int w = (int)dw.d;
  const int n = *count;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count (the bit path's match/reduce needs every lane)
  for (int k0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; k0 < n;
       k0 += gridDim.x * blockDim.x) {
    const int k = k0 + lane;
    int32_t p = -1;
    bool keep = false;
    if (k < n) {
      p = list[k];
      const int32_t b = basin[p];
      int32_t bv[8];
      gather8(basin, w, p, list_nbrs(h, dw, mask, nbm, k, p), 0, bv);
      keep = b > 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) keep &= bv[t] <= b;
      if (!sep_bits) sep[p] = keep;
    }
    if (sep_bits) {
      // the list holds each bit word's pixels back to back (fg_list appends a
      // word's set bits together), so the lanes sharing a word are a run of
      // lanes: its bounds come from a ballot of run heads (no match_any)
      const int32_t wi = p >= 0 ? (p >> 5) : -1;
      const int32_t wprev = __shfl_up_sync(0xFFFFFFFFu, wi, 1);
      const uint32_t heads = __ballot_sync(0xFFFFFFFFu, lane == 0 || wprev != wi);
      const uint32_t upto = lane == 31 ? 0xFFFFFFFFu : (2u << lane) - 1u;
      const int first = 31 - __clz(heads & upto);
      const uint32_t after = heads & ~upto;
      const uint32_t grp = (after ? (after & (0u - after)) - 1u : 0xFFFFFFFFu) & ~((1u << first) - 1u);
      const uint32_t v = __reduce_or_sync(grp, keep ? 1u << (p & 31) : 0u);
      if (wi >= 0 && v && lane == first) atomicOr(sep_bits + wi, v);
    }
  }
}

int grid_for(rtg_ctx* ctx, int64_t n) {
  const int64_t want = ceil_div(n, 256);
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  return (int)(want < cap ? want : cap);
}

}  // namespace

int watershed(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w,
              int32_t ws_h, uint8_t* sep, int32_t* basin, bool want_basin, bool list_ready) {
  const int64_t n = h * w;
  uint16_t* dq = ctx->u16a;
  uint16_t* F = ctx->u16b;
  const int g = ctx->num_sms * 8;
  const FastDiv dwv = make_div((uint32_t)w);
  int32_t* fgl = ctx->fg_list;
  int32_t* fgn = ctx->misc + 4;  // foreground count

  // per-member cache of long component ranges (the arena's second half)
  int2* member_scratch = reinterpret_cast<int2*>(ctx->arena + 8 * n);
  // counters of the whole o6/o7 chain, zeroed here in one launch: misc[1]
  // HMAX suspect count, misc[2..3] EDT flags (edt_list), misc[5] flat-pixel
  // count, misc[16..17] HMAX component allocator, misc[18..19] plateau one
  // (misc[4], the foreground count, was built by the caller or fg_list)
  auto* alloc = reinterpret_cast<unsigned long long*>(ctx->misc + 16);
  auto* walloc = reinterpret_cast<unsigned long long*>(ctx->misc + 18);
  // ... and, in the same launch, what the labelling of the separated mask
  // (o8, ccl_roots(..., prezeroed)) needs cleared
  // (the separated mask itself only when it is written as bytes; the bit
  // plane was cleared by the joint fill/area stage)
  const bool sep_bits = ctx->sep_bits_live && list_ready;  // only the stage path sets it
  ZeroList z{{ctx->misc + 1, ctx->misc + 5, alloc, sep},
             {3 * sizeof(int32_t), sizeof(int32_t), 2 * sizeof(unsigned long long), (size_t)n},
             sep_bits ? 3 : 4};
  ccl_label_zero(ctx, h, w, z);
  RTG_TRY(zero_async(ctx, z));
  if (want_basin)
    RTG_TRY(zero_async(ctx, ZeroList{{basin}, {sizeof(int32_t) * (size_t)n}, 1}));
  prof_mark(ctx, RTG_STAGE_EDT);
  if (!list_ready) RTG_TRY(fg_list(ctx, mask, h, w, fgl, fgn, ctx->fg_bits));
  const uint32_t* fgbits = ctx->fg_bits + kBitPad;  // neighbour tests of the list kernels
  const bool iwpp_hmax = ctx->hmax_impl == 1;
  // 8-neighbour masks of the listed pixels, by list index (k_edt_rowdist
  // builds them; the recon plane is dead by now); the IWPP HMAX path has
  // no list EDT and recomputes them
  uint8_t* nbm = iwpp_hmax ? nullptr : ctx->recon;
  if (iwpp_hmax) {
    RTG_TRY(edt(ctx, mask, h, w, nullptr, dq, F, ws_h));  // every pixel (IWPP reads all)
  } else {
    // the joint stage's mask bytes double as the row-distance plane
    RTG_TRY(edt_list(ctx, h, w, fgl, fgn, ctx->fg_bits, dq, nbm,
                     list_ready && ctx->mask_bytes_live ? const_cast<uint8_t*>(mask) : nullptr));
  }
  prof_mark(ctx, RTG_STAGE_MARKERS);
  uint16_t* Fw;
  if (iwpp_hmax) {
    RTG_TRY(iwpp_recon_u16(ctx, F, dq, h, w, 8));  // HMAX
    Fw = ctx->u16a;                                 // dq is dead now
    RTG_CUDA(launch_k(ctx, k_ws_prep, grid_for(ctx, n), 256, 0, n, mask, F, Fw));
    RTG_LAUNCH("k_ws_prep");
  } else {
    Fw = F;
    int32_t* list = ctx->flat_list;
    int32_t* count = ctx->misc + 1;
    int32_t* par = ctx->i32c;
    int32_t* slot = ctx->i32b;
    uint8_t* sflag = ctx->m1;
    int32_t* smap = ctx->i32a;  // pixel -> suspect slot (the label plane is dead here)
    // compact counters in the arena's first half (the basin plane may be the
    // caller's output, whose background must stay as cleared)
    int32_t* hcnt = reinterpret_cast<int32_t*>(ctx->arena);
    uint8_t* smask = reinterpret_cast<uint8_t*>(ctx->u16c);  // per suspect slot (EDT plane dead)
    RTG_CUDA(launch_k(ctx, k_hmax_init, g, 256, 0, (int)h, dwv, fgl, fgn, fgbits,
                      (const uint8_t*)nbm, dq, ws_h, Fw, sflag,
                                            par, hcnt, list, count, smap, smask));
    RTG_LAUNCH("k_hmax_init");
    RTG_CUDA(launch_k(ctx, k_hmax_union, g, 256, 0, (int)w, (const uint8_t*)sflag,
                      (const int32_t*)list, (const int32_t*)count, (const int32_t*)smap, par,
                      (const uint8_t*)smask));
    RTG_LAUNCH("k_hmax_union");
    RTG_CUDA(launch_k(ctx, k_hmax_roots, g, 256, 0, (const int32_t*)count, par, hcnt, slot));
    RTG_LAUNCH("k_hmax_roots");
    RTG_CUDA(launch_k(ctx, k_hmax_alloc, g, 256, 0, list, count, par, hcnt, alloc));
    RTG_LAUNCH("k_hmax_alloc");
    RTG_CUDA(launch_k(ctx, k_hmax_scatter, g, 256, 0, (const int32_t*)list, (const int32_t*)count,
                      (const int32_t*)par, (const int32_t*)hcnt, (const int32_t*)slot,
                      ctx->lroots));
    RTG_LAUNCH("k_hmax_scatter");
    RTG_CUDA(launch_k(ctx, k_hmax_solve, g, 256, 0, (int)w, (const int32_t*)smap,
                      (const uint8_t*)smask, (const uint16_t*)dq, (const uint8_t*)sflag, ws_h,
                      (const int32_t*)ctx->lroots, (const unsigned long long*)alloc, Fw,
                      member_scratch,
                                             ctx->m2 /* slot map: the EDT row distances are dead */));
    RTG_LAUNCH("k_hmax_solve");
  }
  prof_mark(ctx, RTG_STAGE_WATERSHED);
  uint8_t* dir = reinterpret_cast<uint8_t*>(ctx->i32a);  // arrow codes, 1 B/px
  int32_t* delta = ctx->i32b;
  int32_t* par = ctx->i32c;
  uint8_t* flat = ctx->m1;
  int32_t* flat_count = ctx->misc + 5;
  // compact plateau machinery: forest / counters in the arena's first half
  // (the HMAX ones there are dead), pixel -> slot map in the par plane, which
  // k_ws_classify then overwrites with each marker pixel's label for
  // k_ws_basins
  int32_t* parK = reinterpret_cast<int32_t*>(ctx->arena);
  int32_t* cntK = parK + n;
  uint8_t* eqm = reinterpret_cast<uint8_t*>(ctx->u16c);  // per flat slot (the EDT plane is dead)
  RTG_CUDA(launch_k(ctx, k_ws_arrows, g, 256, 0, (int)h, dwv, fgl, fgn, fgbits,
                    (const uint8_t*)nbm, Fw, dir, par, parK, cntK, flat, ctx->flat_list,
                    flat_count, eqm));
  RTG_LAUNCH("k_ws_arrows");
  RTG_CUDA(launch_k(ctx, k_ws_union, g, 256, 0, (int)w, (const uint8_t*)flat,
                    (const int32_t*)ctx->flat_list, (const int32_t*)flat_count, dir,
                    (const int32_t*)par, parK, (const uint8_t*)eqm));
  RTG_LAUNCH("k_ws_union");
  RTG_CUDA(launch_k(ctx, k_ws_roots_c, g, 256, 0, (const int32_t*)ctx->flat_list, flat_count,
                    (const uint8_t*)dir, parK, cntK, delta));
  RTG_LAUNCH("k_ws_roots_c");
  RTG_CUDA(launch_k(ctx, k_ws_classify, g, 256, 0, (const int32_t*)ctx->flat_list, flat_count,
                    (const int32_t*)parK, cntK, dir, par, walloc));
  RTG_LAUNCH("k_ws_classify");
  RTG_CUDA(launch_k(ctx, k_ws_scatter_c, g, 256, 0, (const int32_t*)ctx->flat_list, flat_count,
                    (const int32_t*)parK, (const int32_t*)cntK, (const int32_t*)delta,
                    ctx->lroots));
  RTG_LAUNCH("k_ws_scatter_c");
  RTG_CUDA(launch_k(ctx, k_ws_plateau, g, 256, 0, (int)w, (const uint8_t*)flat,
                    (const int32_t*)par /* pixel -> flat slot */, (const uint8_t*)eqm,
                    (const int32_t*)ctx->lroots, (const unsigned long long*)walloc, dir, delta,
                    member_scratch, ctx->m2 /* slot map */));
  RTG_LAUNCH("k_ws_plateau");
  RTG_CUDA(launch_k(ctx, k_ws_basins, g, 256, 0, (int)w, fgl, fgn, dir, par, basin));
  RTG_LAUNCH("k_ws_basins");
  RTG_CUDA(launch_k(ctx, k_ws_separate, g, 256, 0, (int)h, dwv, fgl, fgn, fgbits,
                    (const uint8_t*)nbm, basin, sep,
                    sep_bits ? ctx->sep_bits : (uint32_t*)nullptr));
  RTG_LAUNCH("k_ws_separate");
  return RTG_OK;
}

}  // namespace rtg
