// IWPP engine: grayscale reconstruction by dilation on a persistent
// tile-granular wavefront queue ("hierarchical and
// scalable queue to store and manage active elements").
//
// Work unit = one 32x32 tile, owned by one warp while it is processed.  The
// warp stages the tile (+1 px halo) in shared memory, runs alternating
// raster / anti-raster sweeps (down, up, right, left) to a local fixed point,
// writes it back, and enqueues exactly those neighbour tiles whose halo it
// raised.  A per-tile state machine (idle/queued/processing/dirty) guarantees
// one owner per tile; a global `pending` counter terminates the persistent
// grid without host round trips.
//
// When every tile starts active (grayscale reconstruction), the first visit
// of each tile is statically assigned (warp w takes tiles w, w+W, ...) instead
// of going through the queue, and pushes are batched per visit, so the hot
// queue counters only see the (much smaller) wavefront traffic.
//
// Reconstruction by dilation is the greatest fixed point below the mask
// reachable from the marker, so the result is independent of the order in
// which tiles and pixels are relaxed: stale halo reads only cost extra
// visits, never correctness (values only increase and stay <= the answer).
// Precondition: J <= I everywhere on entry (callers clip).
//
// Roofline: HBM/L2 bound; algorithmic bytes 3 B/px (u8: marker + mask in,
// result out) or 6 B/px (u16).  Revisits are the IWPP overhead.
#include "common.cuh"

namespace rtg {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kJS = 35;  // J tile stride (34 used: halo + 32 + halo)
constexpr int kIS = 33;  // I tile stride

struct WarpSmem {
  uint32_t J[34 * kJS];
  uint32_t I[32 * kIS];
};

template <typename T>
struct PlainMask {
  const T* I;
  __device__ __forceinline__ uint32_t operator()(int64_t i) const { return I[i]; }
};
// fill-holes: the reconstruction runs under the complement of a binary mask
struct ComplementMask {
  const uint8_t* bin;
  __device__ __forceinline__ uint32_t operator()(int64_t i) const {
    return bin[i] ? 0u : 1u;
  }
};

template <typename T>
__device__ __forceinline__ uint32_t ld_state(const T* p) {
  return (uint32_t)__ldcg(p);  // bypass L1: other warps update J
}
template <>
__device__ __forceinline__ uint32_t ld_state<uint8_t>(const uint8_t* p) {
  return (uint32_t)__ldcg(reinterpret_cast<const unsigned char*>(p));
}

// ---- queue primitives (lane 0 only) ----------------------------------------

// Marks tile t for processing.  Returns true when the caller must enqueue it
// (state went idle -> queued); a queued tile stays queued, a tile being
// processed is marked dirty (its owner re-runs it).
__device__ bool q_mark(const TileQueue& q, int32_t t) {
  int32_t s = atomicAdd(&q.state[t], 0);
  while (true) {
    if (s == 1 || s == 3) return false;
    if (s == 0) {
      const int32_t old = atomicCAS(&q.state[t], 0, 1);
      if (old == 0) return true;
      s = old;
    } else {
      const int32_t old = atomicCAS(&q.state[t], 2, 3);
      if (old == 2) return false;
      s = old;
    }
  }
}

// Publishes k marked tiles with one pending and one tail update.
__device__ void q_enqueue(const TileQueue& q, int32_t cap, const int32_t* ids, int k) {
  if (k == 0) return;
  atomicAdd(&q.counters[2], (uint32_t)k);  // pending, before publication
  const uint32_t pos = atomicAdd(&q.counters[1], (uint32_t)k);
  for (int i = 0; i < k; ++i) {
    int32_t* slot = &q.slots[(pos + (uint32_t)i) % (uint32_t)cap];
    while (atomicCAS(slot, 0, ids[i] + 1) != 0) __nanosleep(32);
  }
}

// Returns a tile id, or -1 when all work is done (or the run was aborted).
__device__ int32_t q_pop(const TileQueue& q, int32_t cap) {
  const uint32_t pos = atomicAdd(&q.counters[0], 1u);
  int32_t* slot = &q.slots[pos % (uint32_t)cap];
  while (true) {
    const int32_t v = atomicExch(slot, 0);
    if (v != 0) {
      atomicExch(&q.state[v - 1], 2);
      __threadfence();
      return v - 1;
    }
    if (*(volatile uint32_t*)&q.counters[2] == 0u) return -1;
    if (*(volatile uint32_t*)&q.counters[4] != 0u) return -1;
    __nanosleep(64);
  }
}

// Returns true when the tile must be processed again (it was marked dirty).
__device__ bool q_finish(const TileQueue& q, int32_t t) {
  const int32_t old = atomicCAS(&q.state[t], 2, 0);
  if (old == 2) {
    atomicSub(&q.counters[2], 1u);
    return false;
  }
  atomicExch(&q.state[t], 2);  // dirty -> processing again
  __threadfence();             // acquire the neighbour's fenced border writes
  return true;
}

// ---- one tile visit ------------------------------------------------------------

template <typename T, int CONN, class MaskF>
__device__ void visit_tile(int32_t t, T* __restrict__ J, const MaskF& maskf, int h, int w,
                           int tiles_x, const TileQueue& q, int32_t cap, uint32_t* Js,
                           uint32_t* Is, long long& visits, long long& iters,
                           bool static_visit) {
  const unsigned full = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const int ty = t / tiles_x, tx = t - ty * tiles_x;
  const int tiles_y = (h + kTile - 1) / kTile;
  const int y0 = ty * kTile, x0 = tx * kTile;
  const int x = x0 + lane;

  // fully unrolled: all 32 row loads of a lane are in flight at once (the
  // visit is latency-bound, not bandwidth-bound)
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const int y = y0 + r;
    Is[r * kIS + lane] = (y < h && x < w) ? maskf((int64_t)y * w + x) : 0u;
  }
  bool dirty_reload = false;
  do {
    bool tile_changed = false;
    // (re)load J: full tile on the first pass, halo only on a dirty reload
    if (!dirty_reload) {
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int y = y0 + r;
        uint32_t v = 0;
        if (y < h && x < w) {
          const uint32_t j = ld_state(J + (int64_t)y * w + x);
          const uint32_t m = Is[r * kIS + lane];
          v = j < m ? j : m;
          if (v != j) tile_changed = true;  // defensive: marker above the mask
        }
        Js[(r + 1) * kJS + lane + 1] = v;
      }
    }
    {
      const int yt = y0 - 1, yb = y0 + 32;
      Js[lane + 1] = (yt >= 0 && x < w) ? ld_state(J + (int64_t)yt * w + x) : 0u;
      Js[33 * kJS + lane + 1] = (yb < h && x < w) ? ld_state(J + (int64_t)yb * w + x) : 0u;
      for (int k = lane; k < 34; k += 32) {
        const int y = y0 - 1 + k;
        const bool yin = y >= 0 && y < h;
        Js[k * kJS + 0] = (yin && x0 > 0) ? ld_state(J + (int64_t)y * w + x0 - 1) : 0u;
        Js[k * kJS + 33] = (yin && x0 + 32 < w) ? ld_state(J + (int64_t)y * w + x0 + 32) : 0u;
      }
    }
    __syncwarp();
    const uint32_t top0 = Js[1 * kJS + lane + 1];
    const uint32_t bot0 = Js[32 * kJS + lane + 1];
    const uint32_t left0 = Js[(lane + 1) * kJS + 1];
    const uint32_t right0 = Js[(lane + 1) * kJS + 32];

    // a tile already at its upper bound (J == mask everywhere, e.g. an
    // all-background tile of a distance map) cannot change: skip the sweeps
    bool saturated = true;
    uint32_t rows_active = 0;  // rows with a pixel that has mask > 0
    bool col_active = false;
    for (int r = 0; r < 32; ++r) {
      const uint32_t m = Is[r * kIS + lane];
      saturated &= Js[(r + 1) * kJS + lane + 1] == m;
      col_active |= m != 0;
      rows_active |= __ballot_sync(full, m != 0) ? (1u << r) : 0u;
    }
    // sweeps only need the bounding box of the mask-positive pixels: every
    // other pixel has mask 0, so J == 0 there and it neither changes nor
    // feeds a neighbour
    const uint32_t cols_active = __ballot_sync(full, col_active);
    const int r0 = rows_active ? __ffs(rows_active) - 1 : 0;
    const int r1 = rows_active ? 31 - __clz(rows_active) : -1;
    const int c0 = cols_active ? __ffs(cols_active) - 1 : 0;
    const int c1 = cols_active ? 31 - __clz(cols_active) : -1;
    // Sweeps run cyclically (down, up, right, left).  A sweep leaves its own
    // relation satisfied, and a sweep that changes nothing certifies its
    // relation, so the tile is at its local fixed point once the three sweeps
    // after the last changing sweep were quiet (4 quiet sweeps if none ever
    // changed anything).
    if (!__all_sync(full, saturated)) {
      int quiet = 0, done = 0;
      for (int s = 0;; s = (s + 1) & 3) {
        bool ch = false;
        if (s == 0) {  // down: lane = column c, neighbours in the row above
          for (int r = r0; r <= r1; ++r) {
            uint32_t* row = Js + (r + 1) * kJS + lane + 1;
            const uint32_t* up = row - kJS;
            uint32_t n = up[0];
            if (CONN == 8) n = max(n, max(up[-1], up[1]));
            const uint32_t v = *row;
            const uint32_t nv = min(max(v, n), Is[r * kIS + lane]);
            if (nv != v) { *row = nv; ch = true; }
            __syncwarp();
          }
        } else if (s == 1) {  // up
          for (int r = r1; r >= r0; --r) {
            uint32_t* row = Js + (r + 1) * kJS + lane + 1;
            const uint32_t* dn = row + kJS;
            uint32_t n = dn[0];
            if (CONN == 8) n = max(n, max(dn[-1], dn[1]));
            const uint32_t v = *row;
            const uint32_t nv = min(max(v, n), Is[r * kIS + lane]);
            if (nv != v) { *row = nv; ch = true; }
            __syncwarp();
          }
        } else if (s == 2) {  // right: lane = row r, neighbours in the column left
          for (int c = c0; c <= c1; ++c) {
            uint32_t* px = Js + (lane + 1) * kJS + c + 1;
            const uint32_t* lf = px - 1;
            uint32_t n = lf[0];
            if (CONN == 8) n = max(n, max(lf[-kJS], lf[kJS]));
            const uint32_t v = *px;
            const uint32_t nv = min(max(v, n), Is[lane * kIS + c]);
            if (nv != v) { *px = nv; ch = true; }
            __syncwarp();
          }
        } else {  // left
          for (int c = c1; c >= c0; --c) {
            uint32_t* px = Js + (lane + 1) * kJS + c + 1;
            const uint32_t* rt = px + 1;
            uint32_t n = rt[0];
            if (CONN == 8) n = max(n, max(rt[-kJS], rt[kJS]));
            const uint32_t v = *px;
            const uint32_t nv = min(max(v, n), Is[lane * kIS + c]);
            if (nv != v) { *px = nv; ch = true; }
            __syncwarp();
          }
        }
        ++done;
        if (__any_sync(full, ch)) {
          tile_changed = true;
          quiet = 0;
        } else {
          ++quiet;
        }
        if ((quiet >= 3 && done > quiet) || quiet >= 4) break;
      }
      iters += (done + 3) / 4;
    }
    ++visits;
    tile_changed = __any_sync(full, tile_changed);
    if (tile_changed) {
#pragma unroll 4
      for (int r = 0; r < 32; ++r) {
        const int y = y0 + r;
        if (y < h && x < w) J[(int64_t)y * w + x] = (T)Js[(r + 1) * kJS + lane + 1];
      }
      __threadfence();
    }

    // which neighbours did we raise?  A border pixel must have changed in this
    // visit and exceed the neighbour's value we saw (stale halo only
    // over-approximates).  Diagonal neighbours need the corner itself to have
    // changed: static corner inequalities alone could cycle forever.
    bool pn = false, ps = false, pw = false, pe = false;
    if (tile_changed) {
      const uint32_t tv = Js[1 * kJS + lane + 1];
      const uint32_t bv = Js[32 * kJS + lane + 1];
      const uint32_t lv = Js[(lane + 1) * kJS + 1];
      const uint32_t rv = Js[(lane + 1) * kJS + 32];
      uint32_t nt = Js[lane + 1], nb = Js[33 * kJS + lane + 1];
      uint32_t nl = Js[(lane + 1) * kJS], nr = Js[(lane + 1) * kJS + 33];
      if (CONN == 8) {
        nt = min(nt, min(Js[lane], Js[lane + 2]));
        nb = min(nb, min(Js[33 * kJS + lane], Js[33 * kJS + lane + 2]));
        nl = min(nl, min(Js[lane * kJS], Js[(lane + 2) * kJS]));
        nr = min(nr, min(Js[lane * kJS + 33], Js[(lane + 2) * kJS + 33]));
      }
      pn = __any_sync(full, tv != top0 && tv > nt);
      ps = __any_sync(full, bv != bot0 && bv > nb);
      pw = __any_sync(full, lv != left0 && lv > nl);
      pe = __any_sync(full, rv != right0 && rv > nr);
    }
    const uint32_t c00_0 = __shfl_sync(full, top0, 0), c01_0 = __shfl_sync(full, top0, 31);
    const uint32_t c10_0 = __shfl_sync(full, bot0, 0), c11_0 = __shfl_sync(full, bot0, 31);
    int again = 0;
    if (lane == 0) {
      int32_t ids[8];
      int k = 0;
      auto mark = [&](bool cond, int32_t nt) {
        if (cond && q_mark(q, nt)) ids[k++] = nt;
      };
      mark(pn && ty > 0, t - tiles_x);
      mark(ps && ty + 1 < tiles_y, t + tiles_x);
      mark(pw && tx > 0, t - 1);
      mark(pe && tx + 1 < tiles_x, t + 1);
      if (CONN == 8 && tile_changed) {
        const uint32_t c00 = Js[1 * kJS + 1], c01 = Js[1 * kJS + 32];
        const uint32_t c10 = Js[32 * kJS + 1], c11 = Js[32 * kJS + 32];
        mark(ty > 0 && tx > 0 && c00 != c00_0 && c00 > Js[0], t - tiles_x - 1);
        mark(ty > 0 && tx + 1 < tiles_x && c01 != c01_0 && c01 > Js[33], t - tiles_x + 1);
        mark(ty + 1 < tiles_y && tx > 0 && c10 != c10_0 && c10 > Js[33 * kJS], t + tiles_x - 1);
        mark(ty + 1 < tiles_y && tx + 1 < tiles_x && c11 != c11_0 && c11 > Js[33 * kJS + 33],
             t + tiles_x + 1);
      }
      if (static_visit) {
        // colour-phase pass: marked tiles (state 1) are collected into the
        // queue by k_queue_build afterwards; no hot counters touched here
        const int32_t old = atomicCAS(&q.state[t], 2, 0);
        if (old != 2) {
          atomicExch(&q.state[t], 2);
          __threadfence();
          again = 1;
        }
      } else {
        q_enqueue(q, cap, ids, k);
        again = q_finish(q, t) ? 1 : 0;
      }
    }
    again = __shfl_sync(full, again, 0);
    dirty_reload = again != 0;
  } while (dirty_reload);
}

// ---- the persistent kernel ---------------------------------------------------

template <typename T, int CONN, class MaskF>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 3)
k_iwpp(T* __restrict__ J, MaskF maskf, int h, int w, int tiles_x, int ntiles,
       int phase, TileQueue q, int32_t cap, int64_t* kstats, uint32_t max_visits,
       uint32_t* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem& S = reinterpret_cast<WarpSmem*>(smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xFFFFFFFFu;
  long long my_visits = 0, charged = 0, my_iters = 0;

  // budget: a bug that livelocks the queue must not hang the GPU; exceeding
  // it aborts every warp and raises a sticky status bit
  auto over_budget = [&]() -> bool {
    int bad = 0;
    if (lane == 0 && my_visits - charged >= 32) {
      const uint32_t prev = atomicAdd(&q.counters[3], (uint32_t)(my_visits - charged));
      charged = my_visits;
      if (prev > max_visits) {
        atomicExch(&q.counters[4], 1u);
        atomicOr(status, kStatusQueueOverflow);
        bad = 1;
      }
    }
    return __shfl_sync(full, bad, 0) != 0 ||
           *(volatile uint32_t*)&q.counters[4] != 0u;
  };

  if (phase >= 0) {
    // static pass over one checkerboard colour: tiles with (ty + tx) % 2 ==
    // phase share no edge, so each phase sees final-ish halos from the other
    // colour (diagonal neighbours may race: that only costs a revisit).  A
    // push only marks the neighbour (state 1); k_queue_build collects the
    // marked tiles and the phase == -1 launch drains them.
    const int tiles_y = (h + kTile - 1) / kTile;
    const int first = phase == 0 ? (tiles_x + 1) / 2 : tiles_x / 2;  // in even rows
    const int count = (tiles_y / 2) * tiles_x + ((tiles_y & 1) ? first : 0);
    const int warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * kWarpsPerBlock;
    for (int k = warp; k < count; k += nwarps) {
      // k enumerates row pairs (2r, 2r+1): `first` tiles of colour `phase`
      // in the even row, then the rest in the odd row
      const int rp = k / tiles_x, rem = k - rp * tiles_x;
      const int ty = 2 * rp + (rem < first ? 0 : 1);
      const int tx = rem < first ? phase + 2 * rem : (phase ^ 1) + 2 * (rem - first);
      const int t = ty * tiles_x + tx;
      if (lane == 0) {
        atomicExch(&q.state[t], 2);
        __threadfence();
      }
      __syncwarp();
      visit_tile<T, CONN>(t, J, maskf, h, w, tiles_x, q, cap, S.J, S.I, my_visits, my_iters,
                          true);
      if (over_budget()) break;
    }
  } else while (true) {
    int32_t t = 0;
    if (lane == 0) t = q_pop(q, cap);
    t = __shfl_sync(full, t, 0);
    if (t < 0) break;
    visit_tile<T, CONN>(t, J, maskf, h, w, tiles_x, q, cap, S.J, S.I, my_visits, my_iters,
                        false);
    if (over_budget()) break;
  }
  if (lane == 0 && kstats) {
    atomicAdd((unsigned long long*)&kstats[0], (unsigned long long)my_visits);
    atomicAdd((unsigned long long*)&kstats[1], (unsigned long long)my_iters);
  }
}

// Queue initialisation.  mode 0: every tile starts active (state queued,
// visited by the static first pass, nothing in the slot ring); mode 1: only
// border tiles, published in the slot ring.
// Tile states before a run: 1 ("to visit") for every tile when the colour
// phases visit them all, else for border tiles only (fill-holes seeds).
__global__ void k_tiles_init(TileQueue q, int tiles_y, int tiles_x, int border_only) {
  const int ntiles = tiles_y * tiles_x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
    const int ty = t / tiles_x, tx = t - ty * tiles_x;
    const bool take = !border_only || ty == 0 || tx == 0 || ty == tiles_y - 1 || tx == tiles_x - 1;
    q.state[t] = take ? 1 : 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    q.counters[3] = 0;  // visits (budget)
    q.counters[4] = 0;  // abort flag
  }
}

// Publishes every tile in state 1 (in tile order) into the slot ring and arms
// the queue counters for the draining launch.
__global__ void k_queue_build(TileQueue q, int32_t cap, int ntiles) {
  __shared__ int32_t count;
  __shared__ int32_t warp_cnt[32];
  if (threadIdx.x == 0) count = 0;
  __syncthreads();
  for (int base = 0; base < ntiles; base += blockDim.x) {
    const int t = base + threadIdx.x;
    const bool take = t < ntiles && q.state[t] == 1;
    // order-preserving compaction within the chunk
    const unsigned b = __ballot_sync(0xFFFFFFFFu, take);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) warp_cnt[wid] = __popc(b);
    __syncthreads();
    int off = 0;
    for (int k = 0; k < wid; ++k) off += warp_cnt[k];
    if (take) q.slots[count + off + __popc(b & ((1u << lane) - 1u))] = t + 1;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tot += warp_cnt[k];
      count += tot;
    }
    __syncthreads();
  }
  for (int i = count + threadIdx.x; i < cap; i += blockDim.x) q.slots[i] = 0;
  if (threadIdx.x == 0) {
    q.counters[0] = 0;                 // head
    q.counters[1] = (uint32_t)count;   // tail
    q.counters[2] = (uint32_t)count;   // pending
  }
}

// fill-holes seeds: J = 1 on border pixels of the complement, else 0
__global__ void k_fill_seed(const uint8_t* __restrict__ bin, int h, int w,
                            uint8_t* __restrict__ J) {
  const int64_t n = (int64_t)h * w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
    const bool border = y == 0 || x == 0 || y == h - 1 || x == w - 1;
    J[i] = (uint8_t)(border && !bin[i]);
  }
}

// out = bin | !reached
__global__ void k_fill_final(const uint8_t* __restrict__ bin,
                             const uint8_t* __restrict__ reached, int64_t n,
                             uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)(bin[i] || !reached[i]);
}

template <typename T, int CONN, class MaskF>
int run_iwpp(rtg_ctx* ctx, T* J, MaskF maskf, int64_t h, int64_t w, int border_only,
             int kind) {
  const int tiles_y = (int)ceil_div(h, kTile), tiles_x = (int)ceil_div(w, kTile);
  const int ntiles = tiles_y * tiles_x;
  const int32_t cap = 2 * ntiles;
  if (cap > ctx->tq.capacity) return fail(RTG_ERR_DIMENSION, "tile exceeds queue capacity");
  k_tiles_init<<<(unsigned)ceil_div(ntiles, 256), 256, 0, ctx->stream>>>(ctx->tq, tiles_y, tiles_x,
                                                                          border_only);
  RTG_LAUNCH("k_tiles_init");
  const size_t smem = sizeof(WarpSmem) * kWarpsPerBlock;
  RTG_SMEM_OPTIN((k_iwpp<T, CONN, MaskF>), smem);
  int per_sm = 0;
  RTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_iwpp<T, CONN, MaskF>,
                                                         kWarpsPerBlock * 32, smem));
  if (per_sm < 1) per_sm = 1;
  const int max_blocks = ctx->num_sms * per_sm;
  int64_t* kstats = ctx->stats + 4 + 2 * kind;
  const uint32_t budget = (uint32_t)(256u * (uint32_t)ntiles + 65536u);
  if (!border_only) {
    // two checkerboard static passes, then the queue drains the wavefronts
    for (int phase = 0; phase < 2; ++phase) {
      const int first = phase == 0 ? (tiles_x + 1) / 2 : tiles_x / 2;
      const int count = (tiles_y / 2) * tiles_x + ((tiles_y & 1) ? first : 0);
      if (count <= 0) continue;
      int blocks = (int)ceil_div((int64_t)count, kWarpsPerBlock);
      if (blocks > max_blocks) blocks = max_blocks;
      k_iwpp<T, CONN, MaskF><<<blocks, kWarpsPerBlock * 32, smem, ctx->stream>>>(
          J, maskf, (int)h, (int)w, tiles_x, ntiles, phase, ctx->tq, cap, kstats, budget,
          ctx->status);
      RTG_LAUNCH("k_iwpp(phase)");
    }
  }
  k_queue_build<<<1, 1024, 0, ctx->stream>>>(ctx->tq, cap, ntiles);
  RTG_LAUNCH("k_queue_build");
  int blocks = max_blocks;
  const int need = (int)ceil_div(ntiles, kWarpsPerBlock);
  if (blocks > need) blocks = need;
  k_iwpp<T, CONN, MaskF><<<blocks, kWarpsPerBlock * 32, smem, ctx->stream>>>(
      J, maskf, (int)h, (int)w, tiles_x, ntiles, -1, ctx->tq, cap, kstats, budget, ctx->status);
  RTG_LAUNCH("k_iwpp(queue)");
  return RTG_OK;
}

}  // namespace

int iwpp_recon_u8(rtg_ctx* ctx, uint8_t* J, const uint8_t* I, int64_t h,
                  int64_t w, int conn) {
  if (conn == 8) return run_iwpp<uint8_t, 8>(ctx, J, PlainMask<uint8_t>{I}, h, w, 0, 0);
  return run_iwpp<uint8_t, 4>(ctx, J, PlainMask<uint8_t>{I}, h, w, 0, 0);
}

int iwpp_recon_u16(rtg_ctx* ctx, uint16_t* J, const uint16_t* I, int64_t h,
                   int64_t w, int conn, int kind) {
  if (conn == 8) return run_iwpp<uint16_t, 8>(ctx, J, PlainMask<uint16_t>{I}, h, w, 0, kind);
  return run_iwpp<uint16_t, 4>(ctx, J, PlainMask<uint16_t>{I}, h, w, 0, kind);
}

int iwpp_fill_holes(rtg_ctx* ctx, const uint8_t* bin, uint8_t* J, int64_t h,
                    int64_t w, uint8_t* out) {
  const int64_t n = h * w;
  const int blocks = (int)(ceil_div(n, 256) < ctx->num_sms * 8 ? ceil_div(n, 256) : ctx->num_sms * 8);
  k_fill_seed<<<blocks, 256, 0, ctx->stream>>>(bin, (int)h, (int)w, J);
  RTG_LAUNCH("k_fill_seed");
  RTG_TRY((run_iwpp<uint8_t, 4>(ctx, J, ComplementMask{bin}, h, w, 1, 3)));
  k_fill_final<<<blocks, 256, 0, ctx->stream>>>(bin, J, n, out);
  RTG_LAUNCH("k_fill_final");
  return RTG_OK;
}

}  // namespace rtg
