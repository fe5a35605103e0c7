// o5 AreaThreshold + o8 BWLabel (and the components behind o3 / o4):
// union-find connected-component labelling (Oliveira &
// Lotufo union-find: "a forest in which each pixel is a tree ... merges
// adjacent trees ... flattening the trees").
//
// 1. k_ccl_tile    one warp per 32x32 tile (the block only meets to reserve
//                  list slots with one global atomic).  The tile's
//                  rows become 32 ballot bit masks; then each lane owns one
//                  ROW and works on runs with bit arithmetic: a run is one
//                  union-find node (its start), unions are issued once per
//                  pair of overlapping runs of adjacent rows (shared-memory
//                  union-find with path halving), run roots are flattened,
//                  and per-local-root accumulators are built (pixel count,
//                  a "seed" bit for predicates that carry one).  Each lane
//                  then owns one COLUMN again to write every pixel's local
//                  root with coalesced stores.  Tile-local roots go to a short
//                  global list together with their accumulators.
//                  The foreground predicate is a functor, so thresholding /
//                  inversion never needs its own pass over the tile.
// 2. k_ccl_seams   union across tile seams (row and column seams in one launch)
//                  in global memory (atomicMin links,
//                  larger root -> smaller root, path halving); a seam pair
//                  already implied by its neighbour pair plus tile-local
//                  connectivity is skipped, so a large component costs a few
//                  unions per seam instead of one per pixel.
// 3. k_ccl_flatten only the local roots are flattened, so the forest is
//                  two-level: pixel -> local root -> global root, and
//                  consumers read root_of(i) = roots[roots[i]] instead of a
//                  full-image flatten pass.  The global root is the minimum
//                  linear index of the component.  The local accumulators are
//                  added into the global root here (component size, seed
//                  flag), and global roots are set in a bitmap.
// 4. canonical compaction: the root bitmap is prefix-summed (2 MB for a
//    4096^2 tile instead of a 64 MB root plane), so labels are 1..n ordered by
//    each object's minimum pixel index (scipy's ndimage.label order).
//
// Roofline: HBM/L2 bound; algorithmic bytes mask 1 B in + labels 4 B out.
#include "common.cuh"

namespace rtg {
namespace {

// Shared-memory find with path halving, used while unions are running (only
// connectivity matters there; a stale halving store can only move an entry
// to another ancestor).
__device__ __forceinline__ int32_t find_root_c(int32_t* par, int32_t a) {
  int32_t p = par[a];
  while (p != a) {
    const int32_t gp = par[p];
    if (gp != p) par[a] = gp;
    a = p;
    p = gp;
  }
  return a;
}

__device__ __forceinline__ void unite_s(int32_t* par, int32_t a, int32_t b) {
  while (true) {
    a = find_root_c(par, a);
    b = find_root_c(par, b);
    if (a == b) return;
    if (a < b) { const int32_t t = a; a = b; b = t; }  // a is the larger root
    const int32_t old = atomicMin(&par[a], b);
    if (old == a) return;
    a = old;
  }
}

// Flattens a warp's run forest (lane owns entries rb .. rb+nruns-1) by
// pointer jumping until no entry changes.  The rows unite with the row above
// all at once, so chains can be as deep as the tile; jumping halves every
// chain per round where per-entry finds walk them link by link.  A
// concurrent store only replaces a parent by an ancestor, and roots never
// change, so "par[par[k]] == par[k]" read at any time means par[k] is final.
// Only entries not yet pointing at a root are revisited (a mask per lane).
template <typename T>
__device__ __forceinline__ void flatten_jump_t(T* par, int rb, int nruns) {
  uint32_t pend = nruns >= 32 ? 0xFFFFFFFFu : (1u << nruns) - 1u;
  while (true) {
    for (uint32_t m = pend; m; m &= m - 1) {
      const int k = __ffs(m) - 1;
      const int32_t p = par[rb + k];
      const int32_t gp = par[p];
      if (gp == p) {
        pend &= ~(1u << k);
        continue;
      }
      // three links per step; an entry that lands on a root is done now
      // rather than after one more round
      const int32_t ggp = par[gp];
      par[rb + k] = (T)ggp;
      if (ggp == gp) pend &= ~(1u << k);
    }
    __syncwarp();
    if (!__any_sync(0xFFFFFFFFu, pend != 0)) break;
  }
}
__device__ __forceinline__ void flatten_jump(int32_t* par, int rb, int nruns) {
  flatten_jump_t(par, rb, nruns);
}

// ---- foreground predicates ----------------------------------------------------
// eval: one pixel; eval4: four consecutive pixels packed in a u32 (byte k =
// pixel x + k), returning 4-bit masks.
__device__ __forceinline__ uint32_t byte_msbs(uint32_t v) {  // bit 7 of each byte -> nibble
  return ((v >> 7) & 1u) | ((v >> 14) & 2u) | ((v >> 21) & 4u) | ((v >> 28) & 8u);
}
__device__ __forceinline__ uint32_t border_nib(int y, int x, int h, int w) {
  if (y == 0 || y == h - 1) return 0xFu;
  return (x == 0 ? 1u : 0u) | (x + 3 == w - 1 ? 8u : 0u);
}
struct FgMask {  // mask != 0
  static constexpr bool kSeed = false;
  static constexpr bool kRows = false;
  const uint8_t* m;
  __device__ __forceinline__ void eval(int64_t i, int, int, bool& fg, bool&) const {
    fg = m[i] != 0;
  }
  __device__ __forceinline__ void eval4(uint32_t v, int, int, uint32_t& fg, uint32_t&) const {
    fg = byte_msbs(~__vcmpeq4(v, 0u));
  }
  __host__ __device__ __forceinline__ const uint8_t* plane() const { return m; }
};
struct FgThresh {  // v >= t; seed: v >= ts (ts > 255: no seeds)
  static constexpr bool kSeed = true;
  static constexpr bool kRows = false;
  const uint8_t* v;
  int32_t t, ts;
  __device__ __forceinline__ void eval(int64_t i, int, int, bool& fg, bool& sd) const {
    const int32_t a = v[i];
    fg = a >= t;
    sd = a >= ts;
  }
  __device__ __forceinline__ void eval4(uint32_t a, int, int, uint32_t& fg, uint32_t& sd) const {
    fg = t > 255 ? 0u : byte_msbs(__vcmpgeu4(a, 0x01010101u * (uint32_t)t));
    sd = ts > 255 ? 0u : byte_msbs(__vcmpgeu4(a, 0x01010101u * (uint32_t)ts));
  }
  __host__ __device__ __forceinline__ const uint8_t* plane() const { return v; }
};
struct FgCode {  // a precomputed code plane: bit 0 foreground, bit 1 seed
  static constexpr bool kSeed = true;
  static constexpr bool kRows = false;
  const uint8_t* c;
  __device__ __forceinline__ void eval(int64_t i, int, int, bool& fg, bool& sd) const {
    const uint32_t a = c[i];
    fg = a & 1u;
    sd = (a >> 1) & 1u;
  }
  __device__ __forceinline__ void eval4(uint32_t a, int, int, uint32_t& fg, uint32_t& sd) const {
    fg = byte_msbs(__vcmpne4(a & 0x01010101u, 0u));
    sd = byte_msbs(__vcmpne4(a & 0x02020202u, 0u));
  }
  __host__ __device__ __forceinline__ const uint8_t* plane() const { return c; }
};
struct FgBackground {  // m == 0; seed: on the image border
  static constexpr bool kSeed = true;
  static constexpr bool kRows = false;
  const uint8_t* m;
  int h, w;
  __device__ __forceinline__ void eval(int64_t i, int y, int x, bool& fg, bool& sd) const {
    fg = m[i] == 0;
    sd = y == 0 || x == 0 || y == h - 1 || x == w - 1;
  }
  __device__ __forceinline__ void eval4(uint32_t v, int y, int x, uint32_t& fg,
                                        uint32_t& sd) const {
    fg = byte_msbs(__vcmpeq4(v, 0u));
    sd = border_nib(y, x, h, w);
  }
  __host__ __device__ __forceinline__ const uint8_t* plane() const { return m; }
};

// A mask given as a 1-bit plane (linear words; w % 32 == 0, so a tile row is
// one word): phase 1 of the tile kernel is a single load per row.
struct FgBitRows {
  static constexpr bool kSeed = false;
  static constexpr bool kRows = true;
  const uint32_t* b;
  int wpr;  // words per image row
  __device__ __forceinline__ uint32_t row(int y, int x0) const { return b[y * wpr + (x0 >> 5)]; }
  __host__ __device__ __forceinline__ const uint8_t* plane() const { return nullptr; }
};

// The ReconToNuclei threshold pair as 1-bit planes (the streaming kernel's
// recon_bits): foreground and seed rows are one load each.
struct FgSeedRows {
  static constexpr bool kSeed = true;
  static constexpr bool kRows = true;
  const uint32_t* fg;
  const uint32_t* sd;
  int wpr;
  __device__ __forceinline__ uint32_t row(int y, int x0) const { return fg[y * wpr + (x0 >> 5)]; }
  __device__ __forceinline__ uint32_t seed_row(int y, int x0) const {
    return sd[y * wpr + (x0 >> 5)];
  }
  __host__ __device__ __forceinline__ const uint8_t* plane() const { return nullptr; }
};

constexpr int kTileWarps = 4;
constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kSeedBit = 0x80000000u;

// lowest run of ones of v (bit 0 of v set)
__device__ __forceinline__ uint32_t low_run(uint32_t v) { return v & ~(v + 1u); }

// Run-table form of a labelling (w % 32 == 0; cf. the joint fill/area
// labelling's RunTable): instead of a local root for every pixel, each tile
// leaves its row masks, the ordinal of every run's local root within the
// tile's contiguous range of the local-root list, and the local roots of its
// border pixels (all the seams read).  The roots plane then only holds the
// local roots' own entries (the global forest), and the consumers re-derive a
// pixel's run from the row mask.
struct CclRuns {
  uint32_t* rowbits = nullptr;  // [tile * 32 + r]: foreground bits of row r
  uint16_t* rtab = nullptr;     // [tile * 512 + r * 16 + k]: ordinal of run k's local root
  int2* tinfo = nullptr;        // [tile]: (first local-root slot, local-root count)
  int32_t* border = nullptr;    // [tile * 128 + side * 32 + i]: top row, bottom row, left
                                // column, right column: local root (global index) or -1
};

// Runs are named compactly: run k of tile row r is node r * 16 + k (a 32-pixel
// row holds at most 16 runs), so the per-warp forest is 512 entries.
template <int CONN, class P>
__global__ void __launch_bounds__(32 * kTileWarps)
k_ccl_tile(P pred, int h, int w, int tiles_x, int ntiles, int32_t* __restrict__ roots,
           int32_t* __restrict__ lroots, int32_t* __restrict__ lcount,
           int32_t* __restrict__ zero_a, int32_t* __restrict__ zero_b, CclRuns rt) {
  pdl_enter();
  __shared__ int32_t s_par[kTileWarps][512];
  __shared__ uint32_t s_inf[kTileWarps][512];
  __shared__ uint8_t s_pos[kTileWarps][512];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = min(blockIdx.x * kTileWarps + wid, ntiles - 1);
  // a surplus warp of the last block repeats the last tile read-only (it
  // publishes and writes nothing) so every warp reaches the block barrier
  const bool active = blockIdx.x * kTileWarps + wid < ntiles;
  const int x0 = (tile % tiles_x) * 32, y0 = (tile / tiles_x) * 32;
  int32_t* par = s_par[wid];
  uint32_t* inf = s_inf[wid];
  uint8_t* pos = s_pos[wid];
  // 1. row bit masks; lane r keeps row r
  uint32_t bits = 0, seeds = 0;
  const int x = x0 + lane;
  const bool vec = !P::kRows && (w & 3) == 0 && x0 + 32 <= w &&
                   (reinterpret_cast<uintptr_t>(pred.plane()) & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(roots) & 15) == 0;
  if constexpr (P::kRows) {
    if (y0 + lane < h) {
      bits = pred.row(y0 + lane, x0);
      if constexpr (P::kSeed) seeds = pred.seed_row(y0 + lane, x0) & bits;
    }
  } else if (vec) {
    // 4 pixels per load: lane covers row 4k + lane/8, columns 4 (lane % 8) ..
    // + 3; the 8 lanes of a row OR their nibbles together
    const uint8_t* pl = pred.plane();
    const int g = lane >> 3, cq = (lane & 7) * 4;
    uint32_t word[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int y = y0 + 4 * k + g;
      word[k] = y < h ? __ldg(reinterpret_cast<const uint32_t*>(pl + (int64_t)y * w + x0 + cq))
                      : 0u;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int y = y0 + 4 * k + g;
      uint32_t fn = 0, sn = 0;
      if (y < h) pred.eval4(word[k], y, x0 + cq, fn, sn);
      uint32_t m = fn << cq, ms = (fn & sn) << cq;
      m |= __shfl_xor_sync(kFull, m, 1);
      m |= __shfl_xor_sync(kFull, m, 2);
      m |= __shfl_xor_sync(kFull, m, 4);
      const uint32_t t = __shfl_sync(kFull, m, (lane & 3) * 8);
      if ((lane >> 2) == k) bits = t;
      if (P::kSeed) {
        ms |= __shfl_xor_sync(kFull, ms, 1);
        ms |= __shfl_xor_sync(kFull, ms, 2);
        ms |= __shfl_xor_sync(kFull, ms, 4);
        const uint32_t ts = __shfl_sync(kFull, ms, (lane & 3) * 8);
        if ((lane >> 2) == k) seeds = ts;
      }
    }
  } else {
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const int y = y0 + r;
      bool fg = false, sd = false;
      if (y < h && x < w) pred.eval((int64_t)y * w + x, y, x, fg, sd);
      const uint32_t b = __ballot_sync(kFull, fg);
      if (lane == r) bits = b;
      if (P::kSeed) {
        const uint32_t sb = __ballot_sync(kFull, fg && sd);
        if (lane == r) seeds = sb;
      }
    }
  }
  // 2. lane = row: one link per pair of overlapping runs of adjacent rows.
  //    A run's first overlapping run above becomes its parent with a plain
  //    store (every run has at most one such link, pointing to a smaller
  //    index, so these links alone form a forest); only further overlaps
  //    need shared-memory unions.
  const int rb = lane * 16;
  const uint32_t starts = bits & ~(bits << 1);
  uint32_t up = __shfl_up_sync(kFull, bits, 1);
  if (lane == 0) up = 0;
  const uint32_t upstarts = up & ~(up << 1);
  // run of the row above that holds column t (t in up), as a node id
  auto upper = [&](int t) -> int {
    const uint32_t below = upstarts & (t == 31 ? kFull : ((2u << t) - 1u));
    const int su = 31 - __clz(below);
    return rb - 16 + __popc(upstarts & ((1u << su) - 1u));
  };
  uint32_t more = 0;  // runs (by index bit) with further overlaps
  {
    int k = 0;
    for (uint32_t m = starts; m; m &= m - 1, ++k) {
      const int b = __ffs(m) - 1;
      pos[rb + k] = (uint8_t)b;
      const uint32_t run = low_run(bits >> b) << b;
      uint32_t ov = up & (CONN == 8 ? (run | (run << 1) | (run >> 1)) : run);
      if (!ov) {
        par[rb + k] = rb + k;
        continue;
      }
      const int t = __ffs(ov) - 1;
      par[rb + k] = upper(t);
      ov &= ~(low_run(up >> t) << t);
      if (ov) more |= 1u << k;
    }
  }
  __syncwarp();
  if (more) {
    int k = 0;
    for (uint32_t m = starts; m; m &= m - 1, ++k) {
      if (!((more >> k) & 1u)) continue;
      const int b = __ffs(m) - 1;
      const uint32_t run = low_run(bits >> b) << b;
      uint32_t ov = up & (CONN == 8 ? (run | (run << 1) | (run >> 1)) : run);
      ov &= ~(low_run(up >> (__ffs(ov) - 1)) << (__ffs(ov) - 1));  // the linked one
      while (ov) {
        const int t = __ffs(ov) - 1;
        unite_s(par, rb + k, upper(t));
        ov &= ~(low_run(up >> t) << t);
      }
    }
  }
  __syncwarp();
  // 3. flatten the run forest (read-only finds, then own-entry writes), then
  //    accumulate pixel counts / seed bits at the local roots
  const int nruns = __popc(starts);
  flatten_jump(par, rb, nruns);
  uint32_t rootm = 0;  // this row's local roots, by run index
  for (int k = 0; k < nruns; ++k) {
    if (par[rb + k] == rb + k) {
      inf[rb + k] = 0;
      rootm |= 1u << k;
    }
  }
  const int nroot = __popc(rootm);
  __syncwarp();
  {
    int k = 0;
    for (uint32_t m = starts; m; m &= m - 1, ++k) {
      const int b = __ffs(m) - 1;
      const uint32_t run = low_run(bits >> b) << b;
      const int32_t root = par[rb + k];
      if (P::kSeed && (seeds & run)) atomicOr(&inf[root], kSeedBit);
      atomicAdd(&inf[root], (uint32_t)__popc(run));
    }
  }
  // publish the local roots (one global atomic per block)
  __shared__ int32_t s_res[kTileWarps + 1];
  __syncwarp();
  int base = block_reserve(active ? nroot : 0, lcount, s_res);
  if (!active) return;
  const int32_t tbase = __shfl_sync(kFull, base, 0);  // the tile's roots are contiguous
  for (uint32_t m = rootm; m; m &= m - 1) {
    const int k = __ffs(m) - 1;
    const int32_t g = (y0 + lane) * w + x0 + pos[rb + k];
    lroots[2 * base] = g;
    lroots[2 * base + 1] = (int32_t)inf[rb + k];
    if (rt.rtab) {
      inf[rb + k] = (uint32_t)(base - tbase);  // the root's ordinal in the tile
      roots[g] = g;
    }
    ++base;
    if (zero_a) zero_a[g] = 0;
    if (zero_b) zero_b[g] = 0;
  }
  if (rt.rtab) {
    __syncwarp();
    const int32_t tend = __shfl_sync(kFull, base, 31);
    if (lane == 0) rt.tinfo[tile] = make_int2(tbase, tend - tbase);
    rt.rowbits[tile * 32 + lane] = bits;
    // this row's 16 table entries (two 16-byte stores; the warp's are contiguous)
    uint32_t pk[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < 16; ++k) {  // the warp stops at its longest row's run count
      if (k >= nruns) break;
      pk[k >> 1] |= inf[par[rb + k]] << (16 * (k & 1));
    }
    uint4* dst = reinterpret_cast<uint4*>(rt.rtab + (int64_t)tile * 512 + rb);
    dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    // border pixels: rows 0 and 31 (lane = column), columns 0 and 31 (lane = row)
    auto glob = [&](int32_t lr) { return (y0 + (lr >> 4)) * w + x0 + (int32_t)pos[lr]; };
    int32_t* bd = rt.border + (int64_t)tile * 128;
    const uint32_t below = (2u << lane) - 1u;
    const uint32_t b0 = __shfl_sync(kFull, bits, 0), b31 = __shfl_sync(kFull, bits, 31);
    bd[lane] = ((b0 >> lane) & 1u) ? glob(par[__popc(b0 & ~(b0 << 1) & below) - 1]) : -1;
    bd[32 + lane] =
        ((b31 >> lane) & 1u) ? glob(par[31 * 16 + __popc(b31 & ~(b31 << 1) & below) - 1]) : -1;
    bd[64 + lane] = (bits & 1u) ? glob(par[rb]) : -1;
    bd[96 + lane] = (bits >> 31) ? glob(par[rb + nruns - 1]) : -1;
    return;
  }
  // global index of every run's local root (inf is free again)
  __syncwarp();
  for (int k = 0; k < nruns; ++k) {
    const int32_t lr = par[rb + k];
    inf[rb + k] = (uint32_t)((y0 + (lr >> 4)) * w + x0 + pos[lr]);
  }
  __syncwarp();
  // 4. every pixel's local root (global index), coalesced stores
  if (vec) {
    // 4 pixels per lane (one 16-byte store): 8 lanes per row, 4 rows per step
    const int g = lane >> 3, cq = (lane & 7) * 4;
#pragma unroll 2
    for (int k = 0; k < 8; ++k) {
      const int r = 4 * k + g;
      const uint32_t b = __shfl_sync(kFull, bits, r);
      const int y = y0 + r;
      if (y >= h) continue;
      const uint32_t st = b & ~(b << 1);
      int32_t o[4];
      const uint32_t fg4 = (b >> cq) & 0xFu;
      if (!fg4) {
        o[0] = o[1] = o[2] = o[3] = -1;
      } else if (fg4 == 0xFu && !((st >> (cq + 1)) & 7u)) {
        // four foreground pixels of one run: one lookup
        o[0] = o[1] = o[2] = o[3] = (int32_t)inf[r * 16 + __popc(st & ((2u << cq) - 1u)) - 1];
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = cq + j;
          o[j] = ((b >> c) & 1u) ? (int32_t)inf[r * 16 + __popc(st & ((2u << c) - 1u)) - 1] : -1;
        }
      }
      *reinterpret_cast<int4*>(roots + (int64_t)y * w + x0 + cq) = make_int4(o[0], o[1], o[2], o[3]);
    }
  } else {
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      const uint32_t b = __shfl_sync(kFull, bits, r);
      const int y = y0 + r;
      if (y < h && x < w) {
        const uint32_t st = b & ~(b << 1);
        roots[(int64_t)y * w + x] =
            ((b >> lane) & 1u) ? (int32_t)inf[r * 16 + __popc(st & ((2u << lane) - 1u)) - 1] : -1;
      }
    }
  }
}

// Seams between tile rows: pixel (y, x) with y = 32k, k >= 1.  A pair is
// skipped when the same two components are already joined through the pair
// one column to the left (same tile-local runs on both sides).
template <int CONN>
__device__ __forceinline__ void seam_row_px(int h, int w, int32_t* __restrict__ roots, int y,
                                            int x) {
  if (x >= w || y >= h) return;
  const int32_t p = y * w + x;
  if (__ldcg(roots + p) < 0) return;
  const int32_t u = p - w;
  const bool in_run_l = (x & 31) != 0 && __ldcg(roots + p - 1) >= 0;  // p ~ left (same run)
  const bool fu = __ldcg(roots + u) >= 0;
  const bool ful = x > 0 && __ldcg(roots + u - 1) >= 0;
  if (fu && !(in_run_l && ful)) uf_unite_g(roots, p, u);
  if (CONN == 8) {
    // up-left: implied by (left, up-left) when p ~ left, or by (p, up) when up ~ up-left
    if (ful && !in_run_l && !(fu && (x & 31) != 0)) uf_unite_g(roots, p, u - 1);
    // up-right: implied by (p, up) when up ~ up-right
    if (x + 1 < w && __ldcg(roots + u + 1) >= 0 && !(fu && ((x + 1) & 31) != 0))
      uf_unite_g(roots, p, u + 1);
  }
}

// Seams between tile columns: pixel (y, x) with x = 32k, k >= 1 (vertically
// adjacent pixels of one tile are always in one local component).
template <int CONN>
__device__ __forceinline__ void seam_col_px(int h, int w, int32_t* __restrict__ roots, int y,
                                            int x) {
  if (y >= h || x >= w) return;
  const int32_t p = y * w + x;
  if (__ldcg(roots + p) < 0) return;
  const int32_t l = p - 1;
  const bool in_col_u = (y & 31) != 0 && __ldcg(roots + p - w) >= 0;  // p ~ up
  const bool fl = __ldcg(roots + l) >= 0;
  const bool ful = y > 0 && __ldcg(roots + l - w) >= 0;
  if (fl && !(in_col_u && ful)) uf_unite_g(roots, p, l);
  if (CONN == 8) {
    // up-left: implied by (up, up-left) when p ~ up, or by (p, left) when left ~ up-left
    if (ful && !in_col_u && !(fl && (y & 31) != 0)) uf_unite_g(roots, p, l - w);
    // down-left: implied by (p, left) when left ~ down-left
    if (y + 1 < h && __ldcg(roots + l + w) >= 0 && !(fl && ((y + 1) & 31) != 0))
      uf_unite_g(roots, p, l + w);
  }
}

// Both seam families in one launch: blockIdx.y < tiles_y - 1 walks a row
// seam (y = 32 (k + 1)), the rest walk column seams.
template <int CONN>
__global__ void k_ccl_seams(int h, int w, int row_seams, int32_t* __restrict__ roots) {
  pdl_enter();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if ((int)blockIdx.y < row_seams)
    seam_row_px<CONN>(h, w, roots, ((int)blockIdx.y + 1) * 32, t);
  else
    seam_col_px<CONN>(h, w, roots, t, ((int)blockIdx.y - row_seams + 1) * 32);
}

// Seams of the run-table form: the same pairs and skips as seam_row_px /
// seam_col_px, read from the tiles' border arrays (compact, coalesced) and
// united through the local roots themselves.
template <int CONN>
__global__ void k_ccl_seams_rt(int h, int w, int tiles_x, int row_seams,
                               const int32_t* __restrict__ border, int32_t* __restrict__ roots) {
  pdl_enter();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if ((int)blockIdx.y < row_seams) {
    const int y = ((int)blockIdx.y + 1) * 32, x = t;
    if (x >= w || y >= h) return;
    const int tb = (y >> 5) * tiles_x;  // the tile row below the seam
    const int32_t* top = border + (int64_t)(tb + (x >> 5)) * 128;
    auto bot = [&](int xx) {  // bottom rows of the tile row above
      return __ldg(border + (int64_t)(tb - tiles_x + (xx >> 5)) * 128 + 32 + (xx & 31));
    };
    const int32_t vp = __ldg(top + (x & 31));
    if (vp < 0) return;
    const bool in_run_l = (x & 31) != 0 && __ldg(top + (x & 31) - 1) >= 0;  // p ~ left
    const int32_t vu = bot(x), vul = x > 0 ? bot(x - 1) : -1;
    const bool fu = vu >= 0, ful = vul >= 0;
    if (fu && !(in_run_l && ful)) uf_unite_g(roots, vp, vu);
    if (CONN == 8) {
      if (ful && !in_run_l && !(fu && (x & 31) != 0)) uf_unite_g(roots, vp, vul);
      if (x + 1 < w) {
        const int32_t vur = bot(x + 1);
        if (vur >= 0 && !(fu && ((x + 1) & 31) != 0)) uf_unite_g(roots, vp, vur);
      }
    }
  } else {
    const int x = ((int)blockIdx.y - row_seams + 1) * 32, y = t;
    if (y >= h || x >= w) return;
    const int tc = x >> 5;  // the tile column right of the seam
    const int32_t* left = border + (int64_t)((y >> 5) * tiles_x + tc) * 128 + 64;
    auto rcol = [&](int yy) {  // right columns of the tile column left of the seam
      return __ldg(border + (int64_t)((yy >> 5) * tiles_x + tc - 1) * 128 + 96 + (yy & 31));
    };
    const int32_t vp = __ldg(left + (y & 31));
    if (vp < 0) return;
    const bool in_col_u = (y & 31) != 0 && __ldg(left + (y & 31) - 1) >= 0;  // p ~ up
    const int32_t vl = rcol(y), vul = y > 0 ? rcol(y - 1) : -1;
    const bool fl = vl >= 0, ful = vul >= 0;
    if (fl && !(in_col_u && ful)) uf_unite_g(roots, vp, vl);
    if (CONN == 8) {
      if (ful && !in_col_u && !(fl && (y & 31) != 0)) uf_unite_g(roots, vp, vul);
      if (y + 1 < h) {
        const int32_t vdl = rcol(y + 1);
        if (vdl >= 0 && !(fl && ((y + 1) & 31) != 0)) uf_unite_g(roots, vp, vdl);
      }
    }
  }
}

// Flattens the local roots onto the global roots and folds the local
// accumulators into them; global roots are marked in the bitmap.
__global__ void k_ccl_flatten(int32_t* __restrict__ lroots,
                              const int32_t* __restrict__ lcount, int32_t* roots,
                              int32_t* __restrict__ counts, int32_t* __restrict__ flags,
                              uint32_t* __restrict__ bitmap, bool seed_in_counts = false) {
  pdl_enter();
  const int n = *lcount;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count: lanes of one warp stay converged, so the count
  // and flag updates of local roots sharing a global root (a large
  // component spans many tiles) are combined into one atomic per warp
  const int stride = gridDim.x * blockDim.x;
  for (int k0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; k0 < n; k0 += stride) {
    const int k = k0 + lane;
    int32_t g = -1;
    uint32_t info = 0;
    if (k < n) {
      const int32_t r = lroots[2 * k];
      info = (uint32_t)lroots[2 * k + 1];
      g = uf_find_g(roots, r);
      // the accumulator slot is consumed here: it becomes the global root,
      // so the emit kernels skip the roots[] gather
      lroots[2 * k + 1] = g;
      if (g != r) atomicMin(roots + r, g);
      else if (bitmap) atomicOr(bitmap + (r >> 5), 1u << (r & 31));
    }
    const unsigned grp = __match_any_sync(0xFFFFFFFFu, g);
    const uint32_t cnt = __reduce_add_sync(grp, info & ~kSeedBit);
    const uint32_t seed = __reduce_or_sync(grp, info & kSeedBit);
    if (g < 0 || lane != __ffs(grp) - 1) continue;
    if (counts) atomicAdd(counts + g, (int32_t)cnt);
    if (seed_in_counts && seed) atomicOr(counts + g, (int32_t)kSeedBit);
    if (flags && seed) flags[g] = 1;
  }
}

__global__ void k_area_filter(int64_t n, const int32_t* __restrict__ roots,
                              const int32_t* __restrict__ counts, int32_t lo,
                              int32_t hi, uint8_t* __restrict__ out) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = root_of(roots, i);
    uint8_t keep = 0;
    if (r >= 0) {
      const int32_t a = counts[r];
      keep = (uint8_t)(a >= lo && a <= hi);
    }
    out[i] = keep;
  }
}

// ---- canonical compaction -----------------------------------------------------

__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  int off = 0;
  total = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
    if (k < wid) off += warp_tot[k];
    total += warp_tot[k];
  }
  return off + incl - v;
}

// Canonical ranks from the root bitmap: per-word exclusive prefixes in one
// look-back pass, then one rank per global root.
constexpr int kBmPerThread = 16;
constexpr int kBmChunk = 256 * kBmPerThread;  // words per chunk

// Single-pass per-word exclusive prefix of the root bitmap (decoupled
// look-back): each CTA popcounts its chunk, publishes the chunk aggregate,
// then walks back over its predecessors' published values until it meets an
// inclusive prefix.  Replaces count / chunk-scan / prefix (three launches).
// status[c] = flag << 62 | value (flag 1: aggregate, 2: inclusive prefix);
// status[nchunks] is the CTA ticket (chunks are taken in launch order, so
// every predecessor is running or done).  status must be zero on entry.
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(256)
k_bm_scan(int64_t nwords, int nchunks, const uint32_t* __restrict__ bm,
          unsigned long long* status, int32_t* __restrict__ wprefix, int32_t* __restrict__ d_total) {
  pdl_enter();
  __shared__ int warp_tot[8];
  __shared__ int s_bid, s_prefix;
  if (threadIdx.x == 0)
    s_bid = atomicAdd(reinterpret_cast<int*>(status + nchunks), 1);
  __syncthreads();
  const int bid = s_bid;
  const int64_t base = (int64_t)bid * kBmChunk + (int64_t)threadIdx.x * kBmPerThread;
  uint32_t v[kBmPerThread];
  const bool full = base + kBmPerThread <= nwords;  // 16 words = 4 x 16-byte loads
  if (full) {
#pragma unroll
    for (int q = 0; q < kBmPerThread / 4; ++q) {
      const uint4 t = __ldg(reinterpret_cast<const uint4*>(bm + base) + q);
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kBmPerThread; ++k) v[k] = base + k < nwords ? bm[base + k] : 0u;
  }
  int c = 0;
#pragma unroll
  for (int k = 0; k < kBmPerThread; ++k) c += __popc(v[k]);
  int total;
  int run = block_excl_scan(c, warp_tot, total);
  if (threadIdx.x < 32) {
    // warp 0: publish, then look back over windows of 32 predecessors
    const int lane = threadIdx.x;
    if (lane == 0)
      st_release_u64(status + bid, ((bid == 0 ? 2ull : 1ull) << 62) | (uint32_t)total);
    int prefix = 0;
    for (int j = bid - 1; j >= 0;) {
      const int idx = j - lane;
      const unsigned long long st = idx >= 0 ? ld_acquire_u64(status + idx) : (2ull << 62);
      const unsigned flag = (unsigned)(st >> 62);
      const unsigned incl = __ballot_sync(0xFFFFFFFFu, flag == 2);
      const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive prefix
      const unsigned upto = stop == 31 ? 0xFFFFFFFFu : ((2u << stop) - 1u);
      if (__ballot_sync(0xFFFFFFFFu, flag == 0) & upto) continue;  // not published yet
      int v = (lane <= stop) ? (int)(st & 0xFFFFFFFFull) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
      prefix += v;
      if (incl) break;
      j -= 32;
    }
    if (lane == 0) {
      if (bid > 0) st_release_u64(status + bid, (2ull << 62) | (uint32_t)(prefix + total));
      s_prefix = prefix;
      if (bid == nchunks - 1 && d_total) *d_total = prefix + total;
    }
  }
  __syncthreads();
  run += s_prefix;
  int32_t o[kBmPerThread];
#pragma unroll
  for (int k = 0; k < kBmPerThread; ++k) {
    o[k] = run;
    run += __popc(v[k]);
  }
  if (full) {
#pragma unroll
    for (int q = 0; q < kBmPerThread / 4; ++q)
      reinterpret_cast<int4*>(wprefix + base)[q] =
          make_int4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < kBmPerThread; ++k)  // unrolled: o[] stays in registers
      if (base + k < nwords) wprefix[base + k] = o[k];
  }
}

__global__ void k_root_rank(const int32_t* __restrict__ lroots, const int32_t* __restrict__ lcount,
                            const int32_t* __restrict__ roots, const uint32_t* __restrict__ bm,
                            const int32_t* __restrict__ wprefix, int32_t* __restrict__ rank,
                            FeatureAcc acc, bool clear_acc) {
  pdl_enter();
  // the final label (rank of the global root + 1) of every LOCAL root, so the
  // per-pixel relabel needs one gather (local root -> label); the run-table
  // form computes the same inside k_label_emit
  const int n = *lcount;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t lr = lroots[2 * k];
    const int32_t r = roots[lr];
    const int32_t label = wprefix[r >> 5] + __popc(bm[r >> 5] & ((1u << (r & 31)) - 1u)) + 1;
    rank[lr] = label;
    // each label once (at its global root): reset its feature accumulators
    if (clear_acc && lr == r && label <= acc.cap) {
      const int64_t i = label - 1;
#pragma unroll
      for (int f = 0; f < kSumFields; ++f) acc.sums[(int64_t)f * acc.cap + i] = 0ull;
#pragma unroll
      for (int f = 0; f < kMinFields; ++f) acc.mins[(int64_t)f * acc.cap + i] = INT32_MAX;
#pragma unroll
      for (int f = 0; f < kMaxFields; ++f) acc.maxs[(int64_t)f * acc.cap + i] = -1;
    }
  }
}

// 4 pixels per thread with 16-byte loads/stores and staged gathers.
__global__ void k_relabel(int64_t n, const int32_t* __restrict__ roots,
                          const int32_t* __restrict__ rank,
                          int32_t* __restrict__ labels) {
  pdl_enter();
  const bool vec = ((reinterpret_cast<uintptr_t>(roots) | reinterpret_cast<uintptr_t>(labels)) &
                    15) == 0;
  for (int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); i0 < n;
       i0 += 4 * (int64_t)gridDim.x * blockDim.x) {
    if (vec && i0 + 4 <= n) {
      const int4 r4 = __ldg(reinterpret_cast<const int4*>(roots + i0));
      int32_t v[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = v[k] >= 0 ? rank[v[k]] : 0;  // label of the local root
      *reinterpret_cast<int4*>(labels + i0) = make_int4(v[0], v[1], v[2], v[3]);
    } else {
      for (int64_t i = i0; i < n && i < i0 + 4; ++i) {
        const int32_t lr = roots[i];
        labels[i] = lr >= 0 ? rank[lr] : 0;
      }
    }
  }
}

// Labels of the run-table form: one warp per tile.  The tile's labels (its
// slice of the by-slot rank array) are staged in shared memory; lane = row
// resolves its runs' labels, then 8 lanes per row write 4 pixels each
// (16-byte stores, four rows per step).
__global__ void __launch_bounds__(32 * kTileWarps)
k_label_emit(CclRuns rt, const int32_t* __restrict__ lroots, const int32_t* __restrict__ roots,
             const uint32_t* __restrict__ bm, const int32_t* __restrict__ wprefix, FeatureAcc acc,
             bool clear_acc, int h, int w, int tiles_x, int ntiles, int32_t* __restrict__ labels,
             bool vec, uint8_t* __restrict__ mask_out) {
  pdl_enter();
  __shared__ int32_t s_rank[kTileWarps][512];
  __shared__ int32_t s_lab[kTileWarps][512];
  __shared__ uint32_t s_bits[kTileWarps][32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kTileWarps + wid;
  if (tile >= ntiles) return;  // no block-wide barrier below
  const int x0 = (tile % tiles_x) * 32, y0 = (tile / tiles_x) * 32;
  const int2 ti = __ldg(rt.tinfo + tile);
  // the final label of each of the tile's local roots (rank of its global
  // root in the root bitmap + 1, what k_root_rank computes for the
  // per-pixel form), and each label's feature accumulators reset once (at
  // the local root that is the global root)
  for (int j = lane; j < ti.y; j += 32) {
    // (local root, global root): k_ccl_flatten wrote the global root
    const int2 e = __ldg(reinterpret_cast<const int2*>(lroots) + ti.x + j);
    const int32_t lr = e.x, r = e.y;
    const int32_t label =
        __ldg(wprefix + (r >> 5)) + __popc(__ldg(bm + (r >> 5)) & ((1u << (r & 31)) - 1u)) + 1;
    s_rank[wid][j] = label;
    if (clear_acc && lr == r && label <= acc.cap) {
      const int64_t i = label - 1;
#pragma unroll
      for (int f = 0; f < kSumFields; ++f) acc.sums[(int64_t)f * acc.cap + i] = 0ull;
#pragma unroll
      for (int f = 0; f < kMinFields; ++f) acc.mins[(int64_t)f * acc.cap + i] = INT32_MAX;
#pragma unroll
      for (int f = 0; f < kMaxFields; ++f) acc.maxs[(int64_t)f * acc.cap + i] = -1;
    }
  }
  const uint32_t bits = __ldg(rt.rowbits + tile * 32 + lane);
  const uint4* src = reinterpret_cast<const uint4*>(rt.rtab + (int64_t)tile * 512 + lane * 16);
  const uint4 e0 = __ldg(src), e1 = __ldg(src + 1);
  const uint32_t ew[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
  const int nruns = __popc(bits & ~(bits << 1));
  s_bits[wid][lane] = bits;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) {  // the warp stops at its longest row's run count
    if (k >= nruns) break;
    s_lab[wid][lane * 16 + k] = s_rank[wid][(ew[k >> 1] >> (16 * (k & 1))) & 0xFFFFu];
  }
  __syncwarp();
  const int g = lane >> 3, cq = (lane & 7) * 4;
#pragma unroll 2
  for (int k = 0; k < 8; ++k) {
    const int r = 4 * k + g;
    if (y0 + r >= h) break;
    const uint32_t b = s_bits[wid][r], st = b & ~(b << 1);
    const uint32_t nib = (b >> cq) & 0xFu;
    int32_t o[4] = {0, 0, 0, 0};
    if (nib) {
      // no run starting inside cq+1 .. cq+3 (the common case): every set
      // pixel of the four lies in the run holding column cq - one lookup
      const uint32_t inner = (st >> (cq + 1)) & 7u;
      if (!inner) {
        const int32_t lab = s_lab[wid][r * 16 + __popc(st & ((2u << cq) - 1u)) - 1];
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = ((nib >> j) & 1u) ? lab : 0;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = cq + j;
          o[j] = ((b >> c) & 1u) ? s_lab[wid][r * 16 + __popc(st & ((2u << c) - 1u)) - 1] : 0;
        }
      }
    }
    int32_t* dst = labels + (int64_t)(y0 + r) * w + x0 + cq;
    if (mask_out)
      *reinterpret_cast<uint32_t*>(mask_out + (int64_t)(y0 + r) * w + x0 + cq) =
          (((b >> cq) & 0xFu) * 0x00204081u) & 0x01010101u;
    if (vec) {
      *reinterpret_cast<int4*>(dst) = make_int4(o[0], o[1], o[2], o[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = o[j];
    }
  }
}

// Seeded-component mask of the run-table form (ReconToNuclei), per tile:
// each local root's component is kept when its global root carries the
// seed flag; kept runs & tissue -> out bytes (or row masks).
__global__ void __launch_bounds__(32 * kTileWarps)
k_seeded_emit(CclRuns rt, const int32_t* __restrict__ lroots, const int32_t* __restrict__ roots,
              const int32_t* __restrict__ flag, const uint8_t* __restrict__ tissue,
              int h, int w, int tiles_x, int ntiles, uint8_t* __restrict__ out,
              uint32_t* __restrict__ out_bits, const uint32_t* __restrict__ tis_bits) {
  pdl_enter();
  __shared__ uint8_t s_kp[kTileWarps][512];
  __shared__ uint32_t s_kept[kTileWarps][32];
  __shared__ uint32_t s_tis[kTileWarps][32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kTileWarps + wid;
  if (tile >= ntiles) return;
  const int x0 = (tile % tiles_x) * 32, y0 = (tile / tiles_x) * 32;
  const int2 ti = __ldg(rt.tinfo + tile);
  for (int j = lane; j < ti.y; j += 32)  // seeded component? (its global root's flag)
    s_kp[wid][j] = __ldcg(flag + __ldg(lroots + 2 * (ti.x + j) + 1)) != 0;
  const uint32_t bits = __ldg(rt.rowbits + tile * 32 + lane);
  const uint4* src = reinterpret_cast<const uint4*>(rt.rtab + (int64_t)tile * 512 + lane * 16);
  const uint4 e0 = __ldg(src), e1 = __ldg(src + 1);
  const uint32_t ew[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
  __syncwarp();
  uint32_t st = bits & ~(bits << 1), kept = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (!st) break;
    const int b = __ffs(st) - 1;
    st &= st - 1;
    if (s_kp[wid][(ew[k >> 1] >> (16 * (k & 1))) & 0xFFFFu]) kept |= low_run(bits >> b) << b;
  }
  s_kept[wid][lane] = kept;
  __syncwarp();
  const int g = lane >> 3, cq = (lane & 7) * 4;
  if (out_bits && tis_bits) {  // tissue as a 1-bit plane too: one word per row
    const uint32_t tw = y0 + lane < h ? __ldg(tis_bits + (y0 + lane) * (w >> 5) + (x0 >> 5)) : 0u;
    out_bits[tile * 32 + lane] = kept & tw;
    return;
  }
  if (out_bits) {
    // row masks of (kept & tissue) for the joint fill/area tile kernel
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = 4 * k + g;
      uint32_t tn = 0;
      if (y0 + r < h) {
        const uint32_t tv = __ldg(reinterpret_cast<const uint32_t*>(
            tissue + (int64_t)(y0 + r) * w + x0 + cq));
        tn = ((~__vcmpeq4(tv, 0u) & 0x80808080u) * 0x00204081u) >> 28;  // byte MSBs -> nibble
      }
      uint32_t v = tn << cq;
      v |= __shfl_xor_sync(kFull, v, 1);
      v |= __shfl_xor_sync(kFull, v, 2);
      v |= __shfl_xor_sync(kFull, v, 4);
      if ((lane & 7) == 0) s_tis[wid][r] = v;
    }
    __syncwarp();
    out_bits[tile * 32 + lane] = kept & s_tis[wid][lane];
    return;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int r = 4 * k + g;
    if (y0 + r >= h) break;
    const int64_t i = (int64_t)(y0 + r) * w + x0 + cq;
    const uint32_t nib = (s_kept[wid][r] >> cq) & 0xFu;
    const uint32_t tv = __ldg(reinterpret_cast<const uint32_t*>(tissue + i));
    *reinterpret_cast<uint32_t*>(out + i) =
        (nib * 0x00204081u) & 0x01010101u & __vcmpne4(tv, 0u);
  }
}

int grid_for(rtg_ctx* ctx, int64_t n) {
  const int64_t want = ceil_div(n, 256);
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  return (int)(want < cap ? want : cap);
}

// 16-bit shared-memory forest (run ids < 1024).  There is no 16-bit
// atomicMin, so the link is a CAS on the 32-bit word holding the entry; plain
// 16-bit path-halving stores cannot be lost to it (a CAS whose expected word
// changed underneath simply retries).
__device__ __forceinline__ int32_t find_root16_c(uint16_t* par, int32_t a) {
  int32_t p = par[a];
  while (p != a) {
    const int32_t gp = par[p];
    if (gp != p) par[a] = (uint16_t)gp;
    a = p;
    p = gp;
  }
  return a;
}

// flatten_jump on the 16-bit forest.
__device__ __forceinline__ void flatten_jump16(uint16_t* par, int rb, int nruns) {
  flatten_jump_t(par, rb, nruns);
}

__device__ __forceinline__ int32_t atomic_min16(uint16_t* par, int32_t a, int32_t b) {
  uint32_t* wp = reinterpret_cast<uint32_t*>(par) + (a >> 1);
  const uint32_t sh = (uint32_t)(a & 1) * 16u;
  uint32_t old = *reinterpret_cast<volatile uint32_t*>(wp);
  while (true) {
    const int32_t cur = (int32_t)((old >> sh) & 0xFFFFu);
    if (cur <= b) return cur;
    const uint32_t nw = (old & ~(0xFFFFu << sh)) | ((uint32_t)b << sh);
    const uint32_t prev = atomicCAS(wp, old, nw);
    if (prev == old) return cur;
    old = prev;
  }
}

__device__ __forceinline__ void unite_s16(uint16_t* par, int32_t a, int32_t b) {
  while (true) {
    a = find_root16_c(par, a);
    b = find_root16_c(par, b);
    if (a == b) return;
    if (a < b) { const int32_t t = a; a = b; b = t; }  // a is the larger root
    const int32_t old = atomic_min16(par, a, b);
    if (old == a) return;
    a = old;
  }
}

// ---- FillHoles + AreaThreshold in one labelling ------------------------------
// The candidates' foreground (8-connected) and background (4-connected)
// components are labelled together: every pixel belongs to exactly one
// component.  With this (8, 4) pair, the pixel directly above a component's
// root (its topmost-leftmost pixel) lies in the component that encloses it:
// a foreground component's parent is a background component, a hole's parent
// is the foreground component around it.  Background components touching
// the image border are the outside; the others are holes.  A filled object is
// a top-level foreground component (parent = outside) plus every component
// nested in it, so its area is the sum over that subtree, and the output
// mask keeps every pixel whose top-level ancestor has an area in range —
// exactly FillHoles followed by an 8-connected AreaThreshold.

// 5 KB per warp (44 warps per SM): a 16-bit forest flattened in place,
// 16-bit per-root accumulators (count <= 1024 | seed 0x8000, two per word,
// updated with 32-bit atomics), and the flattened forest then holds each
// run's root pixel as a tile-local offset (row * 32 + column) for the stores.
template <int kW>
struct __align__(16) FbSmem {
  uint16_t par[kW][1024];
  uint32_t acc[kW][512];
  uint8_t pos[kW][1024];
};

// Run-table form (w % 32 == 0): instead of a root for every pixel, each tile
// leaves its row bit masks, the ordinal of every run's local root within the
// tile's contiguous slice of the local-root list, and its border pixels'
// local roots; the roots plane then only holds the local roots themselves
// (the global forest).  A pixel's local root is re-derived from the row mask
// (run index = number of run starts up to its column) and one table entry.
struct RunTable {
  const uint32_t* rowbits;  // [tile * 32 + r]: foreground bits of row r of the tile
  const uint16_t* rtab;     // [tile * 1024 + r * 32 + k]: ordinal of run k's local root
  const int2* tinfo;        // [tile]: (first local-root slot, local-root count)
  const int32_t* lroots;    // the local-root list: (global index, accumulator) pairs,
                            // (global index, global root) after k_ccl_flatten
  int w, tiles_x;
  // the global root of q's component (valid after k_ccl_flatten)
  __device__ __forceinline__ int32_t global_root(int32_t q) const {
    const int y = q / w, x = q - y * w;
    const int tile = (y >> 5) * tiles_x + (x >> 5), r = y & 31, c = x & 31;
    const uint32_t fgb = rowbits[tile * 32 + r], bgb = ~fgb;
    const uint32_t st = (fgb & ~(fgb << 1)) | (bgb & ~(bgb << 1));
    const int k = __popc(st & ((2u << c) - 1u)) - 1;
    return lroots[2 * (tinfo[tile].x + rtab[(int64_t)tile * 1024 + r * 32 + k]) + 1];
  }
  __device__ __forceinline__ bool fg(int32_t q) const {
    const int y = q / w, x = q - y * w;
    return (rowbits[((y >> 5) * tiles_x + (x >> 5)) * 32 + (y & 31)] >> (x & 31)) & 1u;
  }
};

__global__ void __launch_bounds__(32 * kTileWarps)
k_ccl_tile_fb(const uint8_t* __restrict__ m, int h, int w, int tiles_x, int ntiles,
              int32_t* __restrict__ roots, int32_t* __restrict__ lroots,
              int32_t* __restrict__ lcount, int32_t* __restrict__ counts,
              int32_t* __restrict__ total, uint32_t* __restrict__ rowbits,
              uint16_t* __restrict__ rtab, int2* __restrict__ tinfo,
              int32_t* __restrict__ border, const uint32_t* __restrict__ in_bits) {
  pdl_enter();
  __shared__ FbSmem<kTileWarps> S;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = min(blockIdx.x * kTileWarps + wid, ntiles - 1);
  const bool active = blockIdx.x * kTileWarps + wid < ntiles;
  const int x0 = (tile % tiles_x) * 32, y0 = (tile / tiles_x) * 32;
  uint16_t* par = S.par[wid];
  uint32_t* acc = S.acc[wid];
  uint16_t* acc16 = reinterpret_cast<uint16_t*>(acc);
  uint8_t* pos = S.pos[wid];
  const FgMask pred{m};
  // 1. foreground row masks (lane r keeps row r)
  uint32_t fgb = 0;
  const int x = x0 + lane;
  const bool vec = (w & 3) == 0 && x0 + 32 <= w && (reinterpret_cast<uintptr_t>(m) & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(roots) & 15) == 0;
  if (in_bits) {
    // the candidates as row masks (k_seeded_emit), the run-table layout
    fgb = __ldg(in_bits + tile * 32 + lane);
  } else if (vec) {
    const int g = lane >> 3, cq = (lane & 7) * 4;
    uint32_t word[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int y = y0 + 4 * k + g;
      word[k] = y < h ? __ldg(reinterpret_cast<const uint32_t*>(m + (int64_t)y * w + x0 + cq)) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t fn = 0, sn = 0;
      pred.eval4(word[k], 0, 0, fn, sn);
      uint32_t v = fn << cq;
      v |= __shfl_xor_sync(kFull, v, 1);
      v |= __shfl_xor_sync(kFull, v, 2);
      v |= __shfl_xor_sync(kFull, v, 4);
      const uint32_t t = __shfl_sync(kFull, v, (lane & 3) * 8);
      if ((lane >> 2) == k) fgb = t;
    }
  } else {
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const int y = y0 + r;
      const bool f = y < h && x < w && m[(int64_t)y * w + x] != 0;
      const uint32_t b = __ballot_sync(kFull, f);
      if (lane == r) fgb = b;
    }
  }
  const int yr = y0 + lane;  // this lane's row
  const uint32_t vcols = x0 + 32 <= w ? kFull : ((1u << (w - x0)) - 1u);
  const uint32_t bgb = yr < h ? (~fgb & vcols) : 0u;
  if (yr >= h) fgb = 0;
  uint32_t seeds = 0;  // background pixels on the image border
  if (yr < h) {
    if (yr == 0 || yr == h - 1) seeds = bgb;
    else seeds = bgb & ((x0 == 0 ? 1u : 0u) | (x0 + 32 >= w ? (1u << (w - 1 - x0)) : 0u));
  }
  // 2. runs of both kinds; unions with the row above (foreground: 8-conn,
  //    background: 4-conn)
  const int rb = lane * 32;
  const uint32_t fst = fgb & ~(fgb << 1), bst = bgb & ~(bgb << 1);
  const uint32_t allst = fst | bst;
  uint32_t upf = __shfl_up_sync(kFull, fgb, 1), upb = __shfl_up_sync(kFull, bgb, 1);
  if (lane == 0) upf = upb = 0;
  const uint32_t upall = (upf & ~(upf << 1)) | (upb & ~(upb << 1));
  // the run of the row above holding column t (t in upf | upb), as a node id
  auto upper = [&](int t) -> int {
    const uint32_t U = ((upf >> t) & 1u) ? upf : upb;
    const uint32_t ust = U & ~(U << 1);
    const int su = 31 - __clz(ust & (t == 31 ? kFull : ((2u << t) - 1u)));
    return rb - 32 + __popc(upall & ((1u << su) - 1u));
  };
  auto overlaps = [&](int b) -> uint32_t {  // the row above's pixels touching run b
    const bool isf = (fgb >> b) & 1u;
    const uint32_t run = low_run((isf ? fgb : bgb) >> b) << b;
    return isf ? upf & (run | (run << 1) | (run >> 1)) : upb & run;
  };
  // every row joins its upper neighbour at once: a run's first overlapping
  // run above becomes its parent with a plain store (these links alone form
  // a forest); only further overlaps need the CAS unions on the 16-bit
  // forest.  (A schedule of log2(32) rounds kept the trees shallower but
  // left 3/4 of the lanes idle: 12 us more per 4096^2 tile.)
  uint32_t more = 0;  // runs (by index bit) with further overlaps
  {
    int k = 0;
    for (uint32_t q = allst; q; q &= q - 1, ++k) {
      const int b = __ffs(q) - 1;
      pos[rb + k] = (uint8_t)b;
      uint32_t ov = overlaps(b);
      if (!ov) {
        par[rb + k] = (uint16_t)(rb + k);
        continue;
      }
      const int t = __ffs(ov) - 1;
      const uint32_t U = ((upf >> t) & 1u) ? upf : upb;
      par[rb + k] = (uint16_t)upper(t);
      ov &= ~(low_run(U >> t) << t);
      if (ov) more |= 1u << k;
    }
  }
  __syncwarp();
  if (more) {
    int k = 0;
    for (uint32_t q = allst; q; q &= q - 1, ++k) {
      if (!((more >> k) & 1u)) continue;
      const int b = __ffs(q) - 1;
      uint32_t ov = overlaps(b);
      {
        const int t = __ffs(ov) - 1;  // the linked one
        const uint32_t U = ((upf >> t) & 1u) ? upf : upb;
        ov &= ~(low_run(U >> t) << t);
      }
      while (ov) {
        const int t = __ffs(ov) - 1;
        const uint32_t U = ((upf >> t) & 1u) ? upf : upb;
        unite_s16(par, rb + k, upper(t));
        ov &= ~(low_run(U >> t) << t);
      }
    }
  }
  __syncwarp();
  // 3. flatten; per local root: pixel count + border-background bit
  const int nruns = __popc(allst);
  // pointer jumping in place (a concurrent store only replaces a parent by an
  // ancestor): the all-at-once unions leave chains up to 31 rows deep, which
  // per-run finds walk link by link; jumping halves every chain per round
  flatten_jump16(par, rb, nruns);
  uint32_t rootm = 0;  // this row's local roots, by run index
  for (int k = 0; k < nruns; ++k)
    if (par[rb + k] == rb + k) {
      acc16[rb + k] = 0;
      rootm |= 1u << k;
    }
  const int nroot = __popc(rootm);
  __syncwarp();
  {
    int k = 0;
    for (uint32_t q = allst; q; q &= q - 1, ++k) {
      const int b = __ffs(q) - 1;
      const uint32_t run = low_run((((fgb >> b) & 1u) ? fgb : bgb) >> b) << b;
      const int32_t root = par[rb + k];
      const uint32_t sh = (root & 1) * 16;
      if (seeds & run) atomicOr(&acc[root >> 1], 0x8000u << sh);
      atomicAdd(&acc[root >> 1], (uint32_t)__popc(run) << sh);
    }
  }
  __shared__ int32_t s_res[kTileWarps + 1];
  __syncwarp();
  int base = block_reserve(active ? nroot : 0, lcount, s_res);
  if (!active) return;
  const int32_t tbase = __shfl_sync(kFull, base, 0);  // the tile's roots are contiguous
  for (uint32_t m = rootm; m; m &= m - 1) {
    const int k = __ffs(m) - 1;
    const int32_t g = (y0 + lane) * w + x0 + pos[rb + k];
    const uint32_t a = acc16[rb + k];
    lroots[2 * base] = g;
    lroots[2 * base + 1] = (int32_t)((a & 0x7FFFu) | ((a & 0x8000u) ? kSeedBit : 0u));
    counts[g] = 0;
    total[g] = 0;  // subtree areas are accumulated straight from k_fb_tree
    if (rtab) {
      roots[g] = g;
      acc16[rb + k] = (uint16_t)(base - tbase);  // the root's ordinal in the tile
    }
    ++base;
  }
  __syncwarp();
  if (rtab) {
    // 4'. row masks, tile range, border local roots, and the run table (the
    //     ordinal of every run's local root: the 2 KB forest, coalesced)
    if (rowbits != in_bits) rowbits[tile * 32 + lane] = fgb;
    const int32_t tend = __shfl_sync(kFull, base, 31);
    if (lane == 0) tinfo[tile] = make_int2(tbase, tend - tbase);
    // border entries: local root (global index), bit 31 set for foreground
    auto glob = [&](int32_t lr, uint32_t fg) {
      return (int32_t)((uint32_t)((y0 + (lr >> 5)) * w + x0 + pos[lr]) | (fg << 31));
    };
    int32_t* bd = border + (int64_t)tile * 128;
    // rows 0 and 31 (lane = column; a partial last row has no seam below),
    // columns 0 and 31 (lane = row: the row's first and last runs)
    const uint32_t below = (2u << lane) - 1u;
    const uint32_t f0 = __shfl_sync(kFull, fgb, 0), f31 = __shfl_sync(kFull, fgb, 31);
    bd[lane] = glob(par[__popc(__shfl_sync(kFull, allst, 0) & below) - 1], (f0 >> lane) & 1u);
    const uint32_t st31 = __shfl_sync(kFull, allst, 31);
    if (y0 + 31 < h) bd[32 + lane] = glob(par[31 * 32 + __popc(st31 & below) - 1], (f31 >> lane) & 1u);
    if (yr < h) {
      bd[64 + lane] = glob(par[rb], fgb & 1u);
      bd[96 + lane] = glob(par[rb + nruns - 1], fgb >> 31);
    }
    __syncwarp();
    // own entries only, four at a time with their loads in flight together
    for (int k0 = 0; k0 < nruns; k0 += 4) {
      uint32_t v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = k0 + j < nruns ? par[rb + k0 + j] : 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = acc16[v[j]];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (k0 + j < nruns) par[rb + k0 + j] = (uint16_t)v[j];
    }
    __syncwarp();
    const uint4* src = reinterpret_cast<const uint4*>(par);
    uint4* dst = reinterpret_cast<uint4*>(rtab + (int64_t)tile * 1024);
#pragma unroll
    for (int j = 0; j < 4; ++j) dst[lane + 32 * j] = src[lane + 32 * j];
    return;
  }
  // each lane rewrites only its own runs' entries
  for (int k = 0; k < nruns; ++k) {
    const int32_t lr = par[rb + k];
    par[rb + k] = (uint16_t)((lr & ~31) | pos[lr]);
  }
  __syncwarp();
  // 4. every valid pixel's local root
  if (vec) {
    const int g = lane >> 3, cq = (lane & 7) * 4;
#pragma unroll 2
    for (int k = 0; k < 8; ++k) {
      const int r = 4 * k + g;
      const int y = y0 + r;
      const uint32_t st = __shfl_sync(kFull, allst, r);
      if (y >= h) continue;
      // run of pixel cq, then the runs starting inside cq+1..cq+3 (usually
      // none: one shared-memory lookup and one index for all four pixels)
      const int i0 = r * 32 + __popc(st & ((2u << cq) - 1u)) - 1;
      const uint32_t inner = (st >> (cq + 1)) & 7u;
      int32_t o[4];
      {
        const int32_t lo = par[i0];
        o[0] = (y0 + (lo >> 5)) * w + x0 + (lo & 31);
      }
      if (!inner) {
        o[1] = o[2] = o[3] = o[0];
      } else {
#pragma unroll
        for (int j = 1; j < 4; ++j) {
          const int32_t lo = par[i0 + __popc(inner & ((1u << j) - 1u))];
          o[j] = (y0 + (lo >> 5)) * w + x0 + (lo & 31);
        }
      }
      *reinterpret_cast<int4*>(roots + (int64_t)y * w + x0 + cq) = make_int4(o[0], o[1], o[2], o[3]);
    }
  } else {
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      const uint32_t st = __shfl_sync(kFull, allst, r);
      const int y = y0 + r;
      if (y < h && x < w) {
        const int32_t lo = par[r * 32 + __popc(st & ((2u << lane) - 1u)) - 1];
        roots[(int64_t)y * w + x] = (y0 + (lo >> 5)) * w + x0 + (lo & 31);
      }
    }
  }
}

// Seams of the joint labelling: foreground pairs 8-connected, background
// pairs 4-connected, with the same redundancy skips as k_ccl_seams.
__device__ __forceinline__ void seam_fb(const uint8_t* __restrict__ m, int32_t* __restrict__ roots,
                                        int32_t p, int32_t q, int32_t p2, int32_t q2,
                                        bool has_prev, int32_t qa, bool has_qa, int32_t qb,
                                        bool has_qb, bool pref_b, bool next_b) {
  // p: seam pixel, q: its partner across the seam; p2/q2: the pair one step
  // back along the seam (valid when has_prev, same tiles); qa/qb: q's
  // neighbours one step back/forward along the seam (the 8-conn diagonals)
  const bool fp = m[p] != 0;
  const bool fq = m[q] != 0;
  if (!fp) {  // background: 4-connected straight pair only
    if (!fq && !(has_prev && !m[p2] && !m[q2])) uf_unite_g(roots, p, q);
    return;
  }
  const bool in_prev = has_prev && m[p2] != 0;  // p ~ p2 (same tile, same kind)
  const bool fqa = has_qa && m[qa] != 0;
  if (fq && !(in_prev && fqa)) uf_unite_g(roots, p, q);
  if (fqa && !in_prev && !(fq && pref_b)) uf_unite_g(roots, p, qa);
  if (has_qb && m[qb] != 0 && !(fq && next_b)) uf_unite_g(roots, p, qb);
}

__global__ void k_ccl_seams_fb(const uint8_t* __restrict__ m, int h, int w, int row_seams,
                               int32_t* __restrict__ roots) {
  pdl_enter();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if ((int)blockIdx.y < row_seams) {
    const int y = ((int)blockIdx.y + 1) * 32, x = t;
    if (x >= w || y >= h) return;
    const int32_t p = y * w + x, u = p - w;
    seam_fb(m, roots, p, u, p - 1, u - 1, (x & 31) != 0, u - 1, x > 0, u + 1, x + 1 < w,
            (x & 31) != 0, ((x + 1) & 31) != 0);
  } else {
    const int x = ((int)blockIdx.y - row_seams + 1) * 32, y = t;
    if (y >= h || x >= w) return;
    const int32_t p = y * w + x, l = p - 1;
    seam_fb(m, roots, p, l, p - w, l - w, (y & 31) != 0, l - w, y > 0, l + w, y + 1 < h,
            (y & 31) != 0, ((y + 1) & 31) != 0);
  }
}

// The same seams in the run-table form, from the tiles' border arrays alone
// (per tile 128 entries: top row, bottom row, left column, right column;
// local root with bit 31 = foreground): coalesced loads, no mask reads.  The
// pair one step back across the seam (q2) is always qa.
__device__ __forceinline__ void seam_fb_rt(int32_t* __restrict__ roots, int32_t vp, int32_t vq,
                                           int32_t vp2, bool has_prev, int32_t vqa, bool has_qa,
                                           int32_t vqb, bool has_qb, bool pref_b, bool next_b) {
  constexpr int32_t kIdx = 0x7FFFFFFF;
  const bool fp = vp < 0, fq = vq < 0;
  if (!fp) {
    if (!fq && !(has_prev && vp2 >= 0 && vqa >= 0)) uf_unite_g(roots, vp, vq);
    return;
  }
  const bool in_prev = has_prev && vp2 < 0;
  const bool fqa = has_qa && vqa < 0;
  if (fq && !(in_prev && fqa)) uf_unite_g(roots, vp & kIdx, vq & kIdx);
  if (fqa && !in_prev && !(fq && pref_b)) uf_unite_g(roots, vp & kIdx, vqa & kIdx);
  if (has_qb && vqb < 0 && !(fq && next_b)) uf_unite_g(roots, vp & kIdx, vqb & kIdx);
}

__global__ void k_ccl_seams_fb_rt(int h, int w, int tiles_x, int row_seams,
                                  const int32_t* __restrict__ border, int32_t* __restrict__ roots) {
  pdl_enter();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if ((int)blockIdx.y < row_seams) {
    const int y = ((int)blockIdx.y + 1) * 32, x = t;
    if (x >= w || y >= h) return;
    const int tb = (y >> 5) * tiles_x;  // the tile row below the seam
    const int32_t* top = border + (int64_t)(tb + (x >> 5)) * 128;
    auto bot = [&](int xx) {
      return __ldg(border + (int64_t)(tb - tiles_x + (xx >> 5)) * 128 + 32 + (xx & 31));
    };
    const bool has_prev = (x & 31) != 0, has_qa = x > 0, has_qb = x + 1 < w;
    seam_fb_rt(roots, __ldg(top + (x & 31)), bot(x), has_prev ? __ldg(top + (x & 31) - 1) : 0,
               has_prev, has_qa ? bot(x - 1) : 0, has_qa, has_qb ? bot(x + 1) : 0, has_qb,
               (x & 31) != 0, ((x + 1) & 31) != 0);
  } else {
    const int x = ((int)blockIdx.y - row_seams + 1) * 32, y = t;
    if (y >= h || x >= w) return;
    const int tc = x >> 5;  // the tile column right of the seam
    const int32_t* left = border + (int64_t)((y >> 5) * tiles_x + tc) * 128 + 64;
    auto rcol = [&](int yy) {
      return __ldg(border + (int64_t)((yy >> 5) * tiles_x + tc - 1) * 128 + 96 + (yy & 31));
    };
    const bool has_prev = (y & 31) != 0, has_qa = y > 0, has_qb = y + 1 < h;
    seam_fb_rt(roots, __ldg(left + (y & 31)), rcol(y), has_prev ? __ldg(left + (y & 31) - 1) : 0,
               has_prev, has_qa ? rcol(y - 1) : 0, has_qa, has_qb ? rcol(y + 1) : 0, has_qb,
               (y & 31) != 0, ((y + 1) & 31) != 0);
  }
}

// Top-level ancestor of every global root (-1 for the outside), and each
// root's area added into its top-level ancestor's subtree total.  With a run
// table (rt.rtab), the pixel above a root finds its local root through it.
__global__ void k_fb_tree(const int32_t* __restrict__ lroots, const int32_t* __restrict__ lcount,
                          const uint8_t* __restrict__ m, int w,
                          const int32_t* __restrict__ roots, const int32_t* __restrict__ counts,
                          int32_t* __restrict__ top, int32_t* __restrict__ total, RunTable rt) {
  pdl_enter();
  const int n = *lcount;
  auto above = [&](int32_t q) {  // global root of the pixel above q
    return rt.rtab ? rt.global_root(q - w) : root_of(roots, q - w);
  };
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t r = lroots[2 * k];
    if (lroots[2 * k + 1] != r) continue;  // not the global root
    int32_t cur = r, t = -1;
    bool fg = rt.rtab ? rt.fg(r) : m[r] != 0;
    if (fg || !(counts[r] & (int32_t)kSeedBit)) {
      for (int guard = 0; guard < (1 << 20); ++guard) {  // nesting depth, never reached
        if (fg) {
          if (cur < w) { t = cur; break; }  // touches the top border
          const int32_t b = above(cur);    // enclosing background
          if (counts[b] & (int32_t)kSeedBit) { t = cur; break; }
          cur = b;
          fg = false;
        } else {
          cur = above(cur);                 // enclosing foreground
          fg = true;
        }
      }
    }
    top[r] = t;
    // totals were cleared at every local root by k_ccl_tile_fb
    if (t >= 0) atomicAdd(total + t, counts[r] & ~(int32_t)kSeedBit);
  }
}

// The keep decision of every LOCAL root (global root -> top-level ancestor
// -> subtree area in range), stored at the local root's pixel: the per-pixel
// filter then needs one byte gather instead of three dependent i32 ones.
__global__ void k_fb_keep(const int32_t* __restrict__ lroots, const int32_t* __restrict__ lcount,
                          const int32_t* __restrict__ roots, const int32_t* __restrict__ top,
                          const int32_t* __restrict__ total, int32_t lo, int32_t hi,
                          uint8_t* __restrict__ keep) {
  pdl_enter();
  const int n = *lcount;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t lr = lroots[2 * k];
    const int32_t t = top[roots[lr]];
    bool kp = false;
    if (t >= 0) {
      const int32_t a = total[t];
      kp = a >= lo && a <= hi;
    }
    keep[lr] = kp ? 1 : 0;
  }
}

// Output of the run-table form: one warp per tile, lane = row.  A run is
// kept when its local root's keep byte (the tile's slice, staged in shared
// memory) is set; the row's kept bits become its 32 mask bytes, its
// word of the 1-bit plane, and its foreground-list entries.  List slots are
// ordered row-major over the block's tiles, so list neighbours stay row
// neighbours (the feature pass reduces runs of them); the block's entries
// are staged in shared memory and leave as one contiguous range.
__global__ void __launch_bounds__(32 * kTileWarps)
k_fb_emit(const uint32_t* __restrict__ rowbits, const uint16_t* __restrict__ rtab,
          const int2* __restrict__ tinfo, const int32_t* __restrict__ lroots,
          const int32_t* __restrict__ roots, const int32_t* __restrict__ top,
          const int32_t* __restrict__ total, int32_t lo, int32_t hi, int h, int w,
          int tiles_x, int ntiles,
          uint8_t* __restrict__ out, uint32_t* __restrict__ bits, int32_t* __restrict__ list,
          int32_t* __restrict__ count, uint32_t* __restrict__ sep_bits) {
  pdl_enter();
  __shared__ __align__(16) uint8_t s_keep[kTileWarps][1024];
  __shared__ int32_t s_cnt[32 * kTileWarps];
  __shared__ uint32_t s_kept[kTileWarps][32];
  __shared__ int32_t s_list[1024 * kTileWarps];
  __shared__ int32_t s_tot[2];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = min(blockIdx.x * kTileWarps + wid, ntiles - 1);
  const bool active = blockIdx.x * kTileWarps + wid < ntiles;
  const int x0 = (tile % tiles_x) * 32, y0 = (tile / tiles_x) * 32;
  const int y = y0 + lane;
  const bool row = active && y < h;
  {
    // keep decision of each of the tile's local roots (k_fb_keep's, inline):
    // global root -> top-level ancestor -> subtree area in range
    const int2 ti = __ldg(tinfo + tile);
    for (int j = lane; j < ti.y; j += 32) {
      const int32_t t = __ldcg(top + __ldg(lroots + 2 * (ti.x + j) + 1));
      bool kp = false;
      if (t >= 0) {
        const int32_t a = __ldcg(total + t);
        kp = a >= lo && a <= hi;
      }
      s_keep[wid][j] = kp;
    }
  }
  const uint32_t fgb = row ? __ldg(rowbits + tile * 32 + lane) : 0u;
  const uint32_t bgb = row ? ~fgb : 0u;
  uint32_t st = (fgb & ~(fgb << 1)) | (bgb & ~(bgb << 1));
  const int nruns = __popc(st);
  __syncwarp();
  uint32_t kept = 0;
  const uint16_t* rt = rtab + (int64_t)tile * 1024 + lane * 32;
  for (int k0 = 0; k0 < nruns; k0 += 8) {
    const uint4 e = __ldg(reinterpret_cast<const uint4*>(rt + k0));
    const uint32_t ew[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (k0 + j >= nruns) break;
      const uint32_t off = (ew[j >> 1] >> (16 * (j & 1))) & 0x3FFu;
      const int b = __ffs(st) - 1;
      st &= st - 1;
      const uint32_t upto = st ? (1u << (__ffs(st) - 1)) - 1u : kFull;  // run = [b, next start)
      if (s_keep[wid][off]) kept |= upto & ~((1u << b) - 1u);
    }
  }
  s_kept[wid][lane] = kept;
  if (row) {
    bits[((int64_t)y * w + x0) >> 5] = kept;
    if (sep_bits) sep_bits[((int64_t)y * w + x0) >> 5] = 0u;  // the watershed ORs into it
  }
  __syncwarp();
  // mask bytes (when a consumer reads them): 8 lanes per row, four rows per
  // store (full 32-byte sectors)
  if (active && out) {
    const int g = lane >> 3, cq = (lane & 7) * 4;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = 4 * k + g;
      if (y0 + r >= h) break;
      const uint32_t nib = (s_kept[wid][r] >> cq) & 0xFu;
      *reinterpret_cast<uint32_t*>(out + (int64_t)(y0 + r) * w + x0 + cq) =
          (nib * 0x00204081u) & 0x01010101u;
    }
  }
  // list slots: exclusive prefix over (row, warp) in row-major order; the
  // block's entries are staged in shared memory and stored contiguously
  s_cnt[lane * kTileWarps + wid] = __popc(kept);
  __syncthreads();
  if (wid == 0) {
    int32_t c[kTileWarps], sum = 0;
#pragma unroll
    for (int j = 0; j < kTileWarps; ++j) {
      c[j] = s_cnt[lane * kTileWarps + j];
      sum += c[j];
    }
    int32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const int32_t tot = __shfl_sync(kFull, incl, 31);
    int32_t base = incl - sum;
#pragma unroll
    for (int j = 0; j < kTileWarps; ++j) {
      s_cnt[lane * kTileWarps + j] = base;
      base += c[j];
    }
    if (lane == 31) {
      s_tot[0] = tot;
      s_tot[1] = tot ? atomicAdd(count, tot) : 0;
    }
  }
  __syncthreads();
  int32_t slot = s_cnt[lane * kTileWarps + wid];
  const int32_t p0 = y * w + x0;
  for (uint32_t r = kept; r; r &= r - 1) s_list[slot++] = p0 + __ffs(r) - 1;
  __syncthreads();
  const int32_t tot = s_tot[0], gbase = s_tot[1];
  for (int i = threadIdx.x; i < tot; i += blockDim.x) list[gbase + i] = s_list[i];
}

// Output mask of the joint path, 4 pixels per thread: local root -> its keep
// byte; plus the foreground list and 1-bit plane of that mask (what
// k_fg_list would build).
__global__ void __launch_bounds__(256)
k_fb_filter(int64_t n, const int32_t* __restrict__ roots, const uint8_t* __restrict__ keep,
            uint8_t* __restrict__ out, uint32_t* __restrict__ bits, int32_t* __restrict__ list,
            int32_t* __restrict__ count) {
  pdl_enter();
  __shared__ int32_t sm[9];
  const bool vec = (reinterpret_cast<uintptr_t>(out) & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(roots) & 15) == 0;
  const int lane = threadIdx.x & 31;
  for (int64_t b0 = (int64_t)blockIdx.x * 1024; b0 < n; b0 += (int64_t)gridDim.x * 1024) {
    const int64_t p0 = b0 + 4 * (int64_t)threadIdx.x;
    int32_t v[4];
    if (vec && p0 + 4 <= n) {
      const int4 r4 = __ldg(reinterpret_cast<const int4*>(roots + p0));
      v[0] = r4.x; v[1] = r4.y; v[2] = r4.z; v[3] = r4.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = p0 + k < n ? roots[p0 + k] : -1;
    }
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (v[k] >= 0 && keep[v[k]]) m |= 1u << k;
    if (vec && p0 + 4 <= n) {
      *reinterpret_cast<uint32_t*>(out + p0) =
          (m & 1u) | ((m & 2u) << 7) | ((m & 4u) << 14) | ((m & 8u) << 21);
    } else {
      for (int k = 0; k < 4 && p0 + k < n; ++k) out[p0 + k] = (uint8_t)((m >> k) & 1u);
    }
    // 32-pixel words from 8 lanes
    uint32_t wv = m << (4 * (lane & 7));
    wv |= __shfl_xor_sync(0xFFFFFFFFu, wv, 1);
    wv |= __shfl_xor_sync(0xFFFFFFFFu, wv, 2);
    wv |= __shfl_xor_sync(0xFFFFFFFFu, wv, 4);
    if (!(lane & 7) && p0 < n) bits[p0 >> 5] = wv;
    int32_t slot = block_reserve(__popc(m), count, sm);
    for (uint32_t r = m; r; r &= r - 1) list[slot++] = (int32_t)(p0 + __ffs(r) - 1);
  }
}

// ---- FillHoles by union-find: background components (4-conn) that touch the
// image border (seed bit of FgBackground) are "reached"; every other
// background pixel is a hole.
__global__ void k_fill_uf_final(int64_t n, const uint8_t* __restrict__ bin,
                                const int32_t* __restrict__ roots,
                                const int32_t* __restrict__ flag, uint8_t* __restrict__ out) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = root_of(roots, i);
    out[i] = (uint8_t)(bin[i] || (r >= 0 && !flag[r]));
  }
}

// ---- thresholded reconstruction (ReconToNuclei candidates) ----------------
// Threshold decomposition: with flat connectivity, R = recon(marker, H)
// satisfies  R(p) >= t  <=>  p lies in a conn-component of {H >= t} that
// contains a pixel with marker >= t.  With marker = max(H - h, 0) and t >= 1
// that is a pixel with H >= t + h (the seed bit of FgThresh).
// 4 pixels per thread: the root, global-root and flag gathers are issued
// stage by stage for the four, so each stage's loads are in flight together.
__global__ void k_seeded_and(int64_t n, const int32_t* __restrict__ roots,
                             const int32_t* __restrict__ flag, const uint8_t* __restrict__ tissue,
                             uint8_t* __restrict__ out) {
  pdl_enter();
  const bool vec = ((reinterpret_cast<uintptr_t>(roots) | reinterpret_cast<uintptr_t>(tissue) |
                     reinterpret_cast<uintptr_t>(out)) & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(roots) & 15) == 0;
  for (int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); i0 < n;
       i0 += 4 * (int64_t)gridDim.x * blockDim.x) {
    if (vec && i0 + 4 <= n) {
      const int4 r4 = __ldg(reinterpret_cast<const int4*>(roots + i0));
      const uint32_t t4 = __ldg(reinterpret_cast<const uint32_t*>(tissue + i0));
      int32_t v[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = v[k] >= 0 ? roots[v[k]] : -1;  // global root
      uint32_t o = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (v[k] >= 0 && flag[v[k]] && ((t4 >> (8 * k)) & 0xFFu)) o |= 1u << (8 * k);
      *reinterpret_cast<uint32_t*>(out + i0) = o;
    } else {
      for (int64_t i = i0; i < n && i < i0 + 4; ++i) {
        const int32_t r = root_of(roots, i);
        out[i] = (uint8_t)(r >= 0 && flag[r] && tissue[i]);
      }
    }
  }
}

// Tile pass + seams + flatten for any foreground predicate.  counts (if
// given) receive component sizes at the global roots, flags (if given) the
// OR of the seed bits; bitmap (if given, zeroed here) marks global roots.
// The run-table buffers for an h x w labelling (u16a: the run table, u16b:
// row masks, tile ranges and border arrays), or all-null when the form does
// not apply (w not a multiple of 32, or the tables would not fit).  The
// planes must be free from the labelling to its consumer (they are between
// the streaming kernel and the EDT, and after the watershed).
CclRuns ccl_runs_for(rtg_ctx* ctx, int64_t h, int64_t w) {
  const int64_t ntiles = ceil_div(w, 32) * ceil_div(h, 32);
  CclRuns r;
  if ((w & 31) != 0 || ntiles * 1024 > ctx->max_px) return r;
  r.rtab = ctx->u16a;
  r.rowbits = reinterpret_cast<uint32_t*>(ctx->u16b);
  r.tinfo = reinterpret_cast<int2*>(r.rowbits + ntiles * 32);
  r.border = reinterpret_cast<int32_t*>(r.tinfo + ntiles);
  return r;
}

template <class P>
int ccl_run(rtg_ctx* ctx, const P& pred, int64_t h, int64_t w, int conn, int32_t* roots,
            int32_t* counts, int32_t* flags, uint32_t* bitmap, bool prezeroed = false,
            const CclRuns& rt = CclRuns{}) {
  int32_t* lcount = ctx->misc + 8;
  if (!prezeroed) {
    // with a bitmap (the canonical labelling follows): also the look-back
    // status words of k_bm_scan
    ZeroList z{{lcount}, {sizeof(int32_t)}, 1};
    if (bitmap) {
      z.count = 0;
      ccl_label_zero(ctx, h, w, z);
    }
    RTG_TRY(zero_async(ctx, z));
  }
  const int tiles_x = (int)ceil_div(w, 32), tiles_y = (int)ceil_div(h, 32);
  const int ntiles = tiles_x * tiles_y;
  const unsigned grid = (unsigned)ceil_div(ntiles, kTileWarps);
  if (conn == 8)
    RTG_CUDA(launch_k(ctx, k_ccl_tile<8, P>, grid, 32 * kTileWarps, 0, pred, (int)h, (int)w,
                      tiles_x, ntiles, roots, ctx->lroots, lcount, counts, flags, rt));
  else
    RTG_CUDA(launch_k(ctx, k_ccl_tile<4, P>, grid, 32 * kTileWarps, 0, pred, (int)h, (int)w,
                      tiles_x, ntiles, roots, ctx->lroots, lcount, counts, flags, rt));
  RTG_LAUNCH("k_ccl_tile");
  if (tiles_x + tiles_y > 2) {
    const dim3 g((unsigned)ceil_div(h > w ? h : w, 256), (unsigned)(tiles_y - 1 + tiles_x - 1));
    const int32_t* bd = rt.border;
    if (rt.rtab && conn == 8)
      RTG_CUDA(launch_k(ctx, k_ccl_seams_rt<8>, g, 256, 0, (int)h, (int)w, tiles_x, tiles_y - 1,
                        bd, roots));
    else if (rt.rtab)
      RTG_CUDA(launch_k(ctx, k_ccl_seams_rt<4>, g, 256, 0, (int)h, (int)w, tiles_x, tiles_y - 1,
                        bd, roots));
    else if (conn == 8)
      RTG_CUDA(launch_k(ctx, k_ccl_seams<8>, g, 256, 0, (int)h, (int)w, tiles_y - 1, roots));
    else
      RTG_CUDA(launch_k(ctx, k_ccl_seams<4>, g, 256, 0, (int)h, (int)w, tiles_y - 1, roots));
    RTG_LAUNCH("k_ccl_seams");
  }
  RTG_CUDA(launch_k(ctx, k_ccl_flatten, ctx->num_sms * 4, 256, 0, ctx->lroots, lcount, roots,
                    counts, flags, bitmap, false));
  RTG_LAUNCH("k_ccl_flatten");
  return RTG_OK;
}

}  // namespace

int recon_threshold_uf(rtg_ctx* ctx, const uint8_t* hema, const uint8_t* tissue, int64_t h,
                       int64_t w, int32_t t, int32_t recon_h, int conn, uint8_t* scratch,
                       uint8_t* out, bool prezeroed, bool runs, bool bits_out,
                       uint32_t* const* in_bits) {
  (void)scratch;
  const int64_t n = h * w;
  ctx->cand_bits = false;
  if (t <= 0) {  // R >= t everywhere: the candidates are the tissue mask
    RTG_CUDA(cudaMemcpyAsync(out, tissue, (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
    return RTG_OK;
  }
  int32_t* roots = ctx->i32a;
  int32_t* flag = ctx->i32b;
  const int64_t seed_t = (int64_t)t + recon_h;  // > 255: no seed, nothing is reconstructed
  const FgThresh pred{hema, t, seed_t <= 255 ? (int32_t)seed_t : 256};
  const bool aligned = ((reinterpret_cast<uintptr_t>(tissue) | reinterpret_cast<uintptr_t>(out) |
                         reinterpret_cast<uintptr_t>(hema)) & 3) == 0;
  const CclRuns rt = runs && aligned ? ccl_runs_for(ctx, h, w) : CclRuns{};
  if (in_bits && (!rt.rtab || !bits_out))
    return fail(RTG_ERR_INTERNAL, "threshold planes without the run-table form");
  if (in_bits)
    RTG_TRY(ccl_run(ctx, FgSeedRows{in_bits[0], in_bits[1], (int)(w / 32)}, h, w, conn, roots,
                    nullptr, flag, nullptr, prezeroed, rt));
  else
    RTG_TRY(ccl_run(ctx, pred, h, w, conn, roots, nullptr, flag, nullptr, prezeroed, rt));
  if (rt.rtab) {
    const int tiles_x = (int)(w / 32);
    const int ntiles = tiles_x * (int)ceil_div(h, 32);
    ctx->cand_bits = bits_out;
    RTG_CUDA(launch_k(ctx, k_seeded_emit, (unsigned)ceil_div(ntiles, kTileWarps), 32 * kTileWarps,
                      0, rt, (const int32_t*)ctx->lroots, (const int32_t*)roots,
                      (const int32_t*)flag, tissue, (int)h, (int)w, tiles_x, ntiles, out,
                      bits_out ? reinterpret_cast<uint32_t*>(out) : (uint32_t*)nullptr,
                      in_bits ? (const uint32_t*)in_bits[2] : (const uint32_t*)nullptr));
    RTG_LAUNCH("k_seeded_emit");
    return RTG_OK;
  }
  RTG_CUDA(launch_k(ctx, k_seeded_and, grid_for(ctx, n), 256, 0, n, roots, flag, tissue, out));
  RTG_LAUNCH("k_seeded_and");
  return RTG_OK;
}

// ---- grayscale reconstruction by level decomposition -------------------------
// R = recon(J, I) (J <= I) satisfies, for every value v:
//   R(x) >= v  <=>  x's conn-component of {I >= v} holds a pixel with J >= v,
// and R only takes values of J or I.  So when J and I hold few distinct
// non-zero values (binary and few-level masks: a maze, a fill-holes style
// complement, a quantised map), R is a handful of seeded labellings, one per
// value, highest first - no wavefront, however long the propagation path.
// (The stage's ReconToNuclei uses the one-threshold case, recon_threshold_uf.)
namespace {

// The marker clip J = min(marker, I) fused with the presence bitmaps of the
// non-zero values of I (words 0-7) and J (8-15), four pixels per thread.
__device__ __forceinline__ void mark_present(uint32_t* s, uint32_t v) {
  // test before setting: each value costs one shared atomic per block
  if (v && !(s[v >> 5] & (1u << (v & 31)))) atomicOr(&s[v >> 5], 1u << (v & 31));
}

__global__ void k_clip_presence(const uint8_t* __restrict__ marker, const uint8_t* __restrict__ I,
                                int64_t n, uint8_t* __restrict__ J, uint32_t* __restrict__ bits) {
  __shared__ uint32_t s[16];
  if (threadIdx.x < 16) s[threadIdx.x] = 0;
  __syncthreads();
  const bool vec = ((reinterpret_cast<uintptr_t>(marker) | reinterpret_cast<uintptr_t>(I) |
                     reinterpret_cast<uintptr_t>(J)) & 3) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n4;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = __ldg(reinterpret_cast<const uint32_t*>(marker) + k);
    const uint32_t b = __ldg(reinterpret_cast<const uint32_t*>(I) + k);
    const uint32_t j = __vminu4(a, b);
    reinterpret_cast<uint32_t*>(J)[k] = j;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      mark_present(s, (b >> (8 * q)) & 0xFFu);
      mark_present(s + 8, (j >> (8 * q)) & 0xFFu);
    }
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = I[i], j = min((uint32_t)marker[i], b);
    J[i] = (uint8_t)j;
    mark_present(s, b);
    mark_present(s + 8, j);
  }
  __syncthreads();
  if (threadIdx.x < 16 && s[threadIdx.x]) atomicOr(bits + threadIdx.x, s[threadIdx.x]);
}

// code = (I >= v) | (J >= v) << 1, four pixels per thread.
__global__ void k_level_code(const uint8_t* __restrict__ I, const uint8_t* __restrict__ J,
                             int64_t n, uint32_t v, uint8_t* __restrict__ code) {
  const uint32_t vv = 0x01010101u * v;
  const int64_t n4 = n / 4;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n4;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = __ldg(reinterpret_cast<const uint32_t*>(I) + k);
    const uint32_t b = __ldg(reinterpret_cast<const uint32_t*>(J) + k);
    reinterpret_cast<uint32_t*>(code)[k] =
        (__vcmpgeu4(a, vv) & 0x01010101u) | (__vcmpgeu4(b, vv) & 0x02020202u);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    code[i] = (uint8_t)((I[i] >= v ? 1u : 0u) | (J[i] >= v ? 2u : 0u));
}

// out = max(out, v) on the foreground pixels of seeded components.
__global__ void k_level_assign(int64_t n, const int32_t* __restrict__ roots,
                               const int32_t* __restrict__ flag, const uint8_t* __restrict__ code,
                               uint8_t v, uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!(code[i] & 1u)) continue;
    const int32_t r = root_of(roots, i);
    if (r >= 0 && flag[r] && out[i] < v) out[i] = v;
  }
}

}  // namespace

int recon_clip_levels(rtg_ctx* ctx, const uint8_t* marker, const uint8_t* I, int64_t h,
                      int64_t w, uint8_t* J, uint8_t levels[kMaxReconLevels], int* count) {
  const int64_t n = h * w;
  *count = -1;
  RTG_CUDA(cudaMemsetAsync(ctx->level_bits, 0, 16 * sizeof(uint32_t), ctx->stream));
  k_clip_presence<<<grid_for(ctx, ceil_div(n, 4)), 256, 0, ctx->stream>>>(marker, I, n, J,
                                                                          ctx->level_bits);
  RTG_LAUNCH("k_clip_presence");
  uint32_t bits[16];
  RTG_CUDA(cudaMemcpyAsync(bits, ctx->level_bits, sizeof(bits), cudaMemcpyDeviceToHost,
                           ctx->stream));
  RTG_CUDA(cudaStreamSynchronize(ctx->stream));
  int k = 0;
  for (int v = 255; v >= 1; --v) {
    const bool present = ((bits[v >> 5] | bits[8 + (v >> 5)]) >> (v & 31)) & 1u;
    if (!present) continue;
    if (k == kMaxReconLevels) return RTG_OK;  // too many values: not this path
    levels[k++] = (uint8_t)v;
  }
  *count = k;
  return RTG_OK;
}

int recon_levels(rtg_ctx* ctx, uint8_t* J, const uint8_t* I, int64_t h, int64_t w, int conn,
                 const uint8_t* levels, int count) {
  const int64_t n = h * w;
  uint8_t* jcopy = ctx->m1;  // J is overwritten by the result
  uint8_t* code = ctx->m2;
  int32_t* roots = ctx->i32a;
  int32_t* flag = ctx->i32b;
  RTG_CUDA(cudaMemcpyAsync(jcopy, J, (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
  RTG_CUDA(cudaMemsetAsync(J, 0, (size_t)n, ctx->stream));
  for (int k = 0; k < count; ++k) {  // highest value first
    k_level_code<<<grid_for(ctx, ceil_div(n, 4)), 256, 0, ctx->stream>>>(I, jcopy, n, levels[k],
                                                                        code);
    RTG_LAUNCH("k_level_code");
    RTG_TRY(ccl_run(ctx, FgCode{code}, h, w, conn, roots, nullptr, flag, nullptr, false));
    k_level_assign<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, roots, flag, code, levels[k], J);
    RTG_LAUNCH("k_level_assign");
  }
  return RTG_OK;
}

int ccl_roots(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w, int conn,
              int32_t* roots, int32_t* counts, bool prezeroed, bool runs) {
  ctx->ccl_runs_live = runs && counts == nullptr && ccl_runs_for(ctx, h, w).rtab != nullptr;
  const CclRuns rt = ctx->ccl_runs_live ? ccl_runs_for(ctx, h, w) : CclRuns{};
  return ccl_run(ctx, FgMask{mask}, h, w, conn, roots, counts, nullptr, ctx->root_bm, prezeroed,
                 rt);
}

bool run_tables_fit(rtg_ctx* ctx, int64_t h, int64_t w) {
  return ccl_runs_for(ctx, h, w).rtab != nullptr;
}

int ccl_roots_bits(rtg_ctx* ctx, const uint32_t* bits, int64_t h, int64_t w, int conn,
                   int32_t* roots, bool prezeroed) {
  const CclRuns rt = ccl_runs_for(ctx, h, w);
  if (!rt.rtab) return fail(RTG_ERR_INTERNAL, "bit-plane labelling without run tables");
  ctx->ccl_runs_live = true;
  return ccl_run(ctx, FgBitRows{bits, (int)(w / 32)}, h, w, conn, roots, nullptr, nullptr,
                 ctx->root_bm, prezeroed, rt);
}

void ccl_label_zero(rtg_ctx* ctx, int64_t h, int64_t w, ZeroList& z) {
  const int64_t nwords = ceil_div(h * w, 32);
  const size_t nstatus = (size_t)ceil_div(nwords, kBmChunk) + 1;
  z.ptr[z.count] = ctx->misc + 8;
  z.bytes[z.count++] = sizeof(int32_t);
  z.ptr[z.count] = ctx->root_bm;
  z.bytes[z.count++] = sizeof(uint32_t) * (size_t)nwords;
  z.ptr[z.count] = ctx->scan_buf;
  z.bytes[z.count++] = sizeof(unsigned long long) * nstatus;
}

int ccl_canonical(rtg_ctx* ctx, const int32_t* roots, int64_t h, int64_t w,
                  int32_t* labels, int32_t* d_n, const FeatureAcc* clear_acc,
                  uint8_t* mask_out) {
  const int64_t n = h * w;
  const int64_t nwords = ceil_div(n, 32);
  const int nchunks = (int)ceil_div(nwords, kBmChunk);
  auto* status = reinterpret_cast<unsigned long long*>(ctx->scan_buf);  // zeroed by ccl_run
  int32_t* rank = ctx->i32c;
  RTG_CUDA(launch_k(ctx, k_bm_scan, nchunks, 256, 0, nwords, nchunks, ctx->root_bm, status,
                    ctx->root_wprefix, d_n));
  RTG_LAUNCH("k_bm_scan");
  // run-table form (ccl_roots left the tables): labels (and the ranks
  // behind them) written per tile
  const bool by_slot = ctx->ccl_runs_live;
  ctx->ccl_runs_live = false;
  if (by_slot) {
    const int tiles_x = (int)(w / 32);
    const int ntiles = tiles_x * (int)ceil_div(h, 32);
    RTG_CUDA(launch_k(ctx, k_label_emit, (unsigned)ceil_div(ntiles, kTileWarps), 32 * kTileWarps,
                      0, ccl_runs_for(ctx, h, w), (const int32_t*)ctx->lroots, roots,
                      (const uint32_t*)ctx->root_bm, (const int32_t*)ctx->root_wprefix,
                      clear_acc ? *clear_acc : ctx->acc, clear_acc != nullptr, (int)h, (int)w,
                      tiles_x, ntiles, labels, (reinterpret_cast<uintptr_t>(labels) & 15) == 0,
                      mask_out));
    RTG_LAUNCH("k_label_emit");
    return RTG_OK;
  }
  RTG_CUDA(launch_k(ctx, k_root_rank, ctx->num_sms * 4, 256, 0, ctx->lroots, ctx->misc + 8, roots,
                                                         ctx->root_bm, ctx->root_wprefix, rank,
                                                         clear_acc ? *clear_acc : ctx->acc,
                                                         clear_acc != nullptr));
  RTG_LAUNCH("k_root_rank");
  if (mask_out) return fail(RTG_ERR_INTERNAL, "mask bytes requested without run tables");
  RTG_CUDA(launch_k(ctx, k_relabel, grid_for(ctx, n), 256, 0, n, roots, rank, labels));
  RTG_LAUNCH("k_relabel");
  return RTG_OK;
}

int area_filter(rtg_ctx* ctx, const int32_t* roots, int64_t n, int32_t min_area,
                int32_t max_area, int32_t* counts, uint8_t* out) {
  // counts were accumulated at the global roots by ccl_roots(..., counts)
  RTG_CUDA(launch_k(ctx, k_area_filter, grid_for(ctx, n), 256, 0, n, roots, counts, min_area,
                                                         max_area, out));
  RTG_LAUNCH("k_area_filter");
  return RTG_OK;
}

ClearList fill_area_clear(rtg_ctx* ctx, int64_t h, int64_t w) {
  const int64_t n = h * w;
  uint32_t* bits_base = ctx->fg_bits;
  return ClearList{{ctx->misc + 4, ctx->misc + 9, reinterpret_cast<int32_t*>(bits_base),
                    reinterpret_cast<int32_t*>(bits_base + kBitPad + n / 32)},
                   {1, 1, kBitPad, kBitPad + 1},
                   4};
}

int fill_area_joint(rtg_ctx* ctx, const uint8_t* cand, int64_t h, int64_t w, int32_t min_area,
                    int32_t max_area, uint8_t* out, bool prezeroed, bool out_bytes,
                    bool sep_bits) {
  const int64_t n = h * w;
  int32_t* roots = ctx->i32a;
  int32_t* counts = ctx->i32b;
  int32_t* top = ctx->i32c;
  int32_t* total = ctx->labels;
  int32_t* lcount = ctx->misc + 9;  // its own word: cleared with the other counters
  // the stage's counters: local-root count, foreground-list count and the
  // pad words of the foreground bit plane (written by k_fb_emit / k_fb_filter)
  uint32_t* bits_base = ctx->fg_bits;
  if (!prezeroed) {
    const ClearList c = fill_area_clear(ctx, h, w);
    ZeroList z{};
    for (int r = 0; r < c.count; ++r) {
      z.ptr[r] = c.p[r];
      z.bytes[r] = sizeof(int32_t) * (uint64_t)c.n[r];
    }
    z.count = c.count;
    RTG_TRY(zero_async(ctx, z));
  }
  const int tiles_x = (int)ceil_div(w, 32), tiles_y = (int)ceil_div(h, 32);
  const int ntiles = tiles_x * tiles_y;
  // run-table form when rows of tiles are whole words of the bit plane and
  // the tables fit their planes (u16a: 1024 entries per tile; u16b: row
  // masks, then the border arrays; m2: keep bytes; all free until the EDT)
  const bool runs = ctx->label_runs && (w & 31) == 0 && (int64_t)ntiles * 1024 <= ctx->max_px;
  // the candidates may arrive as row masks (recon_threshold_uf, bits_out)
  const uint32_t* in_bits = ctx->cand_bits ? reinterpret_cast<const uint32_t*>(cand) : nullptr;
  ctx->cand_bits = false;
  if (in_bits && !runs) return fail(RTG_ERR_INTERNAL, "candidate row masks without run tables");
  uint32_t* rowbits = runs ? reinterpret_cast<uint32_t*>(ctx->u16b) : nullptr;
  if (in_bits) rowbits = const_cast<uint32_t*>(in_bits);
  uint16_t* rtab = runs ? ctx->u16a : nullptr;
  int2* tinfo = runs ? reinterpret_cast<int2*>(reinterpret_cast<uint32_t*>(ctx->u16b) +
                                               (int64_t)ntiles * 32)
                    : nullptr;
  int32_t* border = runs ? reinterpret_cast<int32_t*>(tinfo + ntiles) : nullptr;
  const unsigned tgrid = (unsigned)ceil_div(ntiles, kTileWarps);
  RTG_CUDA(launch_k(ctx, k_ccl_tile_fb, tgrid, 32 * kTileWarps, 0, cand, (int)h, (int)w, tiles_x,
                    ntiles, roots, ctx->lroots, lcount, counts, total, rowbits, rtab, tinfo, border,
                    in_bits));
  RTG_LAUNCH("k_ccl_tile_fb");
  if (tiles_x + tiles_y > 2) {
    const dim3 g((unsigned)ceil_div(h > w ? h : w, 256), (unsigned)(tiles_y - 1 + tiles_x - 1));
    if (runs)
      RTG_CUDA(launch_k(ctx, k_ccl_seams_fb_rt, g, 256, 0, (int)h, (int)w, tiles_x, tiles_y - 1,
                        (const int32_t*)border, roots));
    else
      RTG_CUDA(launch_k(ctx, k_ccl_seams_fb, g, 256, 0, cand, (int)h, (int)w, tiles_y - 1, roots));
    RTG_LAUNCH("k_ccl_seams_fb");
  }
  const int gl = ctx->num_sms * 4;
  RTG_CUDA(launch_k(ctx, k_ccl_flatten, gl, 256, 0, ctx->lroots, lcount, roots, counts,
                    (int32_t*)nullptr, (uint32_t*)nullptr, true));
  RTG_LAUNCH("k_ccl_flatten");
  prof_mark(ctx, RTG_STAGE_AREA);  // enclosure tree, subtree areas, filter
  const RunTable rt{rowbits, rtab, tinfo, ctx->lroots, (int)w, tiles_x};
  RTG_CUDA(launch_k(ctx, k_fb_tree, gl, 256, 0, ctx->lroots, lcount, cand, (int)w, roots, counts, top,
                    total, rt));
  RTG_LAUNCH("k_fb_tree");
  if (runs) {
    RTG_CUDA(launch_k(ctx, k_fb_emit, tgrid, 32 * kTileWarps, 0, (const uint32_t*)rowbits,
                      (const uint16_t*)rtab, (const int2*)tinfo, (const int32_t*)ctx->lroots,
                      (const int32_t*)roots, (const int32_t*)top, (const int32_t*)total,
                      min_area, max_area, (int)h, (int)w, tiles_x, ntiles,
                      out_bytes ? out : nullptr, bits_base + kBitPad, ctx->fg_list, ctx->misc + 4,
                      sep_bits ? ctx->sep_bits : nullptr));
    RTG_LAUNCH("k_fb_emit");
    ctx->sep_bits_live = sep_bits;
    ctx->mask_bytes_live = out_bytes;
    return RTG_OK;
  }
  uint8_t* keep = ctx->m2;  // free until the EDT's row distances
  RTG_CUDA(launch_k(ctx, k_fb_keep, gl, 256, 0, ctx->lroots, lcount, roots, top, total, min_area,
                    max_area, keep));
  RTG_LAUNCH("k_fb_keep");
  int blocks = (int)ceil_div(n, 1024);
  if (blocks > ctx->num_sms * 16) blocks = ctx->num_sms * 16;
  RTG_CUDA(launch_k(ctx, k_fb_filter, blocks, 256, 0, n, roots, (const uint8_t*)keep, out,
                                               bits_base + kBitPad, ctx->fg_list, ctx->misc + 4));
  RTG_LAUNCH("k_fb_filter");
  return RTG_OK;
}

int fill_holes_uf(rtg_ctx* ctx, const uint8_t* bin, int64_t h, int64_t w, uint8_t* scratch,
                  uint8_t* out) {
  (void)scratch;
  const int64_t n = h * w;
  int32_t* roots = ctx->i32a;
  int32_t* flag = ctx->i32b;
  RTG_TRY(ccl_run(ctx, FgBackground{bin, (int)h, (int)w}, h, w, 4, roots, nullptr, flag,
                  nullptr));
  RTG_CUDA(launch_k(ctx, k_fill_uf_final, grid_for(ctx, n), 256, 0, n, bin, roots, flag, out));
  RTG_LAUNCH("k_fill_uf_final");
  return RTG_OK;
}

}  // namespace rtg
