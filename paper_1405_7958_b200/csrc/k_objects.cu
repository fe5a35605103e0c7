// o6 PreWatershed + o7 Watershed, object-parallel (the default stage path).
//
// The paper restructures per-object work "into a set of smaller regions of
// interest: a set of minimum bounding boxes, each of which containing a
// nucleus".  The watershed of DESIGN.md §3 is exactly
// decomposable that way:
//   * objects (8-connected components of the mask) are separated by
//     background, and reconstruction / plateau BFS / marker labelling never
//     cross a zero pixel;
//   * the nearest zero of an object pixel p is 8-adjacent to p's object (walk
//     from that zero one king-step at a time towards p: every pixel on the way
//     is nearer to p, hence foreground, hence in p's object), so it lies in
//     the object's bounding box grown by one pixel;
// so each object's region (bbox + 1, clipped to the tile) is processed by one
// warp entirely in shared memory: exact EDT (column runs + bounded row search),
// HMAX and regional-maximum reconstructions (cyclic sweeps), marker labels
// (min-index propagation), steepest-ascent arrows, plateau BFS, basin
// resolution and the separation rule.  Only the region is read (mask + CCL
// roots) and only object pixels are written.
//
// Size classes: regions up to kSmallPx use 12 KB of shared memory per warp
// (4 warps / CTA); up to kBigPx one warp owns a 227 KB CTA; larger (pathological,
// e.g. long diagonal threads) run on a global-memory arena, one at a time.
//
// Roofline: HBM/L2 bound.  Algorithmic bytes: mask 1 B + roots 4 B over the
// region, separated mask 1 B (+ basin 4 B for the operator API) per object px.
#include "common.cuh"

namespace rtg {
namespace {

constexpr int kSmallPx = 2048;    // 9 B/px -> 18432 B per warp
constexpr int kWarpsSmall = 4;
constexpr int kBigPx = 25000;     // 9 B/px -> 225000 B per CTA
constexpr uint32_t kMember = 1u, kZero = 2u, kRm = 4u, kFg = 8u;

struct ObjView {
  int y0, x0, RH, RW;  // region origin (tile coords) and extent
  int32_t root;        // global CCL root of the object
};

__device__ __forceinline__ uint32_t isqrt_u64(uint64_t v) {
  uint64_t r = (uint64_t)sqrt((double)v);
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return (uint32_t)r;
}

// Directional relaxation sweeps over an RH x RW region (8-connectivity):
// cyclic down / up / right / left; each sweep relaxes every pixel from its
// three neighbours in the previous row (column).  relax(l, q0, q1, q2) gets
// the pixel and its predecessor indices (-1 when outside the region) and
// returns whether it changed the pixel.  A sweep leaves its own relation
// satisfied and a quiet sweep certifies its relation, so the fixed point is
// reached once three quiet sweeps follow the last changing one.
template <class Relax>
__device__ void region_sweeps(int RH, int RW, Relax relax) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xFFFFFFFFu;
  int quiet = 0, done = 0;
  for (int s = 0;; s = (s + 1) & 3) {
    bool ch = false;
    if (s < 2) {  // vertical: lanes over columns, rows sequential
      for (int cs = 0; cs < RW; cs += 32) {
        const int c = cs + lane;
        for (int k = 1; k < RH; ++k) {
          const int r = s == 0 ? k : RH - 1 - k;
          const int rp = s == 0 ? r - 1 : r + 1;
          if (c < RW) {
            const int lp = rp * RW + c;
            ch |= relax(r * RW + c, lp, c > 0 ? lp - 1 : -1, c + 1 < RW ? lp + 1 : -1);
          }
          __syncwarp();
        }
      }
    } else {  // horizontal: lanes over rows, columns sequential
      for (int rs = 0; rs < RH; rs += 32) {
        const int r = rs + lane;
        for (int k = 1; k < RW; ++k) {
          const int c = s == 2 ? k : RW - 1 - k;
          const int cp = s == 2 ? c - 1 : c + 1;
          if (r < RH) {
            const int lp = r * RW + cp;
            ch |= relax(r * RW + c, lp, r > 0 ? lp - RW : -1, r + 1 < RH ? lp + RW : -1);
          }
          __syncwarp();
        }
      }
    }
    ++done;
    if (__any_sync(full, ch)) quiet = 0;
    else ++quiet;
    if ((quiet >= 3 && done > quiet) || quiet >= 4) break;
  }
}

// Reconstruction by dilation of J under mask(l) on the region.
template <typename JT, class MaskFn>
__device__ void region_recon(JT* J, MaskFn mask, int RH, int RW) {
  region_sweeps(RH, RW, [&](int l, int q0, int q1, int q2) -> bool {
    uint32_t n = J[q0];
    if (q1 >= 0) n = max(n, (uint32_t)J[q1]);
    if (q2 >= 0) n = max(n, (uint32_t)J[q2]);
    const uint32_t v = J[l];
    const uint32_t nv = min(max(v, n), (uint32_t)mask(l));
    if (nv == v) return false;
    J[l] = (JT)nv;
    return true;
  });
}

// The whole per-object watershed on one region.  IdxT holds local indices
// (uint16_t when the region has < 65535 pixels, else uint32_t).
//   F8: flags; A: dq -> marker labels; B: F -> Fw; C: column EDT -> arrows;
//   D: plateau distance -> basin (local marker root)
template <typename IdxT>
__device__ void object_watershed(const ObjView& o, int h, int w, const uint8_t* __restrict__ mask,
                                 const int32_t* __restrict__ roots, int32_t ws_h,
                                 uint8_t* F8, IdxT* A, uint16_t* B, IdxT* C, IdxT* D,
                                 uint8_t* __restrict__ sep, int32_t* __restrict__ basin) {
  const int lane = threadIdx.x & 31;
  const int RH = o.RH, RW = o.RW, n = RH * RW;
  const IdxT kNone = (IdxT)~(IdxT)0;
  const uint32_t kInfD = (uint32_t)kNone - 1;  // "not reached" plateau distance

  // 1. foreground / zero flags of the region (regions lie inside the tile):
  //    flat loop over the region, 8 independent mask loads in flight per lane
  {
    int r = lane / RW, c = lane - (lane / RW) * RW;  // (r, c) of l = lane
    const int dr = 32 / RW, dc = 32 - (32 / RW) * RW;  // step of 32 pixels
    for (int l0 = 0; l0 < n; l0 += 32 * 8) {
      uint8_t v[8];
      int rr[8], cc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        rr[j] = r;
        cc[j] = c;
        const int l = l0 + lane + 32 * j;
        v[j] = l < n ? mask[(int64_t)(o.y0 + r) * w + (o.x0 + c)] : 0;
        c += dc;
        r += dr;
        if (c >= RW) { c -= RW; ++r; }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int l = l0 + lane + 32 * j;
        if (l < n) F8[rr[j] * RW + cc[j]] = v[j] ? (uint8_t)kFg : (uint8_t)kZero;
      }
    }
  }
  __syncwarp();
  // membership: the 8-connected component of the object's root pixel (its
  // minimum linear index, inside the region) as a binary reconstruction
  {
    const int lr = (o.root / w - o.y0) * RW + (o.root % w - o.x0);
    for (int l = lane; l < n; l += 32) D[l] = (IdxT)(l == lr ? 1 : 0);
    __syncwarp();
    region_recon<IdxT>(D, [&](int l) { return (F8[l] & kFg) ? 1u : 0u; }, RH, RW);
    __syncwarp();
    for (int l = lane; l < n; l += 32)
      if (D[l]) F8[l] |= (uint8_t)kMember;
    __syncwarp();
  }
  // 2. exact squared EDT: column distances (C), then bounded row search;
  //    dq = floor(4 * EDT) into A, HMAX marker max(dq - ws_h, 0) into B
  for (int cs = 0; cs < RW; cs += 32) {
    const int c = cs + lane;
    if (c < RW) {
      uint32_t run = 0xFFFFu;
      for (int r = 0; r < RH; ++r) {
        const int l = r * RW + c;
        if (F8[l] & kZero) run = 0;
        else if (run < 0xFFFFu) ++run;
        C[l] = (IdxT)run;
      }
      run = 0xFFFFu;
      for (int r = RH - 1; r >= 0; --r) {
        const int l = r * RW + c;
        if (F8[l] & kZero) run = 0;
        else if (run < 0xFFFFu) ++run;
        if (run < (uint32_t)C[l]) C[l] = (IdxT)run;
      }
    }
  }
  __syncwarp();
  for (int r = 0; r < RH; ++r) {
    for (int c = lane; c < RW; c += 32) {
      const int l = r * RW + c;
      uint32_t dq = 0, mk = 0;
      if (F8[l] & kMember) {
        uint64_t best = (uint32_t)C[l] >= 0xFFFFu ? ~0ull : (uint64_t)C[l] * (uint32_t)C[l];
        for (int k = 1; (uint64_t)k * k < best; ++k) {
          const uint64_t k2 = (uint64_t)k * k;
          if (c - k >= 0 && (uint32_t)C[l - k] < 0xFFFFu)
            best = min(best, k2 + (uint64_t)C[l - k] * (uint32_t)C[l - k]);
          if (c + k < RW && (uint32_t)C[l + k] < 0xFFFFu)
            best = min(best, k2 + (uint64_t)C[l + k] * (uint32_t)C[l + k]);
          if (c - k < 0 && c + k >= RW) break;
        }
        // no zero in the region <=> the tile has none (see file header)
        dq = best == ~0ull ? 65534u : min(isqrt_u64(16ull * best), 65534u);
        mk = dq > (uint32_t)ws_h ? dq - (uint32_t)ws_h : 0u;
      }
      A[l] = (IdxT)dq;
      B[l] = (uint16_t)mk;
    }
  }
  __syncwarp();
  // 3. HMAX: B = recon(max(dq - h, 0), dq); non-members have dq = 0 (barrier).
  //    The mask must be read as u16: A itself for u16 indices, else a u16
  //    copy in C (dead after step 2).
  const uint16_t* dq16 = reinterpret_cast<const uint16_t*>(A);
  if (sizeof(IdxT) != sizeof(uint16_t)) {
    uint16_t* cp = reinterpret_cast<uint16_t*>(C);
    for (int l = lane; l < n; l += 32) cp[l] = (uint16_t)A[l];
    __syncwarp();
    dq16 = cp;
  }
  region_recon<uint16_t>(B, [&](int l) { return (uint32_t)dq16[l]; }, RH, RW);
  __syncwarp();
  // 4. Fw = member ? F + 1 : 0
  for (int l = lane; l < n; l += 32) B[l] = (F8[l] & kMember) ? (uint16_t)(B[l] + 1) : (uint16_t)0;
  __syncwarp();
  // 5. steepest-ascent arrows (C) for pixels with a higher neighbour (D = 0);
  //    every other member pixel starts unreached (D = INF)
  for (int r = 0; r < RH; ++r) {
    for (int c = lane; c < RW; c += 32) {
      const int l = r * RW + c;
      IdxT p = kNone, d = kNone;
      const uint32_t f = B[l];
      if (f) {
        uint32_t best = f;
        int arg = -1;
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int rr = r + dy, cc = c + dx;
            if ((dy | dx) == 0 || rr < 0 || rr >= RH || cc < 0 || cc >= RW) continue;
            const int q = rr * RW + cc;
            if (B[q] > best) { best = B[q]; arg = q; }  // raster order: first max = min index
          }
        if (arg >= 0) {
          p = (IdxT)arg;
          d = 0;
        } else {
          d = (IdxT)kInfD;
        }
      }
      C[l] = p;
      D[l] = d;
    }
  }
  __syncwarp();
  // 6. plateau BFS from the pixels with a higher neighbour through
  //    equal-level member pixels.  Unreached pixels are exactly the regional
  //    maxima (their plateau has no exit) == Fw > recon(Fw - 1, Fw).
  region_sweeps(RH, RW, [&](int l, int q0, int q1, int q2) -> bool {
    const uint32_t dl = D[l];
    if (dl == 0 || dl == (uint32_t)kNone) return false;
    const uint32_t f = B[l];
    uint32_t best = dl;
    const int qs[3] = {q0, q1, q2};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int q = qs[j];
      if (q < 0 || B[q] != f) continue;
      const uint32_t dq = D[q];
      if (dq < kInfD && dq + 1 < best) best = dq + 1;
    }
    if (best >= dl) return false;
    D[l] = (IdxT)best;
    return true;
  });
  // 7. markers (self arrows) and plateau arrows: the same-level neighbour at
  //    distance delta-1 with the minimum linear index
  for (int r = 0; r < RH; ++r) {
    for (int c = lane; c < RW; c += 32) {
      const int l = r * RW + c;
      const uint32_t dl = D[l];
      if (dl == 0 || dl == (uint32_t)kNone) continue;
      if (dl == kInfD) {
        F8[l] |= (uint8_t)kRm;
        C[l] = (IdxT)l;
        continue;
      }
      const uint32_t f = B[l];
      IdxT arg = kNone;
      for (int dy = -1; dy <= 1 && arg == kNone; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int rr = r + dy, cc = c + dx;
          if ((dy | dx) == 0 || rr < 0 || rr >= RH || cc < 0 || cc >= RW) continue;
          const int q = rr * RW + cc;
          if (B[q] == f && (uint32_t)D[q] == dl - 1) { arg = (IdxT)q; break; }
        }
      C[l] = arg;
    }
  }
  __syncwarp();
  // 8. marker labels: the minimum local index of each 8-connected marker, as
  //    a reconstruction of (MAX - index) inside the marker set
  const uint32_t kMaxIdx = (uint32_t)kNone;
  for (int l = lane; l < n; l += 32) A[l] = (F8[l] & kRm) ? (IdxT)(kMaxIdx - (uint32_t)l) : (IdxT)0;
  __syncwarp();
  region_recon<IdxT>(A, [&](int l) { return (F8[l] & kRm) ? kMaxIdx : 0u; }, RH, RW);
  __syncwarp();
  // 9. basins: follow the arrows to a marker; basin = its marker's local root
  for (int l = lane; l < n; l += 32) {
    IdxT b = kNone;
    if (F8[l] & kMember) {
      uint32_t q = l;
      uint32_t nx = C[q];
      while (nx != (uint32_t)kNone && nx != q) {
        q = nx;
        nx = C[q];
      }
      if (nx == q) b = (IdxT)(kMaxIdx - (uint32_t)A[q]);
    }
    D[l] = b;
  }
  __syncwarp();
  // 10. separation + write-back (local index order == global index order)
  for (int r = 0; r < RH; ++r) {
    for (int c = lane; c < RW; c += 32) {
      const int l = r * RW + c;
      if (!(F8[l] & kMember)) continue;
      const uint32_t b = D[l];
      uint8_t keep = b != (uint32_t)kNone;
      if (keep) {
        for (int dy = -1; dy <= 1 && keep; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int rr = r + dy, cc = c + dx;
            if ((dy | dx) == 0 || rr < 0 || rr >= RH || cc < 0 || cc >= RW) continue;
            const uint32_t bq = D[rr * RW + cc];
            if (bq != (uint32_t)kNone && bq > b) { keep = 0; break; }
          }
      }
      const int64_t g = (int64_t)(o.y0 + r) * w + (o.x0 + c);
      sep[g] = keep;
      if (basin) {
        int32_t gb = 0;
        if (b != (uint32_t)kNone) {
          const int br = (int)(b / (uint32_t)RW), bc = (int)(b - (uint32_t)br * RW);
          gb = (o.y0 + br) * w + (o.x0 + bc) + 1;
        }
        basin[g] = gb;
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ bool load_view(const int32_t* __restrict__ obj_root,
                                          const int32_t* __restrict__ obj_box, int k, int h,
                                          int w, ObjView& o) {
  const int y0 = obj_box[4 * k + 0], x0 = obj_box[4 * k + 1];
  const int y1 = obj_box[4 * k + 2], x1 = obj_box[4 * k + 3];
  o.y0 = max(y0 - 1, 0);
  o.x0 = max(x0 - 1, 0);
  o.RH = min(y1 + 1, h - 1) - o.y0 + 1;
  o.RW = min(x1 + 1, w - 1) - o.x0 + 1;
  o.root = obj_root[k];
  return y1 >= y0;
}

// small regions: 4 independent warps per CTA, 12 KB of shared memory each
__global__ void __launch_bounds__(32 * kWarpsSmall)
k_obj_ws_small(int h, int w, const uint8_t* __restrict__ mask, const int32_t* __restrict__ roots,
               const int32_t* __restrict__ nobj, const int32_t* __restrict__ obj_root,
               const int32_t* __restrict__ obj_box, int32_t ws_h, uint8_t* __restrict__ sep,
               int32_t* __restrict__ basin) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wid = threadIdx.x >> 5;
  unsigned char* base = smem + (size_t)wid * (kSmallPx * 9 + 16);
  uint8_t* F8 = base;
  uint16_t* A = reinterpret_cast<uint16_t*>(base + ((kSmallPx + 15) & ~15));
  uint16_t* B = A + kSmallPx;
  uint16_t* C = B + kSmallPx;
  uint16_t* D = C + kSmallPx;
  const int total = *nobj;
  for (int k = blockIdx.x * kWarpsSmall + wid; k < total; k += gridDim.x * kWarpsSmall) {
    ObjView o;
    if (!load_view(obj_root, obj_box, k, h, w, o) || o.RH * o.RW > kSmallPx) continue;
    object_watershed<uint16_t>(o, h, w, mask, roots, ws_h, F8, A, B, C, D, sep, basin);
  }
}

// size classes beyond the per-warp budget go to compact lists:
// big ones at list[0 ..), pathological ones at list[cap-1 ..] downwards
__global__ void k_obj_classify(int h, int w, const int32_t* __restrict__ nobj,
                               const int32_t* __restrict__ obj_root,
                               const int32_t* __restrict__ obj_box, int32_t* __restrict__ list,
                               int64_t cap, int32_t* __restrict__ counts2) {
  const int total = *nobj;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    ObjView o;
    if (!load_view(obj_root, obj_box, k, h, w, o)) continue;
    const int64_t n = (int64_t)o.RH * o.RW;
    if (n <= kSmallPx) continue;
    if (n <= kBigPx) list[atomicAdd(&counts2[0], 1)] = k;
    else list[cap - 1 - atomicAdd(&counts2[1], 1)] = k;
  }
}

// big regions: one warp owns a whole CTA's shared memory
__global__ void __launch_bounds__(32)
k_obj_ws_big(int h, int w, const uint8_t* __restrict__ mask, const int32_t* __restrict__ roots,
             const int32_t* __restrict__ list, const int32_t* __restrict__ counts2,
             const int32_t* __restrict__ obj_root, const int32_t* __restrict__ obj_box,
             int32_t ws_h, uint8_t* __restrict__ sep, int32_t* __restrict__ basin) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint8_t* F8 = smem;
  uint16_t* A = reinterpret_cast<uint16_t*>(smem + ((kBigPx + 15) & ~15));
  uint16_t* B = A + kBigPx;
  uint16_t* C = B + kBigPx;
  uint16_t* D = C + kBigPx;
  const int total = counts2[0];
  for (int j = blockIdx.x; j < total; j += gridDim.x) {
    ObjView o;
    load_view(obj_root, obj_box, list[j], h, w, o);
    object_watershed<uint16_t>(o, h, w, mask, roots, ws_h, F8, A, B, C, D, sep, basin);
  }
}

// pathological regions: one warp, global-memory arena, one object at a time
__global__ void __launch_bounds__(32)
k_obj_ws_huge(int h, int w, const uint8_t* __restrict__ mask, const int32_t* __restrict__ roots,
              const int32_t* __restrict__ list, int64_t cap, const int32_t* __restrict__ counts2,
              const int32_t* __restrict__ obj_root, const int32_t* __restrict__ obj_box,
              int32_t ws_h, unsigned char* arena, int64_t arena_px, uint8_t* __restrict__ sep,
              int32_t* __restrict__ basin) {
  uint8_t* F8 = arena;
  uint32_t* A = reinterpret_cast<uint32_t*>(arena + ((arena_px + 15) & ~15ll));
  uint16_t* B = reinterpret_cast<uint16_t*>(A + arena_px);
  uint32_t* C = reinterpret_cast<uint32_t*>(B + ((arena_px + 1) & ~1ll));
  uint32_t* D = C + arena_px;
  const int total = counts2[1];
  for (int j = 0; j < total; ++j) {
    ObjView o;
    load_view(obj_root, obj_box, list[cap - 1 - j], h, w, o);
    object_watershed<uint32_t>(o, h, w, mask, roots, ws_h, F8, A, B, C, D, sep, basin);
  }
}

// object list: global roots (roots[i] == i) whose area passes the filter
// (counts == nullptr: every root); objmap[root] = object index, bbox init.
__global__ void k_obj_collect(int64_t n, const int32_t* __restrict__ roots,
                              const int32_t* __restrict__ counts, int32_t lo, int32_t hi,
                              int32_t* __restrict__ nobj, int32_t* __restrict__ obj_root,
                              int32_t* __restrict__ obj_box, int32_t* __restrict__ objmap) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (roots[i] != (int32_t)i) continue;
    if (counts) {
      const int32_t a = counts[i];
      if (a < lo || a > hi) continue;
    }
    const int k = atomicAdd(nobj, 1);
    obj_root[k] = (int32_t)i;
    obj_box[4 * k + 0] = INT32_MAX;
    obj_box[4 * k + 1] = INT32_MAX;
    obj_box[4 * k + 2] = -1;
    obj_box[4 * k + 3] = -1;
    objmap[i] = k;
  }
}

// bounding boxes of the listed objects (warp-aggregated atomics)
__global__ void __launch_bounds__(256)
k_obj_bbox(int h, int w, const uint8_t* __restrict__ mask, const int32_t* __restrict__ roots,
           const int32_t* __restrict__ objmap, int32_t* __restrict__ obj_box) {
  const unsigned full = 0xFFFFFFFFu;
  const int wpad = (w + 31) & ~31;
  for (int y = blockIdx.y; y < h; y += gridDim.y)
    for (int xb = blockIdx.x * blockDim.x; xb < wpad; xb += gridDim.x * blockDim.x) {
      const int x = xb + threadIdx.x;
      const int64_t i = (int64_t)y * w + x;
      int k = -1;
      if (x < w && mask[i]) k = objmap[root_of(roots, i)];
      const unsigned act = __ballot_sync(full, k >= 0);
      if (k < 0) continue;
      const unsigned grp = __match_any_sync(act, k);
      const int mnx = __reduce_min_sync(grp, (unsigned)x);
      const int mxx = __reduce_max_sync(grp, (unsigned)x);
      if ((threadIdx.x & 31) == __ffs(grp) - 1) {
        atomicMin(&obj_box[4 * k + 0], y);
        atomicMin(&obj_box[4 * k + 1], mnx);
        atomicMax(&obj_box[4 * k + 2], y);
        atomicMax(&obj_box[4 * k + 3], mxx);
      }
    }
}

int grid_for(rtg_ctx* ctx, int64_t n) {
  const int64_t want = ceil_div(n, 256);
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  return (int)(want < cap ? want : cap);
}

}  // namespace

int watershed_objects(rtg_ctx* ctx, const uint8_t* mask, const int32_t* roots,
                      const int32_t* counts, int32_t lo, int32_t hi, int64_t h, int64_t w,
                      int32_t ws_h, uint8_t* sep, int32_t* basin) {
  const int64_t n = h * w;
  int32_t* nobj = ctx->misc + 24;
  int32_t* objmap = ctx->i32c;
  RTG_CUDA(cudaMemsetAsync(nobj, 0, sizeof(int32_t), ctx->stream));
  RTG_CUDA(cudaMemsetAsync(sep, 0, (size_t)n, ctx->stream));
  if (basin) RTG_CUDA(cudaMemsetAsync(basin, 0, sizeof(int32_t) * (size_t)n, ctx->stream));
  k_obj_collect<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, roots, counts, lo, hi, nobj,
                                                           ctx->obj_root, ctx->obj_box, objmap);
  RTG_LAUNCH("k_obj_collect");
  const dim3 g2((unsigned)ceil_div(w, 256), (unsigned)(h < 1024 ? h : 1024));
  k_obj_bbox<<<g2, 256, 0, ctx->stream>>>((int)h, (int)w, mask, roots, objmap, ctx->obj_box);
  RTG_LAUNCH("k_obj_bbox");
  int32_t* counts2 = ctx->misc + 26;  // [0] big, [1] pathological
  RTG_CUDA(cudaMemsetAsync(counts2, 0, 2 * sizeof(int32_t), ctx->stream));
  k_obj_classify<<<ctx->num_sms * 2, 256, 0, ctx->stream>>>((int)h, (int)w, nobj, ctx->obj_root,
                                                            ctx->obj_box, ctx->obj_list,
                                                            ctx->obj_cap, counts2);
  RTG_LAUNCH("k_obj_classify");
  {
    const size_t smem = (size_t)kWarpsSmall * (kSmallPx * 9 + 16);
    RTG_SMEM_OPTIN(k_obj_ws_small, smem);
    k_obj_ws_small<<<ctx->num_sms * 16, 32 * kWarpsSmall, smem, ctx->stream>>>(
        (int)h, (int)w, mask, roots, nobj, ctx->obj_root, ctx->obj_box, ws_h, sep, basin);
    RTG_LAUNCH("k_obj_ws_small");
  }
  {
    const size_t smem = (size_t)kBigPx * 9 + 32;
    RTG_SMEM_OPTIN(k_obj_ws_big, smem);
    k_obj_ws_big<<<ctx->num_sms, 32, smem, ctx->stream>>>((int)h, (int)w, mask, roots,
                                                         ctx->obj_list, counts2, ctx->obj_root,
                                                         ctx->obj_box, ws_h, sep, basin);
    RTG_LAUNCH("k_obj_ws_big");
  }
  k_obj_ws_huge<<<1, 32, 0, ctx->stream>>>((int)h, (int)w, mask, roots, ctx->obj_list,
                                           ctx->obj_cap, counts2, ctx->obj_root, ctx->obj_box,
                                           ws_h, ctx->arena, ctx->max_px, sep, basin);
  RTG_LAUNCH("k_obj_ws_huge");
  return RTG_OK;
}

}  // namespace rtg
