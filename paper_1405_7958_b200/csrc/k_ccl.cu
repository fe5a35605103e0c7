// o5 AreaThreshold + o8 BWLabel: union-find connected-component labelling
// (Oliveira & Lotufo union-find: "a forest in which each
// pixel is a tree ... merges adjacent trees ... flattening the trees").
//
// 1. k_ccl_local   one CTA per 32x32 tile.  Each row is a ballot bit mask, so
//                  a pixel's horizontal run needs no union at all (it points at
//                  the run start); vertical unions are issued once per run
//                  adjacency; shared-memory union-find with path halving.
//                  Every tile-local root is appended to a short global list.
// 2. k_ccl_seam_*  union across tile seams in global memory (atomicMin links,
//                  larger root -> smaller root, path halving).
// 3. k_ccl_flatten_roots  only the local roots are flattened, so the forest
//                  is two-level: pixel -> local root -> global root, and
//                  consumers read root_of(i) = roots[roots[i]] instead of a
//                  full-image flatten pass.  The global root is the minimum
//                  linear index of the component.
// 4. canonical compaction: global roots ranked in raster order by a chunked
//    scan, so labels are 1..n ordered by each object's minimum pixel index
//    (scipy's ndimage.label order).
//
// Roofline: HBM/L2 bound; algorithmic bytes mask 1 B in + labels 4 B out.
#include "common.cuh"

namespace rtg {
namespace {

// Read-only shared-memory find.
__device__ __forceinline__ int32_t find_root(const int32_t* par, int32_t a) {
  int32_t p = par[a];
  while (p != a) {
    a = p;
    p = par[a];
  }
  return a;
}

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

template <int CONN>
__global__ void __launch_bounds__(256)
k_ccl_local(const uint8_t* __restrict__ mask, int h, int w, int32_t* __restrict__ roots,
            int32_t* __restrict__ lroots, int32_t* __restrict__ lcount) {
  __shared__ int32_t par[1024];
  __shared__ uint32_t rowbits[32];
  __shared__ int32_t n_local, base;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int c = threadIdx.x & 31, rb = threadIdx.x >> 5;
  if (threadIdx.x == 0) n_local = 0;
  bool fg[4];
  // 1. rows as bit masks; every pixel points at the start of its horizontal
  //    run (no unions needed inside a run)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = rb + 8 * k, y = y0 + r, x = x0 + c;
    fg[k] = y < h && x < w && mask[(int64_t)y * w + x];
    const uint32_t bits = __ballot_sync(0xFFFFFFFFu, fg[k]);
    if (c == 0) rowbits[r] = bits;
    int32_t v = -1;
    if (fg[k]) {
      const uint32_t upto = c == 31 ? 0xFFFFFFFFu : ((2u << c) - 1u);
      const uint32_t zeros = ~bits & upto;  // background at or left of c
      const int start = zeros ? 32 - __clz(zeros) : 0;
      v = r * 32 + start;
    }
    par[r * 32 + c] = v;
  }
  __syncthreads();
  // 2. one union per run adjacency with the row above: at the first pixel of
  //    every vertical overlap, plus the two diagonal run-end contacts (8-conn)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = rb + 8 * k;
    if (!fg[k] || r == 0) continue;
    const int i = r * 32 + c;
    const uint32_t up = rowbits[r - 1], cur = rowbits[r];
    const bool a = (up >> c) & 1u;
    const bool aL = c > 0 && ((up >> (c - 1)) & 1u);
    const bool aR = c < 31 && ((up >> (c + 1)) & 1u);
    const bool cL = c > 0 && ((cur >> (c - 1)) & 1u);
    const bool cR = c < 31 && ((cur >> (c + 1)) & 1u);
    if (a && !(cL && aL)) unite_s(par, i, i - 32);
    if (CONN == 8) {
      if (!a && aL && !cL) unite_s(par, i, i - 33);
      if (!a && aR && !cR) unite_s(par, i, i - 31);
    }
  }
  __syncthreads();
  // 3. flatten: read-only finds, then (after a barrier) every thread writes
  //    only its own entries — a halving store racing with a finished entry
  //    could otherwise regress it to a non-root ancestor
  int slot[4], lroot[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = rb + 8 * k, i = r * 32 + c;
    slot[k] = -1;
    lroot[k] = fg[k] ? find_root(par, i) : -1;
    if (fg[k] && lroot[k] == i) slot[k] = atomicAdd(&n_local, 1);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (fg[k]) par[(rb + 8 * k) * 32 + c] = lroot[k];
  __syncthreads();
  if (threadIdx.x == 0) base = n_local ? atomicAdd(lcount, n_local) : 0;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = rb + 8 * k, y = y0 + r, x = x0 + c;
    if (y < h && x < w) {
      int32_t out = -1;
      if (fg[k]) {
        const int32_t lr = par[r * 32 + c];
        out = (y0 + (lr >> 5)) * w + x0 + (lr & 31);
        if (slot[k] >= 0) lroots[base + slot[k]] = out;
      }
      roots[(int64_t)y * w + x] = out;
    }
  }
}

// Seams between tile rows: pixel (y, x) with y = 32k, k >= 1.
template <int CONN>
__global__ void k_ccl_seam_rows(int h, int w, int32_t* __restrict__ roots) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = (blockIdx.y + 1) * 32;
  if (x >= w || y >= h) return;
  const int32_t p = y * w + x;
  if (__ldcg(roots + p) < 0) return;
  const int32_t up = p - w;
  if (__ldcg(roots + up) >= 0) uf_unite_g(roots, p, up);
  if (CONN == 8) {
    if (x > 0 && __ldcg(roots + up - 1) >= 0) uf_unite_g(roots, p, up - 1);
    if (x + 1 < w && __ldcg(roots + up + 1) >= 0) uf_unite_g(roots, p, up + 1);
  }
}

// Seams between tile columns: pixel (y, x) with x = 32k, k >= 1.
template <int CONN>
__global__ void k_ccl_seam_cols(int h, int w, int32_t* __restrict__ roots) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  const int x = (blockIdx.y + 1) * 32;
  if (y >= h || x >= w) return;
  const int32_t p = y * w + x;
  if (__ldcg(roots + p) < 0) return;
  const int32_t lf = p - 1;
  if (__ldcg(roots + lf) >= 0) uf_unite_g(roots, p, lf);
  if (CONN == 8) {
    if (y > 0 && __ldcg(roots + lf - w) >= 0) uf_unite_g(roots, p, lf - w);
    if (y + 1 < h && __ldcg(roots + lf + w) >= 0) uf_unite_g(roots, p, lf + w);
  }
}

// Flattens the local roots only; zeroes per-root counters when requested.
__global__ void k_ccl_flatten_roots(const int32_t* __restrict__ lroots,
                                    const int32_t* __restrict__ lcount, int32_t* roots,
                                    int32_t* __restrict__ zero) {
  const int n = *lcount;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int32_t r = lroots[k];
    const int32_t g = uf_find_g(roots, r);
    if (g != r) atomicMin(roots + r, g);
    else if (zero) zero[r] = 0;
  }
}

// Area per root: warp-aggregated atomics.
__global__ void k_area_count(int64_t n, const int32_t* __restrict__ roots,
                             int32_t* __restrict__ counts) {
  const unsigned full = 0xFFFFFFFFu;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int32_t r = i < n ? root_of(roots, i) : -1;
    const unsigned act = __ballot_sync(full, r >= 0);
    if (r >= 0) {
      const unsigned grp = __match_any_sync(act, r);
      if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&counts[r], __popc(grp));
    }
  }
}

__global__ void k_area_filter(int64_t n, const int32_t* __restrict__ roots,
                              const int32_t* __restrict__ counts, int32_t lo,
                              int32_t hi, uint8_t* __restrict__ out) {
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

constexpr int kPerThread = kScanChunk / 256;  // 16 px per thread

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

// global roots are exactly the pixels with roots[i] == i
__global__ void __launch_bounds__(256)
k_root_count(int64_t n, const int32_t* __restrict__ roots,
             int32_t* __restrict__ chunk_cnt) {
  __shared__ int warp_tot[8];
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * kPerThread;
  int c = 0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    const int64_t i = base + k;
    if (i < n && roots[i] == (int32_t)i) ++c;
  }
  int total;
  block_excl_scan(c, warp_tot, total);
  if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024)
k_scan_chunks(int nchunks, const int32_t* __restrict__ cnt,
              int32_t* __restrict__ off, int32_t* __restrict__ d_total) {
  __shared__ int warp_tot[32];
  const int per = (nchunks + 1023) / 1024;
  const int b = threadIdx.x * per;
  int s = 0;
  for (int k = 0; k < per; ++k)
    if (b + k < nchunks) s += cnt[b + k];
  int total;
  int run = block_excl_scan(s, warp_tot, total);
  for (int k = 0; k < per; ++k) {
    if (b + k < nchunks) {
      off[b + k] = run;
      run += cnt[b + k];
    }
  }
  if (threadIdx.x == 0 && d_total) *d_total = total;
}

__global__ void __launch_bounds__(256)
k_root_rank(int64_t n, const int32_t* __restrict__ roots,
            const int32_t* __restrict__ chunk_off, int32_t* __restrict__ rank) {
  __shared__ int warp_tot[8];
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * kPerThread;
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    const int64_t i = base + k;
    if (i < n && roots[i] == (int32_t)i) bits |= 1u << k;
  }
  int total;
  int r = block_excl_scan(__popc(bits), warp_tot, total) + chunk_off[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    if (bits & (1u << k)) rank[base + k] = r++;
  }
}

__global__ void k_relabel(int64_t n, const int32_t* __restrict__ roots,
                          const int32_t* __restrict__ rank,
                          int32_t* __restrict__ labels) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = root_of(roots, i);
    labels[i] = r >= 0 ? rank[r] + 1 : 0;
  }
}

int grid_for(rtg_ctx* ctx, int64_t n) {
  const int64_t want = ceil_div(n, 256);
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  return (int)(want < cap ? want : cap);
}

// ---- FillHoles by union-find: background components (4-conn) that touch the
// tile border are "reached"; every other background pixel is a hole.
__global__ void k_invert(int64_t n, const uint8_t* __restrict__ in, uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)(in[i] == 0);
}

__global__ void k_mark_border_roots(int h, int w, const int32_t* __restrict__ roots,
                                    int32_t* __restrict__ flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;  // walks the perimeter
  const int per = 2 * (h + w);
  if (k >= per) return;
  int y, x;
  if (k < w) { y = 0; x = k; }
  else if (k < 2 * w) { y = h - 1; x = k - w; }
  else if (k < 2 * w + h) { y = k - 2 * w; x = 0; }
  else { y = k - 2 * w - h; x = w - 1; }
  const int32_t r = root_of(roots, (int64_t)y * w + x);
  if (r >= 0) flag[r] = 1;
}

__global__ void k_fill_uf_final(int64_t n, const uint8_t* __restrict__ bin,
                                const int32_t* __restrict__ roots,
                                const int32_t* __restrict__ flag, uint8_t* __restrict__ out) {
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
// that is a pixel with H >= t + h.
__global__ void k_thresh(int64_t n, const uint8_t* __restrict__ hema, int32_t t,
                         uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)(hema[i] >= t);
}

__global__ void k_mark_seeds(int64_t n, const uint8_t* __restrict__ hema, int32_t seed_t,
                             const int32_t* __restrict__ roots, int32_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (hema[i] >= seed_t) {
      const int32_t r = root_of(roots, i);
      if (r >= 0 && !flag[r]) flag[r] = 1;
    }
  }
}

__global__ void k_seeded_and(int64_t n, const int32_t* __restrict__ roots,
                             const int32_t* __restrict__ flag, const uint8_t* __restrict__ tissue,
                             uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = root_of(roots, i);
    out[i] = (uint8_t)(r >= 0 && flag[r] && tissue[i]);
  }
}

}  // namespace

int recon_threshold_uf(rtg_ctx* ctx, const uint8_t* hema, const uint8_t* tissue, int64_t h,
                       int64_t w, int32_t t, int32_t recon_h, int conn, uint8_t* scratch,
                       uint8_t* out) {
  const int64_t n = h * w;
  if (t <= 0) {  // R >= t everywhere: the candidates are the tissue mask
    RTG_CUDA(cudaMemcpyAsync(out, tissue, (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
    return RTG_OK;
  }
  k_thresh<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, hema, t, scratch);
  RTG_LAUNCH("k_thresh");
  int32_t* roots = ctx->i32a;
  int32_t* flag = ctx->i32b;
  RTG_TRY(ccl_roots(ctx, scratch, h, w, conn, roots, flag));
  const int64_t seed_t = (int64_t)t + recon_h;
  if (seed_t <= 255) {
    k_mark_seeds<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, hema, (int32_t)seed_t, roots, flag);
    RTG_LAUNCH("k_mark_seeds");
  }
  k_seeded_and<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, roots, flag, tissue, out);
  RTG_LAUNCH("k_seeded_and");
  return RTG_OK;
}

int ccl_roots(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w, int conn,
              int32_t* roots, int32_t* zero_at_roots) {
  int32_t* lcount = ctx->misc + 8;
  RTG_CUDA(cudaMemsetAsync(lcount, 0, sizeof(int32_t), ctx->stream));
  const dim3 tiles((unsigned)ceil_div(w, 32), (unsigned)ceil_div(h, 32));
  if (conn == 8)
    k_ccl_local<8><<<tiles, 256, 0, ctx->stream>>>(mask, (int)h, (int)w, roots, ctx->lroots, lcount);
  else
    k_ccl_local<4><<<tiles, 256, 0, ctx->stream>>>(mask, (int)h, (int)w, roots, ctx->lroots, lcount);
  RTG_LAUNCH("k_ccl_local");
  if (tiles.y > 1) {
    const dim3 g((unsigned)ceil_div(w, 256), tiles.y - 1);
    if (conn == 8) k_ccl_seam_rows<8><<<g, 256, 0, ctx->stream>>>((int)h, (int)w, roots);
    else k_ccl_seam_rows<4><<<g, 256, 0, ctx->stream>>>((int)h, (int)w, roots);
    RTG_LAUNCH("k_ccl_seam_rows");
  }
  if (tiles.x > 1) {
    const dim3 g((unsigned)ceil_div(h, 256), tiles.x - 1);
    if (conn == 8) k_ccl_seam_cols<8><<<g, 256, 0, ctx->stream>>>((int)h, (int)w, roots);
    else k_ccl_seam_cols<4><<<g, 256, 0, ctx->stream>>>((int)h, (int)w, roots);
    RTG_LAUNCH("k_ccl_seam_cols");
  }
  k_ccl_flatten_roots<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->lroots, lcount, roots,
                                                                 zero_at_roots);
  RTG_LAUNCH("k_ccl_flatten_roots");
  return RTG_OK;
}

int ccl_canonical(rtg_ctx* ctx, const int32_t* roots, int64_t h, int64_t w,
                  int32_t* labels, int32_t* d_n) {
  const int64_t n = h * w;
  const int nchunks = (int)ceil_div(n, kScanChunk);
  int32_t* cnt = ctx->scan_buf;
  int32_t* off = ctx->scan_buf + nchunks;
  int32_t* rank = ctx->i32c;
  k_root_count<<<nchunks, 256, 0, ctx->stream>>>(n, roots, cnt);
  RTG_LAUNCH("k_root_count");
  k_scan_chunks<<<1, 1024, 0, ctx->stream>>>(nchunks, cnt, off, d_n);
  RTG_LAUNCH("k_scan_chunks");
  k_root_rank<<<nchunks, 256, 0, ctx->stream>>>(n, roots, off, rank);
  RTG_LAUNCH("k_root_rank");
  k_relabel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, roots, rank, labels);
  RTG_LAUNCH("k_relabel");
  return RTG_OK;
}

int area_filter(rtg_ctx* ctx, const int32_t* roots, int64_t n, int32_t min_area,
                int32_t max_area, int32_t* counts, uint8_t* out) {
  // counts were zeroed at the global roots by ccl_roots(..., counts)
  k_area_count<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, roots, counts);
  RTG_LAUNCH("k_area_count");
  k_area_filter<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, roots, counts, min_area,
                                                         max_area, out);
  RTG_LAUNCH("k_area_filter");
  return RTG_OK;
}

int fill_holes_uf(rtg_ctx* ctx, const uint8_t* bin, int64_t h, int64_t w, uint8_t* scratch,
                  uint8_t* out) {
  const int64_t n = h * w;
  k_invert<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, bin, scratch);
  RTG_LAUNCH("k_invert");
  int32_t* roots = ctx->i32a;
  int32_t* flag = ctx->i32b;
  RTG_TRY(ccl_roots(ctx, scratch, h, w, 4, roots, flag));  // flags zeroed at roots
  const int per = (int)(2 * (h + w));
  k_mark_border_roots<<<(unsigned)ceil_div(per, 256), 256, 0, ctx->stream>>>((int)h, (int)w,
                                                                             roots, flag);
  RTG_LAUNCH("k_mark_border_roots");
  k_fill_uf_final<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, bin, roots, flag, out);
  RTG_LAUNCH("k_fill_uf_final");
  return RTG_OK;
}

}  // namespace rtg
