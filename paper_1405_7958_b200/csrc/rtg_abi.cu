// extern "C" boundary (include/rtg.h): context arena, error mapping and the
// stage pipeline.  Every compute entry point requires a CUDA device; there is
// no CPU fallback anywhere in this library.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>

#include "common.cuh"

namespace rtg {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  const std::string msg = std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                          cudaGetErrorString(e) + ")";
  if (e == cudaErrorMemoryAllocation) return fail(RTG_ERR_OUT_OF_MEMORY, msg);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ||
      e == cudaErrorInvalidDevice)
    return fail(RTG_ERR_NO_DEVICE, msg);
  return fail(RTG_ERR_DEVICE, msg);
}

cudaError_t smem_optin(const void* kernel, int device, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kernel, device})) return cudaSuccess;
  // the attribute applies to the current device: the caller's ctx device
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return e;
  if (cur != device && (e = cudaSetDevice(device)) != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (cur != device) cudaSetDevice(cur);
  if (e == cudaSuccess) done.insert({kernel, device});
  return e;
}

int check_ctx(rtg_ctx* ctx, int64_t h, int64_t w) {
  if (!ctx) return fail(RTG_ERR_INVALID_ARG, "null rtg_ctx");
  if (h <= 0 || w <= 0) return fail(RTG_ERR_DIMENSION, "tile extent must be positive");
  if (h > ctx->max_h || w > ctx->max_w || h * w > ctx->max_px)
    return fail(RTG_ERR_DIMENSION, "tile " + std::to_string(h) + "x" + std::to_string(w) +
                                       " exceeds context capacity " +
                                       std::to_string(ctx->max_h) + "x" +
                                       std::to_string(ctx->max_w));
  RTG_CUDA(cudaSetDevice(ctx->device));
  return RTG_OK;
}

void prof_mark(rtg_ctx* ctx, int stage) {
  if (!ctx->prof || ctx->prof_used >= ctx->prof_cap) return;
  const int k = ctx->prof_used++;
  cudaEventRecord(ctx->prof_ev[k], ctx->stream);
  ctx->prof_stage[k] = stage;
}

namespace {

int check_params_impl(const rtg_params* p) {
  if (p && p->texture != 0 && p->texture != 1)
    return fail(RTG_ERR_INVALID_ARG, "params.texture must be 0 or 1");
  if (!p) return fail(RTG_ERR_INVALID_ARG, "null rtg_params");
  if (p->recon_conn != 4 && p->recon_conn != 8)
    return fail(RTG_ERR_INVALID_ARG, "recon_conn must be 4 or 8");
  if (!(p->h_scale > 0.0)) return fail(RTG_ERR_INVALID_ARG, "h_scale must be positive");
  if (p->min_area < 0 || p->max_area < p->min_area)
    return fail(RTG_ERR_INVALID_ARG, "need 0 <= min_area <= max_area");
  if (p->ws_h < 0 || p->recon_h < 0) return fail(RTG_ERR_INVALID_ARG, "heights must be >= 0");
  return RTG_OK;
}

constexpr unsigned char kGuardByte = 0xA5;

template <typename T>
int dalloc(rtg_ctx* c, T** p, size_t count, const char* name) {
  const size_t bytes = sizeof(T) * (count ? count : 1);
  RTG_CUDA(cudaMalloc((void**)p, bytes + c->guard_bytes));
  if (c->guard_bytes) {
    unsigned char* end = reinterpret_cast<unsigned char*>(*p) + bytes;
    RTG_CUDA(cudaMemset(end, kGuardByte, c->guard_bytes));
    c->guards.push_back({end, name});
  }
  return RTG_OK;
}
#define DALLOC(field, count) dalloc(c, &c->field, (count), #field)

template <typename T>
__global__ void k_clip_copy(const T* __restrict__ marker, const T* __restrict__ mask,
                            int64_t n, T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T a = marker[i], b = mask[i];
    out[i] = a < b ? a : b;
  }
}

int grid_for(rtg_ctx* ctx, int64_t n) {
  const int64_t want = ceil_div(n, 256);
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  return (int)(want < cap ? want : cap);
}

// o4 with the context's implementation choice; `out` may be any buffer except
// `bin` (ctx->m2 is the IWPP J plane / union-find scratch when out differs).
int run_fill_holes(rtg_ctx* ctx, const uint8_t* bin, int64_t h, int64_t w, uint8_t* out) {
  if (ctx->fill_impl == 1) return iwpp_fill_holes(ctx, bin, out == bin ? ctx->m2 : out, h, w, out);
  return fill_holes_uf(ctx, bin, h, w, out, out);
}

__global__ void k_rows_pack(const int32_t* __restrict__ d_n, int32_t cap,
                            const float* __restrict__ shape, const float* __restrict__ tex,
                            float* __restrict__ out);

// The stage: o1 .. o9 on device buffers, all asynchronous on ctx->stream.
int pipeline(rtg_ctx* ctx, const uint8_t* d_rgb, int64_t h, int64_t w, int64_t pitch,
             const rtg_params* p, uint8_t* d_mask, int32_t* d_labels, uint8_t* d_hema,
             float* d_features, int32_t* d_n, bool with_features) {
  uint8_t* hema = d_hema ? d_hema : ctx->hema;
  uint8_t* mask = d_mask ? d_mask : ctx->m4;
  int32_t* labels = d_labels ? d_labels : ctx->labels;
  int32_t* n_out = d_n ? d_n : ctx->misc;
  const bool iwpp_recon = ctx->recon_impl == 1;
  ctx->cand_bits = false;
  ctx->ccl_runs_live = false;
  ctx->sep_bits_live = false;
  ctx->mask_bytes_live = false;
  // o1+o2: hematoxylin, tissue (+ the HMAX marker for the grayscale IWPP path)
  prof_mark(ctx, RTG_STAGE_COLORDECONV);
  // the streaming kernel's first CTA clears the reconstruction CCL's
  // local-root count (uf path) and the joint fill/area stage's counters
  const bool joint = ctx->fill_impl == 0 && ctx->ws_impl == 0;
  ClearList cl = joint ? fill_area_clear(ctx, h, w) : ClearList{};
  if (!iwpp_recon) {
    cl.p[cl.count] = ctx->misc + 8;
    cl.n[cl.count++] = 1;
  }
  // run-table path: the streaming kernel also emits ReconToNuclei's two
  // threshold planes and the tissue plane as 1-bit planes (in m3, free
  // until the joint fill/area stage) instead of the tissue bytes
  const int64_t nw32 = h * w / 32;
  uint32_t* rbits[3] = {reinterpret_cast<uint32_t*>(ctx->m3),
                        reinterpret_cast<uint32_t*>(ctx->m3) + nw32,
                        reinterpret_cast<uint32_t*>(ctx->m3) + 2 * nw32};
  const bool want_bits = !iwpp_recon && joint && ctx->label_runs && p->nuc_thresh > 0 &&
                         run_tables_fit(ctx, h, w);
  bool have_bits = false;
  RTG_TRY(launch_colordeconv(ctx, d_rgb, h, w, pitch, p, hema, iwpp_recon ? ctx->recon : nullptr,
                             ctx->tissue, &cl, want_bits ? rbits : nullptr, &have_bits));
  // o3 ReconToNuclei: candidates = recon(max(H - h, 0), H) >= nuc_thresh && tissue
  prof_mark(ctx, RTG_STAGE_RECON);
  if (iwpp_recon) {
    RTG_TRY(iwpp_recon_u8(ctx, ctx->recon, hema, h, w, p->recon_conn));
    RTG_TRY(launch_candidate(ctx, ctx->recon, ctx->tissue, h * w, p->nuc_thresh, ctx->m1));
  } else {
    RTG_TRY(recon_threshold_uf(ctx, hema, ctx->tissue, h, w, p->nuc_thresh, p->recon_h,
                               p->recon_conn, ctx->m1, ctx->m1, /*prezeroed=*/true,
                               ctx->label_runs != 0, /*bits_out=*/joint,
                               have_bits ? rbits : nullptr));
  }
  if (ctx->fill_impl == 0 && ctx->ws_impl == 0) {
    // o4 FillHoles + o5 AreaThreshold as one joint labelling (the filled
    // mask itself is never materialised)
    prof_mark(ctx, RTG_STAGE_FILL_HOLES);
    // the mask bytes: the IWPP HMAX path reads them (whole-tile EDT), the
    // sparse EDT reuses them in place as its row-distance plane
    // the separated mask goes through a bit plane when the labelling can
    // write its bytes (4-byte stores)
    RTG_TRY(fill_area_joint(ctx, ctx->m1, h, w, p->min_area, p->max_area, ctx->m3,
                            /*prezeroed=*/true, /*out_bytes=*/true,
                            /*sep_bits=*/(reinterpret_cast<uintptr_t>(mask) & 3) == 0));
  } else {
    // o4 FillHoles of the nucleus candidates
    prof_mark(ctx, RTG_STAGE_FILL_HOLES);
    RTG_TRY(run_fill_holes(ctx, ctx->m1, h, w, ctx->m2));
    // o5 AreaThreshold (its forest + counts also feed the object-parallel
    // watershed)
    prof_mark(ctx, RTG_STAGE_AREA);
    RTG_TRY(ccl_roots(ctx, ctx->m2, h, w, 8, ctx->i32a, ctx->i32b));
    RTG_TRY(area_filter(ctx, ctx->i32a, h * w, p->min_area, p->max_area, ctx->i32b, ctx->m3));
  }
  // o6 + o7 PreWatershed + Watershed (basin ids staged in the labels buffer);
  // watershed() marks its own EDT / MARKERS / WATERSHED stages
  if (ctx->ws_impl == 0) {
    // the joint fill/area path already listed the foreground of m3
    const bool listed = ctx->fill_impl == 0;
    RTG_TRY(watershed(ctx, ctx->m3, h, w, p->ws_h, mask, labels, false, listed));
  } else {
    // the area-threshold forest and counts already name the kept objects
    prof_mark(ctx, RTG_STAGE_WATERSHED);
    RTG_TRY(watershed_objects(ctx, ctx->m3, ctx->i32a, ctx->i32b, p->min_area, p->max_area, h,
                              w, p->ws_h, mask, nullptr));
  }
  // o8 BWLabel (canonical)
  prof_mark(ctx, RTG_STAGE_LABEL);
  // the tiled watershed cleared the labelling's counters with its own
  // (run-table path: the watershed left the separated mask as a bit plane;
  // the labelling reads it and writes the mask bytes with the labels)
  const bool sep_bits = ctx->sep_bits_live;
  ctx->sep_bits_live = false;
  if (sep_bits)
    RTG_TRY(ccl_roots_bits(ctx, ctx->sep_bits, h, w, 8, ctx->i32a, /*prezeroed=*/true));
  else
    RTG_TRY(ccl_roots(ctx, mask, h, w, 8, ctx->i32a, nullptr, ctx->ws_impl == 0,
                      ctx->label_runs != 0));
  // the ranking pass also resets the feature accumulators of every label
  RTG_TRY(ccl_canonical(ctx, ctx->i32a, h, w, labels, n_out, with_features ? &ctx->acc : nullptr,
                        sep_bits ? mask : nullptr));
  // o9 features
  if (with_features) {
    prof_mark(ctx, RTG_STAGE_FEATURES);
    // the tiled watershed left the foreground list of the area mask (a
    // superset of the labelled pixels)
    const bool sparse = ctx->ws_impl == 0;
    float* shape_rows = p->texture ? ctx->feat20 : d_features;
    RTG_TRY(features(ctx, labels, hema, h, w, n_out, shape_rows, sparse ? ctx->fg_list : nullptr,
                     sparse ? ctx->misc + 4 : nullptr, /*acc_cleared=*/true));
    if (p->texture) {
      // f4: Canny + histogram / co-occurrence columns appended to every row
      prof_mark(ctx, RTG_STAGE_TEXTURE);
      RTG_TRY(texture(ctx, labels, hema, h, w, n_out, ctx->tex14, &ctx->acc));
      RTG_CUDA(launch_k(ctx, k_rows_pack, (unsigned)ceil_div(ctx->max_objects, 256), 256, 0,
                        n_out, ctx->max_objects, ctx->feat20, ctx->tex14, d_features));
      RTG_LAUNCH("k_rows_pack");
    }
  }
  prof_mark(ctx, -1);
  return RTG_OK;
}

constexpr int kGraphCap = 256;

// Replays the whole-tile pipeline as a CUDA graph.  The pipeline makes no
// host-side decisions (persistent IWPP queues, device-side counts), so one
// capture per distinct argument tuple is exact; the cache holds kGraphCap
// instantiated graphs (least recently used evicted).
int pipeline_graph(rtg_ctx* ctx, const uint8_t* d_rgb, int64_t h, int64_t w, int64_t pitch,
                   const rtg_params* p, uint8_t* d_mask, int32_t* d_labels, uint8_t* d_hema,
                   float* d_features, int32_t* d_n) {
  std::string key(sizeof(rtg_params) + 12 * sizeof(int64_t), '\0');
  const int64_t fields[12] = {(int64_t)d_rgb, h, w, pitch, (int64_t)d_mask, (int64_t)d_labels,
                              (int64_t)d_hema, (int64_t)d_features, (int64_t)d_n,
                              (int64_t)ctx->fill_impl, (int64_t)ctx->stream,
                              (int64_t)ctx->recon_impl | ((int64_t)ctx->ws_impl << 8) |
                                  ((int64_t)ctx->hmax_impl << 16) |
                                  ((int64_t)ctx->use_pdl << 24) |
                                  ((int64_t)ctx->stream_impl << 32) |
                                  ((int64_t)ctx->label_runs << 40)};
  std::memcpy(&key[0], fields, sizeof(fields));
  std::memcpy(&key[sizeof(fields)], p, sizeof(rtg_params));
  if (!ctx->graphs) ctx->graphs = new rtg_ctx::GraphEntry[kGraphCap];
  ++ctx->graph_clock;
  for (int i = 0; i < ctx->n_graphs; ++i) {
    rtg_ctx::GraphEntry& g = ctx->graphs[i];
    if (g.key == key) {
      g.last_use = ctx->graph_clock;
      RTG_CUDA(cudaGraphLaunch(g.exec, ctx->stream));
      ctx->launches += g.launches;
      return RTG_OK;
    }
  }
  // capture (kernels are not executed while capturing)
  const int64_t before = ctx->launches;
  RTG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  const int st = pipeline(ctx, d_rgb, h, w, pitch, p, d_mask, d_labels, d_hema, d_features, d_n,
                          true);
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
  if (st != RTG_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
  const int64_t per_replay = ctx->launches - before;
  ctx->launches = before;
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) return cuda_fail(ie, "cudaGraphInstantiate");
  int slot = ctx->n_graphs;
  if (slot == kGraphCap) {
    slot = 0;
    for (int i = 1; i < kGraphCap; ++i)
      if (ctx->graphs[i].last_use < ctx->graphs[slot].last_use) slot = i;
    cudaGraphExecDestroy(ctx->graphs[slot].exec);
  } else {
    ++ctx->n_graphs;
  }
  ctx->graphs[slot].key = key;
  ctx->graphs[slot].exec = exec;
  ctx->graphs[slot].launches = per_replay;
  ctx->graphs[slot].last_use = ctx->graph_clock;
  RTG_CUDA(cudaGraphLaunch(exec, ctx->stream));
  ctx->launches += per_replay;
  return RTG_OK;
}

int upload_rgb(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w, int64_t pitch) {
  if (!rgb) return fail(RTG_ERR_INVALID_ARG, "null rgb");
  if (pitch < 3 * w) return fail(RTG_ERR_DIMENSION, "pitch_bytes < 3 * w");
  if (pitch == 3 * w) {
    RTG_CUDA(cudaMemcpyAsync(ctx->rgb, rgb, (size_t)(3 * h * w), cudaMemcpyHostToDevice,
                             ctx->stream));
  } else {
    RTG_CUDA(cudaMemcpy2DAsync(ctx->rgb, (size_t)(3 * w), rgb, (size_t)pitch, (size_t)(3 * w),
                               (size_t)h, cudaMemcpyHostToDevice, ctx->stream));
  }
  return RTG_OK;
}

// Copies the first min(n, cap) feature rows (n = device object count) into
// pinned host memory with a kernel (zero-copy stores: exactly the rows that
// exist cross PCIe); pageable destinations get a cudaMemcpyAsync of cap rows.
// Rows are an even number of floats (20 or 34): float2 stores.
__global__ void k_rows_to_host(const float2* __restrict__ src, const int32_t* __restrict__ d_n,
                               int32_t cap, int cols, float2* __restrict__ dst) {
  const int64_t rows = min(*d_n, cap);
  const int64_t n2 = rows * (cols / 2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Interleaves the shape / intensity rows and the texture rows of the first
// min(n, cap) objects into RTG_MAX_FEATURE_COLUMNS-wide rows.
__global__ void k_rows_pack(const int32_t* __restrict__ d_n, int32_t cap,
                            const float* __restrict__ shape, const float* __restrict__ tex,
                            float* __restrict__ out) {
  pdl_enter();
  const int n = min(*d_n, cap);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    float* o = out + (int64_t)k * RTG_MAX_FEATURE_COLUMNS;
#pragma unroll
    for (int j = 0; j < RTG_NUM_FEATURES; ++j) o[j] = shape[(int64_t)k * RTG_NUM_FEATURES + j];
#pragma unroll
    for (int j = 0; j < RTG_NUM_TEXTURE; ++j)
      o[RTG_NUM_FEATURES + j] = tex[(int64_t)k * RTG_NUM_TEXTURE + j];
  }
}

}  // namespace

int rows_to_host(rtg_ctx* ctx, cudaStream_t stream, const float* src, const int32_t* d_n,
                 float* dst, int32_t cap, int cols) {
  cudaPointerAttributes a{};
  const cudaError_t e = cudaPointerGetAttributes(&a, dst);
  if (e == cudaSuccess && a.type == cudaMemoryTypeHost && a.devicePointer &&
      (reinterpret_cast<uintptr_t>(a.devicePointer) & 7) == 0) {
    k_rows_to_host<<<64, 256, 0, stream>>>(reinterpret_cast<const float2*>(src), d_n, cap, cols,
                                           static_cast<float2*>(a.devicePointer));
    RTG_LAUNCH("k_rows_to_host");
    return RTG_OK;
  }
  cudaGetLastError();  // clear a failed attribute query on pageable memory
  RTG_CUDA(cudaMemcpyAsync(dst, src, sizeof(float) * (size_t)cols * (size_t)cap,
                           cudaMemcpyDeviceToHost, stream));
  return RTG_OK;
}

int run_stage(rtg_ctx* ctx, const uint8_t* d_rgb, int64_t h, int64_t w, int64_t pitch,
              const rtg_params* p, uint8_t* d_mask, int32_t* d_labels, uint8_t* d_hema,
              float* d_features, int32_t* d_n) {
  if (ctx->use_graphs && !ctx->prof)
    return pipeline_graph(ctx, d_rgb, h, w, pitch, p, d_mask, d_labels, d_hema, d_features, d_n);
  return pipeline(ctx, d_rgb, h, w, pitch, p, d_mask, d_labels, d_hema, d_features, d_n, true);
}

int check_params(const rtg_params* p) { return check_params_impl(p); }

namespace {
}  // namespace
}  // namespace rtg

using namespace rtg;

extern "C" {

const char* rtg_last_error(void) { return g_last_error.c_str(); }

int rtg_params_default(rtg_params* p) {
  if (!p) return fail(RTG_ERR_INVALID_ARG, "null rtg_params");
  std::memset(p, 0, sizeof(*p));
  // column 0 of inv(row-normalised Ruifrok-Johnston H&E stain matrix)
  p->h_coef[0] = 1.874787447891341;
  p->h_coef[1] = -0.06579592311838535;
  p->h_coef[2] = -0.6008832496835673;
  p->h_scale = 1.25;
  p->bg_thresh = 215;
  p->rbc_rg10 = 25;
  p->rbc_rb10 = 22;
  p->recon_h = 24;
  p->recon_conn = 8;
  p->nuc_thresh = 70;
  p->min_area = 24;
  p->max_area = 2500;
  p->ws_h = 3;
  return RTG_OK;
}

int rtg_feature_columns(const rtg_params* p, int32_t* cols) {
  if (!p || !cols) return fail(RTG_ERR_INVALID_ARG, "null argument");
  RTG_TRY(check_params(p));
  *cols = feature_cols(p);
  return RTG_OK;
}

int rtg_device_count(int* n) {
  if (!n) return fail(RTG_ERR_INVALID_ARG, "null out");
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  cudaGetLastError();
  *n = c;
  return RTG_OK;
}

int rtg_ctx_create(int device, int64_t max_h, int64_t max_w, int32_t max_objects,
                   rtg_ctx** out) {
  if (!out) return fail(RTG_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  if (max_h <= 0 || max_w <= 0 || max_h > 8192 || max_w > 8192)
    return fail(RTG_ERR_DIMENSION, "context tile extent must be in [1, 8192]");
  if (max_objects <= 0) return fail(RTG_ERR_INVALID_ARG, "max_objects must be positive");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(RTG_ERR_NO_DEVICE, "no CUDA device: the rtg stage has no CPU fallback");
  }
  if (device < 0 || device >= count) return fail(RTG_ERR_NO_DEVICE, "device index out of range");
  RTG_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  RTG_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(RTG_ERR_DEVICE, std::string("rtg kernels are built for sm_100a (B200); found ") +
                                    prop.name);
  rtg_ctx* c = new rtg_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->max_h = max_h;
  c->max_w = max_w;
  c->max_px = max_h * max_w;
  c->max_objects = max_objects;
  if (const char* g = getenv("RTG_GUARD_BYTES")) {
    const long long v = atoll(g);
    c->guard_bytes = v > 0 ? (size_t)v : 0;
  }
  auto cleanup = [&](int st) {
    rtg_ctx_destroy(c);
    return st;
  };
  int st;
  if ((st = [&]() -> int {
        RTG_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        const size_t n = (size_t)c->max_px;
        RTG_TRY(DALLOC(rgb, 3 * n));
        RTG_TRY(DALLOC(hema, n));
        RTG_TRY(DALLOC(recon, n));
        RTG_TRY(DALLOC(tissue, n));
        RTG_TRY(DALLOC(m1, n));
        RTG_TRY(DALLOC(m2, n));
        RTG_TRY(DALLOC(m3, n));
        RTG_TRY(DALLOC(m4, n));
        RTG_TRY(DALLOC(rm, n));
        RTG_TRY(DALLOC(u16a, n));
        RTG_TRY(DALLOC(u16b, n));
        RTG_TRY(DALLOC(u16c, n));
        RTG_TRY(DALLOC(i32a, n));
        RTG_TRY(DALLOC(i32b, n));
        RTG_TRY(DALLOC(i32c, n));
        RTG_TRY(DALLOC(labels, n));
        RTG_TRY(DALLOC(features, (size_t)max_objects * RTG_MAX_FEATURE_COLUMNS));
        RTG_TRY(DALLOC(feat20, (size_t)max_objects * RTG_NUM_FEATURES));
        RTG_TRY(DALLOC(tex14, (size_t)max_objects * RTG_NUM_TEXTURE));
        RTG_TRY(DALLOC(seg_summary, (size_t)ceil_div(max_h, 32) * (size_t)max_w));
        RTG_TRY(DALLOC(scan_buf, 2 * (size_t)ceil_div(c->max_px, kScanChunk) + 2));
        RTG_TRY(DALLOC(flat_list, n));
        RTG_TRY(DALLOC(lroots, n));
        RTG_TRY(DALLOC(root_bm, n / 32 + 1));
        RTG_TRY(DALLOC(root_wprefix, n / 32 + 1));
        RTG_TRY(DALLOC(fg_list, n));
        RTG_TRY(DALLOC(fg_bits, n / 32 + 8));
        RTG_TRY(DALLOC(sep_bits, n / 32 + 8));
        c->obj_cap = (int64_t)n / 4 + 16;  // 8-connected objects are >= 1 px, <= 1 per 2x2
        RTG_TRY(DALLOC(obj_root, (size_t)c->obj_cap));
        RTG_TRY(DALLOC(obj_box, 4 * (size_t)c->obj_cap));
        RTG_TRY(DALLOC(obj_list, (size_t)c->obj_cap));
        RTG_TRY(DALLOC(arena, 16 * n + 64));
        RTG_TRY(DALLOC(misc, 128 + (size_t)max_h));
        RTG_TRY(DALLOC(status, 1));
        RTG_TRY(DALLOC(stats, RTG_NUM_STATS));
        RTG_TRY(DALLOC(level_bits, 16));
        const int64_t ntiles = ceil_div(max_h, kTile) * ceil_div(max_w, kTile);
        c->tq.capacity = (int32_t)(2 * ntiles);
        RTG_TRY(DALLOC(tq.state, (size_t)ntiles));
        RTG_TRY(DALLOC(tq.slots, (size_t)(2 * ntiles)));
        RTG_TRY(DALLOC(tq.counters, 8));
        c->acc.cap = max_objects;
        RTG_TRY(DALLOC(acc.sums, (size_t)kSumFields * max_objects));
        RTG_TRY(DALLOC(acc.mins, (size_t)kMinFields * max_objects));
        RTG_TRY(DALLOC(acc.maxs, (size_t)kMaxFields * max_objects));
        RTG_TRY(DALLOC(tex_bbox, 4 * (size_t)max_objects));
        RTG_TRY(DALLOC(tex_hist, 17 * (size_t)max_objects));
        RTG_TRY(DALLOC(tex_glcm, 64 * (size_t)max_objects));
        RTG_TRY(DALLOC(tex_mom, 4 * (size_t)max_objects));
        // the checker's own control: one byte into the arena's band
        if (c->guard_bytes && getenv("RTG_GUARD_SELFTEST"))
          for (const auto& g : c->guards)
            if (std::string(g.name) == "arena") RTG_CUDA(cudaMemset(g.end + 5, 0, 1));
        RTG_CUDA(cudaMemsetAsync(c->misc, 0, sizeof(int32_t) * (128 + (size_t)max_h), c->stream));
        RTG_CUDA(cudaMemsetAsync(c->status, 0, sizeof(uint32_t), c->stream));
        RTG_CUDA(cudaMemsetAsync(c->stats, 0, sizeof(int64_t) * RTG_NUM_STATS, c->stream));
        RTG_CUDA(cudaMemsetAsync(c->tq.state, 0, sizeof(int32_t) * (size_t)ntiles, c->stream));
        RTG_CUDA(cudaStreamSynchronize(c->stream));
        return RTG_OK;
      }()) != RTG_OK)
    return cleanup(st);
  *out = c;
  return RTG_OK;
}

int rtg_ctx_destroy(rtg_ctx* c) {
  if (!c) return RTG_OK;
  cudaSetDevice(c->device);
  if (c->own_stream) cudaStreamSynchronize(c->own_stream);
  release_slots(c);
  void* bufs[] = {c->rgb, c->hema, c->recon, c->tissue, c->m1, c->m2, c->m3, c->m4, c->rm,
                  c->u16a, c->u16b, c->u16c, c->i32a, c->i32b, c->i32c, c->labels,
                  c->features, c->feat20, c->tex14, c->seg_summary, c->scan_buf, c->flat_list, c->lroots,
                  c->root_bm, c->root_wprefix, c->fg_list, c->fg_bits, c->sep_bits,
                  c->obj_root, c->obj_box, c->obj_list, c->arena, c->misc,
                  c->status, c->stats, c->level_bits, c->tq.state, c->tq.slots, c->tq.counters,
                  c->acc.sums, c->acc.mins, c->acc.maxs, c->tex_bbox, c->tex_hist,
                  c->tex_glcm, c->tex_mom};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  for (int b = 0; b < 2; ++b) {
    if (c->ev_copied[b]) cudaEventDestroy(c->ev_copied[b]);
    if (c->ev_consumed[b]) cudaEventDestroy(c->ev_consumed[b]);
  }
  if (c->rgb2) cudaFree(c->rgb2);
  if (c->h_counts) cudaFreeHost(c->h_counts);
  if (c->prof_ev) {
    for (int i = 0; i < c->prof_cap; ++i) cudaEventDestroy(c->prof_ev[i]);
    delete[] c->prof_ev;
    delete[] c->prof_stage;
  }
  if (c->graphs) {
    for (int i = 0; i < c->n_graphs; ++i) cudaGraphExecDestroy(c->graphs[i].exec);
    delete[] c->graphs;
  }
  delete c;
  return RTG_OK;
}

int rtg_ctx_stream(rtg_ctx* ctx, void** stream) {
  if (!ctx || !stream) return fail(RTG_ERR_INVALID_ARG, "null argument");
  *stream = (void*)ctx->stream;
  return RTG_OK;
}

int rtg_ctx_set_stream(rtg_ctx* ctx, void* stream) {
  if (!ctx) return fail(RTG_ERR_INVALID_ARG, "null rtg_ctx");
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return RTG_OK;
}

int rtg_ctx_sync(rtg_ctx* ctx) {
  if (!ctx) return fail(RTG_ERR_INVALID_ARG, "null rtg_ctx");
  RTG_CUDA(cudaSetDevice(ctx->device));
  RTG_CUDA(cudaStreamSynchronize(ctx->stream));
  uint32_t st = 0;
  RTG_CUDA(cudaMemcpy(&st, ctx->status, sizeof(st), cudaMemcpyDeviceToHost));
  if (st & kStatusObjectOverflow) {
    RTG_CUDA(cudaMemset(ctx->status, 0, sizeof(uint32_t)));
    return fail(RTG_ERR_OVERFLOW, "object count exceeded the context's max_objects");
  }
  if (st & kStatusQueueOverflow) {
    RTG_CUDA(cudaMemset(ctx->status, 0, sizeof(uint32_t)));
    return fail(RTG_ERR_INTERNAL, "IWPP visit budget exceeded (reconstruction aborted)");
  }
  return RTG_OK;
}

int rtg_ctx_stats(rtg_ctx* ctx, int64_t out[RTG_NUM_STATS]) {
  if (!ctx || !out) return fail(RTG_ERR_INVALID_ARG, "null argument");
  RTG_CUDA(cudaSetDevice(ctx->device));
  RTG_CUDA(cudaStreamSynchronize(ctx->stream));
  int32_t misc[8];
  int64_t st[RTG_NUM_STATS];
  RTG_CUDA(cudaMemcpy(misc, ctx->misc, sizeof(misc), cudaMemcpyDeviceToHost));
  RTG_CUDA(cudaMemcpy(st, ctx->stats, sizeof(st), cudaMemcpyDeviceToHost));
  RTG_CUDA(cudaMemset(ctx->stats, 0, sizeof(st)));
  for (int i = 0; i < RTG_NUM_STATS; ++i) out[i] = st[i];
  out[0] = misc[0];
  out[1] = st[4] + st[6] + st[8] + st[10];
  out[2] = misc[5];  // flat (plateau) pixels of the watershed
  out[3] = misc[3];
  return RTG_OK;
}

int rtg_ctx_profile(rtg_ctx* ctx, int enable) {
  if (!ctx) return fail(RTG_ERR_INVALID_ARG, "null rtg_ctx");
  RTG_CUDA(cudaSetDevice(ctx->device));
  if (enable && !ctx->prof_ev) {
    ctx->prof_cap = 1 << 15;
    ctx->prof_ev = new cudaEvent_t[ctx->prof_cap];
    ctx->prof_stage = new int32_t[ctx->prof_cap];
    for (int i = 0; i < ctx->prof_cap; ++i) RTG_CUDA(cudaEventCreate(&ctx->prof_ev[i]));
  }
  ctx->prof = enable != 0;
  ctx->prof_used = 0;
  for (int i = 0; i < RTG_NUM_STAGES; ++i) {
    ctx->prof_ms[i] = 0.0;
    ctx->prof_calls[i] = 0;
  }
  return RTG_OK;
}

int rtg_ctx_profile_read(rtg_ctx* ctx, double ms[RTG_NUM_STAGES], int64_t calls[RTG_NUM_STAGES]) {
  if (!ctx || !ms || !calls) return fail(RTG_ERR_INVALID_ARG, "null argument");
  RTG_CUDA(cudaSetDevice(ctx->device));
  RTG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k + 1 < ctx->prof_used; ++k) {
    const int st = ctx->prof_stage[k];
    if (st < 0) continue;
    float e = 0.f;
    RTG_CUDA(cudaEventElapsedTime(&e, ctx->prof_ev[k], ctx->prof_ev[k + 1]));
    ctx->prof_ms[st] += e;
    ctx->prof_calls[st] += 1;
  }
  for (int i = 0; i < RTG_NUM_STAGES; ++i) {
    ms[i] = ctx->prof_ms[i];
    calls[i] = ctx->prof_calls[i];
    ctx->prof_ms[i] = 0.0;
    ctx->prof_calls[i] = 0;
  }
  ctx->prof_used = 0;
  return RTG_OK;
}

int rtg_ctx_set_option(rtg_ctx* ctx, int option, int64_t value) {
  if (!ctx) return fail(RTG_ERR_INVALID_ARG, "null rtg_ctx");
  switch (option) {
    case RTG_OPT_FILL_HOLES_IMPL:
      if (value != 0 && value != 1) return fail(RTG_ERR_INVALID_ARG, "fill impl must be 0 or 1");
      ctx->fill_impl = (int)value;
      return RTG_OK;
    case RTG_OPT_USE_GRAPHS:
      ctx->use_graphs = value != 0;
      return RTG_OK;
    case RTG_OPT_WATERSHED_IMPL:
      if (value != 0 && value != 1) return fail(RTG_ERR_INVALID_ARG, "watershed impl must be 0 or 1");
      ctx->ws_impl = (int)value;
      return RTG_OK;
    case RTG_OPT_PDL:
      ctx->use_pdl = value != 0;
      return RTG_OK;
    case RTG_OPT_STREAM_IMPL:
      if (value != 0 && value != 1) return fail(RTG_ERR_INVALID_ARG, "stream impl must be 0 or 1");
      ctx->stream_impl = (int)value;
      return RTG_OK;
    case RTG_OPT_LABEL_RUNS:
      if (value != 0 && value != 1) return fail(RTG_ERR_INVALID_ARG, "label runs must be 0 or 1");
      ctx->label_runs = (int)value;
      return RTG_OK;
    case RTG_OPT_RECON_ENTRY_IMPL:
      if (value != 0 && value != 1) return fail(RTG_ERR_INVALID_ARG, "recon entry impl must be 0 or 1");
      ctx->recon_entry_impl = (int)value;
      return RTG_OK;
    case RTG_OPT_HMAX_IMPL:
      if (value != 0 && value != 1) return fail(RTG_ERR_INVALID_ARG, "hmax impl must be 0 or 1");
      ctx->hmax_impl = (int)value;
      return RTG_OK;
    case RTG_OPT_RECON_IMPL:
      if (value != 0 && value != 1) return fail(RTG_ERR_INVALID_ARG, "recon impl must be 0 or 1");
      ctx->recon_impl = (int)value;
      return RTG_OK;
    default:
      return fail(RTG_ERR_INVALID_ARG, "unknown option " + std::to_string(option));
  }
}

int rtg_ctx_launches(rtg_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return fail(RTG_ERR_INVALID_ARG, "null argument");
  *out = ctx->launches;
  return RTG_OK;
}

int rtg_ctx_guard_check(rtg_ctx* ctx, int32_t* n_checked) {
  if (!ctx) return fail(RTG_ERR_INVALID_ARG, "null context");
  RTG_CUDA(cudaSetDevice(ctx->device));
  RTG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<unsigned char> host(ctx->guard_bytes);
  int32_t n = 0;
  for (const auto& g : ctx->guards) {
    RTG_CUDA(cudaMemcpy(host.data(), g.end, ctx->guard_bytes, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < ctx->guard_bytes; ++i)
      if (host[i] != kGuardByte)
        return fail(RTG_ERR_INTERNAL, std::string("guard band after scratch buffer '") + g.name +
                                          "' overwritten at +" + std::to_string(i));
    ++n;
  }
  if (n_checked) *n_checked = n;
  return RTG_OK;
}

int rtg_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(RTG_ERR_INVALID_ARG, "null out");
  RTG_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
  return RTG_OK;
}

int rtg_host_free(void* p) {
  if (p) RTG_CUDA(cudaFreeHost(p));
  return RTG_OK;
}

// ---- whole tile, host buffers ------------------------------------------------

int rtg_process_tiles(rtg_ctx* ctx, int32_t count, const uint8_t* const* rgb, int64_t h,
                      int64_t w, int64_t pitch_bytes, const rtg_params* params,
                      float* const* features_out, int32_t max_rows, int32_t* n_objects) {
  RTG_TRY(check_ctx(ctx, h, w));
  RTG_TRY(check_params(params));
  if (count < 0 || (count > 0 && (!rgb || !n_objects)))
    return fail(RTG_ERR_INVALID_ARG, "bad tile batch");
  if (max_rows < 0) return fail(RTG_ERR_INVALID_ARG, "max_rows < 0");
  if (pitch_bytes < 3 * w) return fail(RTG_ERR_DIMENSION, "pitch_bytes < 3 * w");
  for (int32_t i = 0; i < count; ++i)
    if (!rgb[i]) return fail(RTG_ERR_INVALID_ARG, "null rgb in batch");
  if (count == 0) return RTG_OK;
  // lazily created double-buffering resources
  if (!ctx->rgb2) {
    void* p = nullptr;
    RTG_CUDA(cudaMalloc(&p, (size_t)(3 * ctx->max_px)));
    ctx->rgb2 = static_cast<uint8_t*>(p);
    RTG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      RTG_CUDA(cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming));
      RTG_CUDA(cudaEventCreateWithFlags(&ctx->ev_consumed[b], cudaEventDisableTiming));
    }
  }
  if (ctx->h_counts_cap < count) {
    if (ctx->h_counts) RTG_CUDA(cudaFreeHost(ctx->h_counts));
    ctx->h_counts = nullptr;
    void* p = nullptr;
    RTG_CUDA(cudaMallocHost(&p, sizeof(int32_t) * (size_t)count));
    ctx->h_counts = static_cast<int32_t*>(p);
    ctx->h_counts_cap = count;
  }
  uint8_t* buf[2] = {ctx->rgb, ctx->rgb2};
  const int32_t rows = max_rows < ctx->max_objects ? max_rows : ctx->max_objects;
  // both buffers start free
  for (int b = 0; b < 2; ++b) RTG_CUDA(cudaEventRecord(ctx->ev_consumed[b], ctx->stream));
  for (int32_t i = 0; i < count; ++i) {
    const int b = i & 1;
    // upload tile i into buffer b once tile i-2 has released it
    RTG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_consumed[b], 0));
    if (pitch_bytes == 3 * w)
      RTG_CUDA(cudaMemcpyAsync(buf[b], rgb[i], (size_t)(3 * h * w), cudaMemcpyHostToDevice,
                               ctx->copy_stream));
    else
      RTG_CUDA(cudaMemcpy2DAsync(buf[b], (size_t)(3 * w), rgb[i], (size_t)pitch_bytes,
                                 (size_t)(3 * w), (size_t)h, cudaMemcpyHostToDevice,
                                 ctx->copy_stream));
    RTG_CUDA(cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
    RTG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[b], 0));
    if (ctx->use_graphs && !ctx->prof)
      RTG_TRY(pipeline_graph(ctx, buf[b], h, w, 3 * w, params, ctx->m4, ctx->labels, ctx->hema,
                             ctx->features, ctx->misc));
    else
      RTG_TRY(pipeline(ctx, buf[b], h, w, 3 * w, params, ctx->m4, ctx->labels, ctx->hema,
                       ctx->features, ctx->misc, true));
    RTG_CUDA(cudaEventRecord(ctx->ev_consumed[b], ctx->stream));
    RTG_CUDA(cudaMemcpyAsync(ctx->h_counts + i, ctx->misc, sizeof(int32_t),
                             cudaMemcpyDeviceToHost, ctx->stream));
    if (features_out && features_out[i] && rows > 0)
      RTG_TRY(rows_to_host(ctx, ctx->stream, ctx->features, ctx->misc, features_out[i], rows,
                           feature_cols(params)));
  }
  RTG_TRY(rtg_ctx_sync(ctx));
  int over = -1;
  for (int32_t i = 0; i < count; ++i) {
    n_objects[i] = ctx->h_counts[i];
    if (features_out && features_out[i] && (n_objects[i] > max_rows ||
                                            n_objects[i] > ctx->max_objects) && over < 0)
      over = i;
  }
  if (over >= 0)
    return fail(RTG_ERR_OVERFLOW, "tile " + std::to_string(over) + " has " +
                                      std::to_string(n_objects[over]) + " objects; feature rows: " +
                                      std::to_string(rows));
  return RTG_OK;
}

int rtg_process_tile(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w,
                     int64_t pitch_bytes, const rtg_params* params, uint8_t* mask_out,
                     int32_t* labels_out, uint8_t* hema_out, float* features_out,
                     int32_t max_rows, int32_t* n_objects) {
  RTG_TRY(check_ctx(ctx, h, w));
  RTG_TRY(check_params(params));
  if (!n_objects) return fail(RTG_ERR_INVALID_ARG, "null n_objects");
  if (features_out && max_rows < 0) return fail(RTG_ERR_INVALID_ARG, "max_rows < 0");
  RTG_TRY(upload_rgb(ctx, rgb, h, w, pitch_bytes));
  if (ctx->use_graphs && !ctx->prof)
    RTG_TRY(pipeline_graph(ctx, ctx->rgb, h, w, 3 * w, params, ctx->m4, ctx->labels, ctx->hema,
                           ctx->features, ctx->misc));
  else
    RTG_TRY(pipeline(ctx, ctx->rgb, h, w, 3 * w, params, ctx->m4, ctx->labels, ctx->hema,
                     ctx->features, ctx->misc, true));
  int32_t n = 0;
  RTG_CUDA(cudaMemcpyAsync(&n, ctx->misc, sizeof(n), cudaMemcpyDeviceToHost, ctx->stream));
  RTG_CUDA(cudaStreamSynchronize(ctx->stream));
  *n_objects = n;
  const size_t px = (size_t)(h * w);
  if (mask_out)
    RTG_CUDA(cudaMemcpyAsync(mask_out, ctx->m4, px, cudaMemcpyDeviceToHost, ctx->stream));
  if (labels_out)
    RTG_CUDA(cudaMemcpyAsync(labels_out, ctx->labels, px * 4, cudaMemcpyDeviceToHost,
                             ctx->stream));
  if (hema_out)
    RTG_CUDA(cudaMemcpyAsync(hema_out, ctx->hema, px, cudaMemcpyDeviceToHost, ctx->stream));
  const int32_t rows = n < max_rows ? n : max_rows;
  const int32_t dev_rows = rows < ctx->max_objects ? rows : ctx->max_objects;
  if (features_out && dev_rows > 0)
    RTG_CUDA(cudaMemcpyAsync(features_out, ctx->features,
                             sizeof(float) * (size_t)feature_cols(params) * (size_t)dev_rows,
                             cudaMemcpyDeviceToHost, ctx->stream));
  RTG_TRY(rtg_ctx_sync(ctx));
  if (features_out && (n > max_rows || n > ctx->max_objects))
    return fail(RTG_ERR_OVERFLOW, "tile has " + std::to_string(n) + " objects; feature rows: " +
                                      std::to_string(dev_rows));
  return RTG_OK;
}

int rtg_segment_tile(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w,
                     int64_t pitch_bytes, const rtg_params* params, uint8_t* mask_out,
                     int32_t* labels_out, int32_t* n_objects) {
  RTG_TRY(check_ctx(ctx, h, w));
  RTG_TRY(check_params(params));
  if (!n_objects) return fail(RTG_ERR_INVALID_ARG, "null n_objects");
  RTG_TRY(upload_rgb(ctx, rgb, h, w, pitch_bytes));
  RTG_TRY(pipeline(ctx, ctx->rgb, h, w, 3 * w, params, ctx->m4, ctx->labels, ctx->hema,
                   nullptr, ctx->misc, false));
  const size_t px = (size_t)(h * w);
  if (mask_out)
    RTG_CUDA(cudaMemcpyAsync(mask_out, ctx->m4, px, cudaMemcpyDeviceToHost, ctx->stream));
  if (labels_out)
    RTG_CUDA(cudaMemcpyAsync(labels_out, ctx->labels, px * 4, cudaMemcpyDeviceToHost,
                             ctx->stream));
  int32_t n = 0;
  RTG_CUDA(cudaMemcpyAsync(&n, ctx->misc, sizeof(n), cudaMemcpyDeviceToHost, ctx->stream));
  RTG_TRY(rtg_ctx_sync(ctx));
  *n_objects = n;
  return RTG_OK;
}

int rtg_features(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity, int64_t h,
                 int64_t w, int32_t n_objects, float* out) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!labels || !intensity || (!out && n_objects > 0))
    return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (n_objects < 0 || n_objects > ctx->max_objects)
    return fail(RTG_ERR_OVERFLOW, "n_objects outside [0, max_objects]");
  const size_t px = (size_t)(h * w);
  RTG_CUDA(cudaMemcpyAsync(ctx->labels, labels, px * 4, cudaMemcpyHostToDevice, ctx->stream));
  RTG_CUDA(cudaMemcpyAsync(ctx->hema, intensity, px, cudaMemcpyHostToDevice, ctx->stream));
  RTG_CUDA(cudaMemcpyAsync(ctx->misc, &n_objects, sizeof(int32_t), cudaMemcpyHostToDevice,
                           ctx->stream));
  RTG_TRY(features(ctx, ctx->labels, ctx->hema, h, w, ctx->misc, ctx->features));
  if (n_objects > 0)
    RTG_CUDA(cudaMemcpyAsync(out, ctx->features,
                             sizeof(float) * RTG_NUM_FEATURES * (size_t)n_objects,
                             cudaMemcpyDeviceToHost, ctx->stream));
  return rtg_ctx_sync(ctx);
}

// ---- whole tile, device buffers ------------------------------------------------

int rtg_process_tile_dev(rtg_ctx* ctx, const uint8_t* d_rgb, int64_t h, int64_t w,
                         int64_t pitch_bytes, const rtg_params* params, uint8_t* d_mask,
                         int32_t* d_labels, uint8_t* d_hema, float* d_features,
                         int32_t* d_n_objects) {
  RTG_TRY(check_ctx(ctx, h, w));
  RTG_TRY(check_params(params));
  if (!d_rgb || !d_features || !d_n_objects) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (pitch_bytes < 3 * w) return fail(RTG_ERR_DIMENSION, "pitch_bytes < 3 * w");
  if (!ctx->use_graphs || ctx->prof)
    return pipeline(ctx, d_rgb, h, w, pitch_bytes, params, d_mask, d_labels, d_hema, d_features,
                    d_n_objects, true);
  return pipeline_graph(ctx, d_rgb, h, w, pitch_bytes, params, d_mask, d_labels, d_hema,
                        d_features, d_n_objects);
}

// ---- per-operator entry points ---------------------------------------------------

int rtg_colordeconv_dev(rtg_ctx* ctx, const uint8_t* d_rgb, int64_t h, int64_t w,
                        int64_t pitch_bytes, const rtg_params* params, uint8_t* d_hema,
                        uint8_t* d_marker, uint8_t* d_tissue) {
  RTG_TRY(check_ctx(ctx, h, w));
  RTG_TRY(check_params(params));
  if (!d_rgb) return fail(RTG_ERR_INVALID_ARG, "null rgb");
  if (pitch_bytes < 3 * w) return fail(RTG_ERR_DIMENSION, "pitch_bytes < 3 * w");
  return launch_colordeconv(ctx, d_rgb, h, w, pitch_bytes, params, d_hema, d_marker, d_tissue);
}

int rtg_recon_u8_dev(rtg_ctx* ctx, const uint8_t* d_marker, const uint8_t* d_mask, int64_t h,
                     int64_t w, int conn, uint8_t* d_out) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_marker || !d_mask || !d_out) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (conn != 4 && conn != 8) return fail(RTG_ERR_INVALID_ARG, "conn must be 4 or 8");
  // Few distinct values (a maze, a binary or quantised mask): one seeded
  // labelling per value, immune to long propagation paths that make the
  // wavefront engine crawl tile by tile.  The clip pass also collects the
  // values present; reading them back synchronises, so the choice is skipped
  // while the stream is being captured into a graph.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  RTG_CUDA(cudaStreamIsCapturing(ctx->stream, &cap));
  if (cap == cudaStreamCaptureStatusNone && ctx->recon_entry_impl != 1) {
    uint8_t levels[kMaxReconLevels];
    int count = -1;
    RTG_TRY(recon_clip_levels(ctx, d_marker, d_mask, h, w, d_out, levels, &count));
    if (count >= 0) return recon_levels(ctx, d_out, d_mask, h, w, conn, levels, count);
  } else {
    k_clip_copy<uint8_t><<<grid_for(ctx, h * w), 256, 0, ctx->stream>>>(d_marker, d_mask, h * w,
                                                                        d_out);
    RTG_LAUNCH("k_clip_copy");
  }
  return iwpp_recon_u8(ctx, d_out, d_mask, h, w, conn);
}

int rtg_recon_u16_dev(rtg_ctx* ctx, const uint16_t* d_marker, const uint16_t* d_mask,
                      int64_t h, int64_t w, int conn, uint16_t* d_out) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_marker || !d_mask || !d_out) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (conn != 4 && conn != 8) return fail(RTG_ERR_INVALID_ARG, "conn must be 4 or 8");
  k_clip_copy<uint16_t><<<grid_for(ctx, h * w), 256, 0, ctx->stream>>>(d_marker, d_mask,
                                                                       h * w, d_out);
  RTG_LAUNCH("k_clip_copy");
  return iwpp_recon_u16(ctx, d_out, d_mask, h, w, conn);
}

int rtg_fill_holes_dev(rtg_ctx* ctx, const uint8_t* d_in, int64_t h, int64_t w,
                       uint8_t* d_out) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_in || !d_out) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (d_in == d_out) return fail(RTG_ERR_INVALID_ARG, "fill holes cannot run in place");
  return run_fill_holes(ctx, d_in, h, w, d_out);
}

int rtg_bwlabel_dev(rtg_ctx* ctx, const uint8_t* d_mask, int64_t h, int64_t w, int conn,
                    int32_t* d_labels, int32_t* d_n) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_mask || !d_labels) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (conn != 4 && conn != 8) return fail(RTG_ERR_INVALID_ARG, "conn must be 4 or 8");
  RTG_TRY(ccl_roots(ctx, d_mask, h, w, conn, ctx->i32a));
  return ccl_canonical(ctx, ctx->i32a, h, w, d_labels, d_n ? d_n : ctx->misc);
}

int rtg_area_threshold_dev(rtg_ctx* ctx, const uint8_t* d_mask, int64_t h, int64_t w,
                           int conn, int32_t min_area, int32_t max_area, uint8_t* d_out) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_mask || !d_out) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (conn != 4 && conn != 8) return fail(RTG_ERR_INVALID_ARG, "conn must be 4 or 8");
  RTG_TRY(ccl_roots(ctx, d_mask, h, w, conn, ctx->i32a, ctx->i32b));
  return area_filter(ctx, ctx->i32a, h * w, min_area, max_area, ctx->i32b, d_out);
}

int rtg_edt_dev(rtg_ctx* ctx, const uint8_t* d_mask, int64_t h, int64_t w, int32_t* d_dist2) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_mask || !d_dist2) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  return edt(ctx, d_mask, h, w, d_dist2, nullptr, nullptr, 0);
}

int rtg_watershed_dev(rtg_ctx* ctx, const uint8_t* d_mask, int64_t h, int64_t w, int32_t ws_h,
                      uint8_t* d_sep_mask, int32_t* d_basin) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_mask || !d_sep_mask) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (ws_h < 0) return fail(RTG_ERR_INVALID_ARG, "ws_h must be >= 0");
  if (ctx->ws_impl == 0)
    return watershed(ctx, d_mask, h, w, ws_h, d_sep_mask, d_basin ? d_basin : ctx->labels);
  RTG_TRY(ccl_roots(ctx, d_mask, h, w, 8, ctx->i32a));
  return watershed_objects(ctx, d_mask, ctx->i32a, nullptr, 0, 0, h, w, ws_h, d_sep_mask, d_basin);
}

int rtg_features_dev(rtg_ctx* ctx, const int32_t* d_labels, const uint8_t* d_intensity,
                     int64_t h, int64_t w, const int32_t* d_n, float* d_features) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_labels || !d_intensity || !d_n || !d_features)
    return fail(RTG_ERR_INVALID_ARG, "null buffer");
  return features(ctx, d_labels, d_intensity, h, w, d_n, d_features);
}

int rtg_texture_features_dev(rtg_ctx* ctx, const int32_t* d_labels, const uint8_t* d_intensity,
                             int64_t h, int64_t w, const int32_t* d_n, float* d_texture) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_labels || !d_intensity || !d_n || !d_texture)
    return fail(RTG_ERR_INVALID_ARG, "null buffer");
  return texture(ctx, d_labels, d_intensity, h, w, d_n, d_texture);
}

int rtg_canny_dev(rtg_ctx* ctx, const uint8_t* d_intensity, int64_t h, int64_t w, int32_t low,
                  int32_t high, uint8_t* d_edges) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_intensity || !d_edges) return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (low < 0 || high < low || high > 46341)
    return fail(RTG_ERR_INVALID_ARG, "Canny thresholds need 0 <= low <= high <= 46341");
  return canny(ctx, d_intensity, h, w, low, high, d_edges);
}

int rtg_texture_features(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity, int64_t h,
                         int64_t w, int32_t n_objects, float* out) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!labels || !intensity || (!out && n_objects > 0))
    return fail(RTG_ERR_INVALID_ARG, "null buffer");
  if (n_objects < 0 || n_objects > ctx->max_objects)
    return fail(RTG_ERR_OVERFLOW, "n_objects outside [0, max_objects]");
  const size_t px = (size_t)(h * w);
  RTG_CUDA(cudaMemcpyAsync(ctx->labels, labels, px * 4, cudaMemcpyHostToDevice, ctx->stream));
  RTG_CUDA(cudaMemcpyAsync(ctx->hema, intensity, px, cudaMemcpyHostToDevice, ctx->stream));
  RTG_CUDA(cudaMemcpyAsync(ctx->misc, &n_objects, sizeof(int32_t), cudaMemcpyHostToDevice,
                           ctx->stream));
  // rows land in the feature buffer (max_objects x 20 >= n x 12 floats)
  RTG_TRY(texture(ctx, ctx->labels, ctx->hema, h, w, ctx->misc, ctx->features));
  if (n_objects > 0)
    RTG_CUDA(cudaMemcpyAsync(out, ctx->features,
                             sizeof(float) * RTG_NUM_TEXTURE * (size_t)n_objects,
                             cudaMemcpyDeviceToHost, ctx->stream));
  return rtg_ctx_sync(ctx);
}

int rtg_synth_tile_dev(rtg_ctx* ctx, uint64_t global_seed, int64_t tile_row, int64_t tile_col,
                       int64_t h, int64_t w, uint8_t* d_rgb) {
  RTG_TRY(check_ctx(ctx, h, w));
  if (!d_rgb) return fail(RTG_ERR_INVALID_ARG, "null rgb");
  return synth_dev(ctx, global_seed, tile_row, tile_col, h, w, d_rgb);
}

}  // extern "C"
