// Shared device/host helpers for the rtg CUDA library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "rtg.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "rtg kernels are written for sm_100a (B200); compile with -gencode arch=compute_100a,code=sm_100a"
#endif

namespace rtg {

// ---- error plumbing (no exceptions cross extern "C") -----------------------

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define RTG_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return ::rtg::cuda_fail(e_, #call); \
  } while (0)

// every kernel launch site goes through this (counts launches per ctx)
#define RTG_LAUNCH(what)                                          \
  do {                                                            \
    ++ctx->launches;                                              \
    cudaError_t e_ = cudaGetLastError();                          \
    if (e_ != cudaSuccess) return ::rtg::cuda_fail(e_, what);     \
  } while (0)

// Opts `kernel` into `bytes` of dynamic shared memory on `device` once.  The
// attribute is per device, so it is remembered per (kernel, device) pair
// under a lock (contexts on different devices and threads share kernels).
cudaError_t smem_optin(const void* kernel, int device, int bytes);
#define RTG_SMEM_OPTIN(kernel, bytes) \
  RTG_CUDA(::rtg::smem_optin(reinterpret_cast<const void*>(kernel), ctx->device, (int)(bytes)))

#define RTG_TRY(call)               \
  do {                              \
    int s_ = (call);                \
    if (s_ != RTG_OK) return s_;    \
  } while (0)

// ---- sticky device status bits ---------------------------------------------
enum : uint32_t {
  kStatusObjectOverflow = 1u << 0,
  kStatusQueueOverflow = 1u << 1,
  kStatusEdtFallback = 1u << 2,  // informational: exact row fallback used
};

// ---- tile-queue state of the IWPP engine ------------------------------------
struct TileQueue {
  int32_t* state;     // per tile: 0 idle, 1 queued, 2 processing, 3 dirty
  int32_t* slots;     // circular queue of tile+1 (0 = empty), 2*ntiles
  uint32_t* counters; // [0] head, [1] tail, [2] pending, [3] visits, [4] abort
  int32_t capacity;   // ntiles of the largest tile
};

// Per-object accumulators of the feature step (SoA, PAPER.md:1162-1177
// "intermediate results ... fixed sized per nucleus").
struct FeatureAcc {
  unsigned long long* sums;  // kSumFields x cap
  int32_t* mins;             // kMinFields x cap
  int32_t* maxs;             // kMaxFields x cap
  int32_t cap;
};
enum { kSumArea = 0, kSumY, kSumX, kSumYY, kSumXX, kSumXY, kSumI, kSumII,
       kSumG, kSumGG, kSumPerim, kSumFields };
enum { kMinI = 0, kMinY, kMinX, kMinFields };
enum { kMaxI = 0, kMaxY, kMaxX, kMaxFields };

struct HemaLut {
  int32_t v[3][256];
};

}  // namespace rtg

namespace rtg {
// One in-flight tile of the asynchronous host-buffer entry point
// (rtg_process_tile_async): its own device RGB / output planes so the upload
// of tile t+1, the stage of tile t and the download of tile t-1 overlap (the
// paper's 3-phase pipeline, reference wrm.cpp:385-415 prefetch_pipeline).
struct AsyncSlot {
  uint8_t* rgb = nullptr;     // 3 * max_px
  uint8_t* mask = nullptr;    // max_px
  int32_t* labels = nullptr;  // max_px
  uint8_t* hema = nullptr;    // max_px
  float* feats = nullptr;     // max_objects x RTG_NUM_FEATURES
  int32_t* d_n = nullptr;     // object count (device)
  int32_t* h_n = nullptr;     // object count (pinned host)
  cudaEvent_t up = nullptr, comp = nullptr, down = nullptr;
  uint64_t ticket = 0;        // 0 = free
  int32_t max_rows = 0;       // feature rows the caller asked for (-1: no table)
};
constexpr int kAsyncSlots = 3;
}  // namespace rtg

// The context: every device allocation of the stage lives here (arena).
struct rtg_ctx {
  // debug guard bands (RTG_GUARD_BYTES at creation): every scratch buffer is
  // followed by this many canary bytes that rtg_ctx_guard_check verifies
  struct Guard {
    unsigned char* end;
    const char* name;
  };
  std::vector<Guard> guards;
  size_t guard_bytes = 0;
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int64_t max_h = 0, max_w = 0, max_px = 0;
  int32_t max_objects = 0;

  // planes (max_px elements)
  uint8_t* rgb = nullptr;     // 3 * max_px, for host-buffer entry points
  uint8_t* rgb2 = nullptr;    //   second buffer (rtg_process_tiles double buffering)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_consumed[2] = {nullptr, nullptr};
  int32_t* h_counts = nullptr;  // pinned per-tile object counts (batch entry)
  int32_t h_counts_cap = 0;
  // rtg_process_tile_async: slots (created on first use), upload / download
  // streams, and the results of tickets retired before the caller waited
  rtg::AsyncSlot* slots = nullptr;
  cudaStream_t up_stream = nullptr, down_stream = nullptr;
  uint64_t next_ticket = 1;
  struct Retired {
    uint64_t ticket;
    int32_t n, max_rows;
  };
  std::vector<Retired> retired;
  uint8_t* hema = nullptr;
  uint8_t* recon = nullptr;   // marker in, reconstruction out
  uint8_t* tissue = nullptr;
  uint8_t* m1 = nullptr;
  uint8_t* m2 = nullptr;
  uint8_t* m3 = nullptr;
  uint8_t* m4 = nullptr;
  uint8_t* rm = nullptr;
  uint16_t* u16a = nullptr;
  uint16_t* u16b = nullptr;
  uint16_t* u16c = nullptr;
  int32_t* i32a = nullptr;
  int32_t* i32b = nullptr;
  int32_t* i32c = nullptr;
  int32_t* labels = nullptr;
  float* features = nullptr;  // max_objects x RTG_MAX_FEATURE_COLUMNS (host-entry staging)
  float* feat20 = nullptr;    // max_objects x RTG_NUM_FEATURES (texture runs: the shape part)
  float* tex14 = nullptr;     // max_objects x RTG_NUM_TEXTURE (texture runs: the texture part)

  // small scratch
  int32_t* seg_summary = nullptr;  // EDT column-segment summaries
  int32_t* scan_buf = nullptr;     // CCL compaction per-chunk counts/offsets
  int32_t* flat_list = nullptr;    // watershed plateau pixel list
  int32_t* lroots = nullptr;       // CCL tile-local roots: (root, count | seed bit) pairs
  uint32_t* root_bm = nullptr;     // CCL global-root bitmap (max_px / 32 words)
  int32_t* fg_list = nullptr;      // watershed foreground pixel list (max_px)
  uint32_t* fg_bits = nullptr;     //   and 1-bit plane (+ pad words)
  uint32_t* sep_bits = nullptr;    // the separated mask as a 1-bit plane (run-table path)
  int32_t* root_wprefix = nullptr; //   and its per-word exclusive prefix
  int32_t* obj_root = nullptr;     // object-parallel watershed: object roots
  int32_t* obj_box = nullptr;      //   and bounding boxes (4 per object)
  int32_t* obj_list = nullptr;     //   big / pathological size-class lists
  int64_t obj_cap = 0;
  unsigned char* arena = nullptr;  //   global scratch for pathological regions
  int32_t* misc = nullptr;         // [0] n_objects, [1] flat count, [2] any_zero, [3] changed, ...
  uint32_t* status = nullptr;      // sticky status bits
  int64_t* stats = nullptr;        // device-side counters for rtg_ctx_stats
  uint32_t* level_bits = nullptr;  // value-presence bitmaps (rtg_recon_u8_dev)
  rtg::TileQueue tq{};
  rtg::FeatureAcc acc{};
  // texture intermediates (max_objects each): bbox, histogram, GLCM, moments
  int32_t* tex_bbox = nullptr;
  uint32_t* tex_hist = nullptr;
  uint32_t* tex_glcm = nullptr;
  unsigned long long* tex_mom = nullptr;

  // implementation options (rtg_ctx_set_option)
  int fill_impl = 0;  // 0: union-find on the background, 1: IWPP tile queue
  int use_graphs = 1; // replay rtg_process_tile_dev as a cached CUDA graph
  int recon_impl = 0; // 0: threshold decomposition (union-find), 1: IWPP grayscale
  int ws_impl = 0;    // 0: tiled whole-tile watershed, 1: object-parallel
  int hmax_impl = 0;  // 0: sparse components, 1: IWPP
  int recon_entry_impl = 0;  // rtg_recon_u8_dev: 0 auto (levels / IWPP), 1 IWPP
  int stream_impl = 1;  // colour deconvolution: 1 TMA bulk-copy ring (default), 0 LDG.128 stream
  int label_runs = 1;   // stage labellings in run-table form (k_ccl.cu CclRuns) when the shape allows
  bool ccl_runs_live = false;  // the last ccl_roots left run tables for ccl_canonical
  bool cand_bits = false;      // recon left the candidates as row masks (fill_area_joint reads them)
  bool mask_bytes_live = false;  // fill_area_joint wrote its mask bytes (the EDT reuses them)
  bool sep_bits_live = false;  // fill_area_joint cleared sep_bits: the watershed writes the
                               // separated mask there, the labelling reads it and writes the bytes
  int use_pdl = 0;    // programmatic dependent launch between the stage's kernels

  // CUDA-graph cache of whole-tile pipelines, keyed by every argument
  struct GraphEntry {
    std::string key;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;  // kernel launches one replay stands for
    uint64_t last_use = 0;
  };
  GraphEntry* graphs = nullptr;
  int n_graphs = 0;
  uint64_t graph_clock = 0;

  // host-side instrumentation
  int64_t launches = 0;           // kernels launched through this ctx
  bool prof = false;              // stage timing with CUDA events
  cudaEvent_t* prof_ev = nullptr; // ring of boundary events
  int32_t* prof_stage = nullptr;  // stage id that starts at each event (-1 = end)
  int prof_cap = 0, prof_used = 0;
  double prof_ms[RTG_NUM_STAGES] = {};
  int64_t prof_calls[RTG_NUM_STAGES] = {};
};

namespace rtg {

constexpr int kTile = 32;  // IWPP tile edge (one warp per tile)
constexpr int kScanChunk = 4096;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int check_ctx(rtg_ctx* ctx, int64_t h, int64_t w);
int check_params(const rtg_params* p);
// Frees the rtg_process_tile_async slots and streams (rtg_ctx_destroy).
void release_slots(rtg_ctx* c);
// The whole stage o1..o9 on device buffers, enqueued on ctx->stream (a
// cached CUDA graph per argument tuple unless graphs are off / profiling).
int run_stage(rtg_ctx* ctx, const uint8_t* d_rgb, int64_t h, int64_t w, int64_t pitch,
              const rtg_params* p, uint8_t* d_mask, int32_t* d_labels, uint8_t* d_hema,
              float* d_features, int32_t* d_n);
// First min(*d_n, cap) feature rows (`cols` floats each) of `src` into host
// `dst` on `stream`:
// zero-copy stores of exactly the live rows for pinned destinations, a
// cudaMemcpyAsync of cap rows otherwise.
int rows_to_host(rtg_ctx* ctx, cudaStream_t stream, const float* src, const int32_t* d_n,
                 float* dst, int32_t cap, int cols);
// Feature-row width of the stage under p (RTG_NUM_FEATURES [+ RTG_NUM_TEXTURE]).
inline int feature_cols(const rtg_params* p) {
  return RTG_NUM_FEATURES + (p->texture ? RTG_NUM_TEXTURE : 0);
}
// Stage boundary for rtg_ctx_profile (no-op unless profiling is enabled):
// stage >= 0 starts that stage, -1 closes the current one.
void prof_mark(rtg_ctx* ctx, int stage);
void hema_lut(const rtg_params* p, HemaLut* lut);

// Zeroes up to four device regions with one kernel of the launch chain.
struct ZeroList {
  void* ptr[8];
  uint64_t bytes[8];
  int count;
};
int zero_async(rtg_ctx* ctx, const ZeroList& z);

// ---- launchers (one translation unit each) ---------------------------------
// Up to six small int32 regions (counters, pad words) for a kernel's first
// CTA to clear on the way.
struct ClearList {
  int32_t* p[6];
  int32_t n[6];
  int count;
};
// clear (optional): counters the next stages need zeroed, cleared by the
// streaming kernel itself (zeroing launches fewer in the pipeline).
// recon_bits (optional): {fg, seed, tissue} 1-bit planes for ReconToNuclei
// (H >= nuc_thresh, H >= nuc_thresh + recon_h, tissue), written by the vector
// kernels; *bits_written says whether they were (contiguous, 16-aligned,
// unpitched input).  tissue may then be nullptr (no tissue bytes).
int launch_colordeconv(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w,
                       int64_t pitch, const rtg_params* p, uint8_t* hema,
                       uint8_t* marker, uint8_t* tissue, const ClearList* clear = nullptr,
                       uint32_t* const* recon_bits = nullptr, bool* bits_written = nullptr);
int launch_candidate(rtg_ctx* ctx, const uint8_t* recon, const uint8_t* tissue,
                     int64_t n, int32_t thresh, uint8_t* out);

// IWPP reconstruction by dilation on the tile queue.  J is updated in place.
// mode 0: J and I are plain planes, all tiles initially queued.
// mode 1: fill-holes: I = complement of `bin`, J seeded on the border, only
//         border tiles initially queued; on exit J = reached background.
int iwpp_recon_u8(rtg_ctx* ctx, uint8_t* J, const uint8_t* I, int64_t h,
                  int64_t w, int conn);
// kind selects the rtg_ctx_stats slot: 1 = HMAX, 2 = regional maxima
int iwpp_recon_u16(rtg_ctx* ctx, uint16_t* J, const uint16_t* I, int64_t h,
                   int64_t w, int conn, int kind = 1);
int iwpp_fill_holes(rtg_ctx* ctx, const uint8_t* bin, uint8_t* J, int64_t h,
                    int64_t w, uint8_t* out);

// Union-find CCL into a two-level forest: roots[p] is p's tile-local root
// (or, for a local root, the global root); root_of(roots, p) is the minimum
// linear index of p's component (-1 = background).  counts, when given,
// receives every component's pixel count at its global root.
// prezeroed: the caller already cleared the counters ccl_label_zero names.
// Whether an h x w labelling can take the run-table form (w % 32 == 0 and
// the tables fit the context's planes).
bool run_tables_fit(rtg_ctx* ctx, int64_t h, int64_t w);
// runs: the run-table form (k_ccl.cu CclRuns; the roots plane then only
// holds the local roots' entries) when the shape allows it; only for a
// ccl_canonical that follows directly.
int ccl_roots(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w,
              int conn, int32_t* roots, int32_t* counts = nullptr, bool prezeroed = false,
              bool runs = false);
// Appends to z the buffers a labelling CCL (ccl_roots + ccl_canonical) of an
// h x w mask needs cleared: local-root count, root bitmap, look-back status.
void ccl_label_zero(rtg_ctx* ctx, int64_t h, int64_t w, ZeroList& z);
__device__ __forceinline__ int32_t root_of(const int32_t* __restrict__ roots, int64_t i) {
  const int32_t v = roots[i];
  return v < 0 ? -1 : roots[v];
}

// ---- programmatic dependent launch (PDL) ------------------------------------
// The stage is a chain of ~40 short kernels; launched with programmatic
// stream serialisation, kernel N+1 is scheduled while kernel N drains
// instead of after it.  Every kernel launched that way begins with
// pdl_enter(): griddepcontrol.wait blocks until the predecessor grid has
// completed and its memory is visible, then launch_dependents lets the next
// kernel be scheduled once all of this grid's CTAs are running.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(rtg_ctx* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                            size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->use_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Division of pixel indices by the tile width without the ~20-instruction
// integer divide: q = (umulhi(n, m) + n) >> s with a 33-bit magic (exact for
// every n < 2^31, d >= 1), built on the host.
struct FastDiv {
  uint32_t m, s, d;
};
inline FastDiv make_div(uint32_t d) {
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  const uint64_t m = ((1ull << 32) * ((1ull << s) - d)) / d + 1;
  return FastDiv{(uint32_t)m, s, d};
}
__device__ __forceinline__ int32_t fdiv(int32_t n, const FastDiv& f) {
  const uint32_t t = __umulhi((uint32_t)n, f.m);
  return (int32_t)((t + (uint32_t)n) >> f.s);
}

// Block-wide reservation of `cnt` consecutive slots per thread from a global
// counter with ONE atomic per block (same-address global atomics serialise
// at about one per clock, so per-warp appends of a whole-tile pass cost tens
// of microseconds).  Every thread of the block must call it; sm holds
// (blockDim.x / 32 + 1) ints.  Returns the thread's first slot.
__device__ __forceinline__ int32_t block_reserve(int32_t cnt, int32_t* counter, int32_t* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sm[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t tot = 0;
    for (int k = 0; k < nw; ++k) {
      const int32_t t = sm[k];
      sm[k] = tot;
      tot += t;
    }
    sm[nw] = tot ? atomicAdd(counter, tot) : 0;
  }
  __syncthreads();
  const int32_t r = sm[nw] + sm[wid] + incl - cnt;
  __syncthreads();
  return r;
}

// block_reserve for one slot per flagged thread (a ballot instead of the
// shuffle scan).
__device__ __forceinline__ int32_t block_reserve_flag(bool f, int32_t* counter, int32_t* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t b = __ballot_sync(0xFFFFFFFFu, f);
  if (lane == 0) sm[wid] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t tot = 0;
    for (int k = 0; k < nw; ++k) {
      const int32_t t = sm[k];
      sm[k] = tot;
      tot += t;
    }
    sm[nw] = tot ? atomicAdd(counter, tot) : 0;
  }
  __syncthreads();
  const int32_t r = sm[nw] + sm[wid] + __popc(b & ((1u << lane) - 1u));
  __syncthreads();
  return r;
}

// Same for (a, b) pairs packed in one u64 counter (hi: a, lo: b); the block's
// sums must stay below 2^32.  Returns the packed first slots.
__device__ __forceinline__ unsigned long long block_reserve2(uint32_t a, uint32_t b,
                                                             unsigned long long* counter,
                                                             unsigned long long* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned long long v = ((unsigned long long)a << 32) | b;
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sm[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int k = 0; k < nw; ++k) {
      const unsigned long long t = sm[k];
      sm[k] = tot;
      tot += t;
    }
    sm[nw] = tot ? atomicAdd(counter, tot) : 0ull;
  }
  __syncthreads();
  const unsigned long long r = sm[nw] + sm[wid] + incl - v;
  __syncthreads();
  return r;
}

// Global union-find over an i32 parent plane.  Every link points to a smaller
// index and the root is the component minimum, so path halving by atomicMin
// never passes the root and never disconnects a node; concurrent unions only
// touch roots (entries equal to themselves).
__device__ __forceinline__ int32_t uf_find_g(int32_t* par, int32_t a) {
  int32_t p = __ldcg(par + a);
  while (p != a) {
    const int32_t gp = __ldcg(par + p);
    if (gp != p) atomicMin(par + a, gp);
    a = p;
    p = gp;
  }
  return a;
}

__device__ __forceinline__ void uf_unite_g(int32_t* par, int32_t a, int32_t b) {
  while (true) {
    a = uf_find_g(par, a);
    b = uf_find_g(par, b);
    if (a == b) return;
    if (a < b) { const int32_t t = a; a = b; b = t; }  // a is the larger root
    const int32_t old = atomicMin(&par[a], b);
    if (old == a) return;
    a = old;
  }
}
// Canonical compaction: labels = 1 + rank of root in raster order; *d_n.
// Must directly follow the ccl_roots call that built `roots` (it reuses that
// call's local-root list and root bitmap).
// clear_acc (optional): the feature accumulators are reset for every label
// while the ranks are assigned (the feature stage then skips k_feat_clear).
// mask_out (run-table form after ccl_roots_bits): also writes the labelled
// mask's bytes (label != 0).
int ccl_canonical(rtg_ctx* ctx, const int32_t* roots, int64_t h, int64_t w,
                  int32_t* labels, int32_t* d_n, const FeatureAcc* clear_acc = nullptr,
                  uint8_t* mask_out = nullptr);
// ccl_roots in the run-table form over a mask given as a 1-bit plane
// (linear words, w % 32 == 0); the caller checked ccl_runs_for.
int ccl_roots_bits(rtg_ctx* ctx, const uint32_t* bits, int64_t h, int64_t w, int conn,
                   int32_t* roots, bool prezeroed);
// Grayscale reconstruction by level decomposition (k_ccl.cu): when J and I
// hold at most kMaxReconLevels distinct non-zero values, R is one seeded
// labelling per value.  recon_clip_levels writes J = min(marker, I) and reads
// the values of J and I back in the same pass (a stream synchronisation);
// *count = -1 when there are more than kMaxReconLevels.
constexpr int kMaxReconLevels = 4;
int recon_clip_levels(rtg_ctx* ctx, const uint8_t* marker, const uint8_t* I, int64_t h,
                      int64_t w, uint8_t* J, uint8_t levels[kMaxReconLevels], int* count);
// J (clipped to I on entry) becomes recon(J, I); uses ctx->m1, m2, i32a, i32b.
int recon_levels(rtg_ctx* ctx, uint8_t* J, const uint8_t* I, int64_t h, int64_t w, int conn,
                 const uint8_t* levels, int count);
// ReconToNuclei candidates = (recon(max(H - h, 0), H) >= t) && tissue by
// threshold decomposition: union-find components of {H >= t} holding a pixel
// with H >= t + h.  scratch may alias out; scratch must differ from hema/tissue.
// prezeroed: the local-root counter (misc[8]) is already zero.
// runs: run-table form (uses u16a, u16b and m2 as scratch) when the shape allows;
// bits_out: in that form `out` receives the candidates as tile row masks
// (ctx->cand_bits says whether it did) for the joint fill/area labelling.
// in_bits (run-table form only): the {fg, seed, tissue} planes of
// launch_colordeconv replace the hema / tissue bytes.
int recon_threshold_uf(rtg_ctx* ctx, const uint8_t* hema, const uint8_t* tissue, int64_t h,
                       int64_t w, int32_t t, int32_t recon_h, int conn, uint8_t* scratch,
                       uint8_t* out, bool prezeroed = false, bool runs = false,
                       bool bits_out = false, uint32_t* const* in_bits = nullptr);
// FillHoles via union-find of the 4-connected background; scratch may alias out.
int fill_holes_uf(rtg_ctx* ctx, const uint8_t* bin, int64_t h, int64_t w,
                  uint8_t* scratch, uint8_t* out);
// FillHoles + 8-connected AreaThreshold of the candidates in one joint
// labelling of foreground (8-conn) and background (4-conn) components.
// Also builds the foreground list + bit plane of `out` (ctx->fg_list,
// misc[4], ctx->fg_bits) for the sparse watershed.
// prezeroed: its counters (misc[9], misc[4]) and the bit-plane pads were
// cleared upstream (the streaming kernel's ClearList).
// out_bytes = false: in the run-table form `out` is not written (the list
// and the bit plane are the output; the sparse watershed reads only those).
// sep_bits: in that form also clear ctx->sep_bits for the watershed's
// separated mask (ctx->sep_bits_live says whether it did).
int fill_area_joint(rtg_ctx* ctx, const uint8_t* cand, int64_t h, int64_t w, int32_t min_area,
                    int32_t max_area, uint8_t* out, bool prezeroed = false, bool out_bytes = true,
                    bool sep_bits = false);
// What fill_area_joint needs cleared, as a ClearList.
ClearList fill_area_clear(rtg_ctx* ctx, int64_t h, int64_t w);
int area_filter(rtg_ctx* ctx, const int32_t* roots, int64_t n,
                int32_t min_area, int32_t max_area, int32_t* counts,
                uint8_t* out);

int edt(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w,
        int32_t* dist2, uint16_t* dq, uint16_t* mk, int32_t ws_h);

// basin doubles as i32 scratch; the ids are only written when want_basin.
// Sparse path: list of the mask's foreground indices + 1-bit plane (bits_base
// has 2 pad words before the plane), and the EDT of the listed pixels only
// (dq of background pixels is not written; a gated whole-tile pass takes over
// when some distance exceeds the windowed search).
constexpr int kBitPad = 2;
// 8-neighbour foreground mask of p (bit t = row-major neighbour t of 8) from
// the 1-bit foreground plane: three funnel-shifted 3-bit windows instead of
// eight byte loads (fgb: the plane after its kBitPad leading pad words).
__device__ __forceinline__ uint32_t fg_nbrs(int h, int w, const uint32_t* __restrict__ fgb,
                                            int32_t p, int y, int x) {
  auto row3 = [&](int32_t q) -> uint32_t {  // bits of columns x-1, x, x+1 of the row of q
    const int32_t b = q - 1;
    const int32_t wi = b >> 5;  // arithmetic shift: -1 before the first word (pad)
    return __funnelshift_r(fgb[wi], fgb[wi + 1], (uint32_t)b & 31u) & 7u;
  };
  const uint32_t edge = (x == 0 ? 1u : 0u) | (x == w - 1 ? 4u : 0u);  // columns outside
  const uint32_t up = y > 0 ? row3(p - w) & ~edge : 0u;
  const uint32_t mid = row3(p) & ~edge;
  const uint32_t dn = y + 1 < h ? row3(p + w) & ~edge : 0u;
  return up | ((mid & 1u) << 3) | ((mid & 4u) << 2) | (dn << 5);
}

// fg_nbrs of the k-th listed pixel p: from the per-list-index cache nbm
// (k_edt_rowdist fills it) or recomputed.
__device__ __forceinline__ uint32_t list_nbrs(int h, const FastDiv& dw,
                                              const uint32_t* __restrict__ fgb,
                                              const uint8_t* __restrict__ nbm, int k, int32_t p) {
  if (nbm) return nbm[k];
  const int w = (int)dw.d;
  const int y = fdiv(p, dw), x = p - y * w;
  return fg_nbrs(h, w, fgb, p, y, x);
}
int fg_list(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w, int32_t* list,
            int32_t* count, uint32_t* bits_base);
// nbm (optional): receives fg_nbrs of every listed pixel by list index.
// hd_mask (optional): the mask's bytes (0 = background), reused in place as
// the row-distance plane (foreground bytes are overwritten with values >= 1,
// so it stays a valid mask).
int edt_list(rtg_ctx* ctx, int64_t h, int64_t w, const int32_t* list,
             const int32_t* count, const uint32_t* bits_base, uint16_t* dq,
             uint8_t* nbm = nullptr, uint8_t* hd_mask = nullptr);
// basin doubles as i32 scratch; the ids are only written when want_basin.
// list_ready: ctx->fg_list / misc[4] / fg_bits already describe `mask`.
int watershed(rtg_ctx* ctx, const uint8_t* mask, int64_t h, int64_t w,
              int32_t ws_h, uint8_t* sep, int32_t* basin, bool want_basin = true,
              bool list_ready = false);
// Object-parallel o6+o7 (default): objects are the global roots of `roots`
// (a ccl_roots forest of `mask`) whose counts lie in [lo, hi] (all roots when
// counts == nullptr).  Writes sep (and basin if non-null) for the whole tile.
int watershed_objects(rtg_ctx* ctx, const uint8_t* mask, const int32_t* roots,
                      const int32_t* counts, int32_t lo, int32_t hi, int64_t h, int64_t w,
                      int32_t ws_h, uint8_t* sep, int32_t* basin);

// list (optional): a foreground list covering every labelled pixel.
int features(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity,
             int64_t h, int64_t w, const int32_t* d_n, float* out,
             const int32_t* list = nullptr, const int32_t* list_count = nullptr,
             bool acc_cleared = false);

// f4 Canny edges (u8 0/1) of an intensity plane; uses i32a/i32b and m1/m2.
int canny(rtg_ctx* ctx, const uint8_t* intensity, int64_t h, int64_t w, int32_t low, int32_t high,
          uint8_t* edges);
// f4 texture table for labels 1..*d_n (out: n x RTG_NUM_TEXTURE).  boxes:
// the feature stage's accumulators (their min / max y, x are the objects'
// bounding boxes), or null to reduce the boxes here.
int texture(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity, int64_t h, int64_t w,
            const int32_t* d_n, float* out, const FeatureAcc* boxes = nullptr);

int synth_dev(rtg_ctx* ctx, uint64_t global_seed, int64_t tile_row,
              int64_t tile_col, int64_t h, int64_t w, uint8_t* d_rgb);

}  // namespace rtg
