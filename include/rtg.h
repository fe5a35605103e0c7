/*
 * rtg.h — C-ABI of the B200 per-tile nucleus segmentation + feature stage.
 *
 * This is the drop-in boundary for the Region Templates hot path
 * (arXiv 1405.7958).  In the reference (/root/reference/proj) the slot where
 * pixels are computed is empty:
 *   - TaskNode::body is a `std::function<void()>` (include/rt/wrm.hpp:63-64),
 *     produced by StageInstance::body (include/rt/dataflow.hpp:48) and invoked
 *     by the executor after WrmState::next (tests/test_acceptance.cpp:590-596);
 *   - the simulator materialises stage outputs with a constant payload
 *     (src/sim.cpp:557-582, run_finalize) and only charges virtual time for
 *     the compute (src/sim.cpp:630-685, start_task).
 * A GPU TaskNode variant calls the functions below from its body.  Payloads
 * are the reference's dense layout: row-major, last axis contiguous
 * (include/rt/data_region.hpp:84-92; put_chunk length check
 * src/data_region.cpp:171-192).  RGB tiles are interleaved HWC u8
 * (RegionKind::kDense3D box <y0,x0,0;y1,x1,2>).
 *
 * Conventions
 *   - Every function returns an rtg_status (0 == RTG_OK).  No C++ exception
 *     crosses this boundary; the failing call's message is available from
 *     rtg_last_error() (thread-local).  The C++ host layer maps codes back
 *     onto the rt::Error taxonomy (include/rt/error.hpp:24-100) exactly the
 *     way throw_wire_error maps WireErrorCode (src/service.cpp:181-219).
 *   - Host-buffer functions (rtg_segment_tile, rtg_features,
 *     rtg_process_tile) are synchronous: H2D copy, kernels, D2H copy.
 *   - *_dev functions take device pointers, enqueue on the context's stream
 *     and return without synchronising (capturable in a CUDA graph).
 *   - The library never frees caller buffers.  Device scratch is owned by the
 *     rtg_ctx arena (no per-call cudaMalloc).
 *   - One rtg_ctx per (GPU, host thread); calls on one ctx are serialised by
 *     the caller.  Contexts on different GPUs run concurrently.
 *   - There is no CPU fallback: without a usable B200 every compute call
 *     fails with RTG_ERR_NO_DEVICE / RTG_ERR_DEVICE.
 */
#ifndef RTG_H
#define RTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTG_ABI_VERSION 1

/* Status codes.  Mapping onto rt::Error subclasses (error.hpp:24-100):
 *   INVALID_ARG -> ConfigError, DIMENSION -> DimensionError,
 *   RANGE -> RangeError, NOT_FOUND -> NotFoundError,
 *   OUT_OF_MEMORY / DEVICE / NO_DEVICE -> DeviceError (added, derives Error),
 *   OVERFLOW -> RangeError, INTERNAL -> Error. */
typedef enum rtg_status {
  RTG_OK = 0,
  RTG_ERR_INVALID_ARG = 1,
  RTG_ERR_DIMENSION = 2,
  RTG_ERR_RANGE = 3,
  RTG_ERR_NOT_FOUND = 4,
  RTG_ERR_OUT_OF_MEMORY = 5,
  RTG_ERR_DEVICE = 6,
  RTG_ERR_NO_DEVICE = 7,
  RTG_ERR_OVERFLOW = 8,
  RTG_ERR_INTERNAL = 9
} rtg_status;

typedef struct rtg_ctx rtg_ctx;

/* Pipeline parameters.  CPU (oracle) and GPU consume the same struct, so the
 * two variants provably run with identical parameters. */
typedef struct rtg_params {
  /* o1 colour deconvolution: H concentration
   * c_H = sum_c h_coef[c] * OD(v_c), OD(v) = -log10((v + 1) / 256),
   * quantised to u8 as round(c_H * 255 / h_scale) via 16.16 fixed-point LUTs. */
  double h_coef[3];
  double h_scale;
  /* o2 thresholds: background = r,g,b all > bg_thresh;
   * RBC = 10*r > rbc_rg10*g && 10*r > rbc_rb10*b.  tissue = !bg && !RBC. */
  int32_t bg_thresh;
  int32_t rbc_rg10;
  int32_t rbc_rb10;
  /* o3 ReconToNuclei: R = reconstruct_by_dilation(max(H - recon_h, 0), H);
   * candidate = R >= nuc_thresh && tissue. */
  int32_t recon_h;
  int32_t recon_conn; /* 4 or 8 */
  int32_t nuc_thresh;
  /* o5 AreaThreshold: keep 8-connected objects with min_area <= area <= max_area. */
  int32_t min_area;
  int32_t max_area;
  /* o6 PreWatershed: d = floor(4 * EDT); F = reconstruct(max(d - ws_h, 0), d). */
  int32_t ws_h;
  /* o9: 1 appends the RTG_NUM_TEXTURE texture columns (histogram, GLCM,
   * Canny edge statistics, PAPER.md:343-345 / :1161-1177) to every feature
   * row, 0 (default) gives the RTG_NUM_FEATURES shape / intensity columns.
   * Row width: rtg_feature_columns(). */
  int32_t texture;
  int32_t reserved[6];
} rtg_params;

/* Per-object feature row (float32, RTG_NUM_FEATURES columns). */
#define RTG_NUM_FEATURES 20
enum rtg_feature {
  RTG_F_AREA = 0,
  RTG_F_PERIMETER = 1,   /* # 4-neighbour pixel edges leaving the object */
  RTG_F_BBOX_Y0 = 2,
  RTG_F_BBOX_X0 = 3,
  RTG_F_BBOX_Y1 = 4,     /* inclusive */
  RTG_F_BBOX_X1 = 5,
  RTG_F_CENTROID_Y = 6,
  RTG_F_CENTROID_X = 7,
  RTG_F_MEAN_I = 8,      /* intensity = hematoxylin plane (u8) */
  RTG_F_STD_I = 9,
  RTG_F_MIN_I = 10,
  RTG_F_MAX_I = 11,
  RTG_F_MEAN_GRAD = 12,  /* Sobel magnitude, floor(4|g|)/4, replicate border */
  RTG_F_STD_GRAD = 13,
  RTG_F_MAJOR_AXIS = 14,
  RTG_F_MINOR_AXIS = 15,
  RTG_F_ECCENTRICITY = 16,
  RTG_F_ORIENTATION = 17,
  RTG_F_CIRCULARITY = 18,
  RTG_F_EXTENT = 19
};

/* Per-object texture row (float32, RTG_NUM_TEXTURE columns): the
 * "histograms and co-occurrence matrices" intermediates of the paper's
 * feature stage.  Intensity is the
 * hematoxylin plane; histogram: 16 bins (v >> 4); grey-level co-occurrence
 * matrix (GLCM): 8 levels (v >> 5), symmetric, summed over the offsets
 * (0,1) (1,0) (1,1) (1,-1) for pixel pairs inside the same object.  All
 * statistics are fp64 over integer intermediates. */
#define RTG_NUM_TEXTURE 14
enum rtg_texture_feature {
  RTG_T_HIST_ENTROPY = 0,   /* -sum p log2 p over the 16-bin histogram */
  RTG_T_HIST_ENERGY = 1,    /* sum p^2 */
  RTG_T_SKEWNESS = 2,       /* third standardised moment of intensity */
  RTG_T_KURTOSIS = 3,       /* fourth standardised moment - 3 */
  RTG_T_GLCM_ASM = 4,       /* sum P^2 */
  RTG_T_GLCM_CONTRAST = 5,  /* sum (i-j)^2 P */
  RTG_T_GLCM_HOMOGENEITY = 6, /* sum P / (1 + (i-j)^2) */
  RTG_T_GLCM_ENTROPY = 7,   /* -sum P log2 P */
  RTG_T_GLCM_CORRELATION = 8, /* (sum ij P - mu^2) / sigma^2 */
  RTG_T_GLCM_DISSIMILARITY = 9, /* sum |i-j| P */
  RTG_T_GLCM_MAX_PROB = 10, /* max P */
  RTG_T_GLCM_CLUSTER_SHADE = 11, /* sum (i + j - 2 mu)^3 P */
  RTG_T_EDGE_PIXELS = 12,   /* Canny edge pixels inside the object (RTG_CANNY_*) */
  RTG_T_EDGE_DENSITY = 13   /* edge pixels / area */
};
/* Canny thresholds the texture table uses (Sobel magnitude of the smoothed
 * intensity; see rtg_canny_dev). */
#define RTG_CANNY_LOW 64
#define RTG_CANNY_HIGH 128

/* ---- lifecycle ---------------------------------------------------------- */

/* Default parameters tuned for H&E tiles (Ruifrok-Johnston stain matrix). */
int rtg_params_default(rtg_params* out);
/* Floats per feature row of the stage under `params`: RTG_NUM_FEATURES, plus
 * RTG_NUM_TEXTURE when params->texture is set (texture columns follow the
 * shape / intensity ones).  Every stage entry point's feature table uses it. */
#define RTG_MAX_FEATURE_COLUMNS (RTG_NUM_FEATURES + RTG_NUM_TEXTURE)
int rtg_feature_columns(const rtg_params* params, int32_t* cols);

/* Number of visible CUDA devices (0 on a CPU-only host; never fails). */
int rtg_device_count(int* n);

/* Creates a context bound to `device` with scratch for tiles up to
 * max_h x max_w and up to max_objects objects per tile.  All device memory is
 * allocated here. */
int rtg_ctx_create(int device, int64_t max_h, int64_t max_w,
                   int32_t max_objects, rtg_ctx** out);
int rtg_ctx_destroy(rtg_ctx* ctx);
/* The cudaStream_t every *_dev call is enqueued on. */
int rtg_ctx_stream(rtg_ctx* ctx, void** stream);
/* Re-targets the context to a caller-owned cudaStream_t (NULL = own stream). */
int rtg_ctx_set_stream(rtg_ctx* ctx, void* stream);
/* Waits for the context's stream and reports sticky device-side errors
 * (object-capacity overflow, queue overflow). */
int rtg_ctx_sync(rtg_ctx* ctx);
/* Device-side counters accumulated since the last call (then reset),
 * for tests / profiling; synchronises:
 *   out[0] objects of the last tile, out[1] IWPP tile visits (all kinds),
 *   out[2] watershed plateau pixels of the last tile,
 *   out[3] 1 if the last EDT needed the whole-tile exact pass (a distance
 *   beyond the windowed EDT's exact range), else 0,
 *   out[4 + 2k] tile visits and out[5 + 2k] sweep iterations of IWPP kind k
 *   (k = 0 ReconToNuclei, 1 HMAX, 2 regional maxima, 3 IWPP fill-holes). */
#define RTG_NUM_STATS 16
int rtg_ctx_stats(rtg_ctx* ctx, int64_t out[RTG_NUM_STATS]);

/* Stage timing (CUDA events on the ctx stream, bracketing each stage of the
 * pipeline).  rtg_ctx_profile_read synchronises, returns the accumulated
 * milliseconds and call counts per stage since the last read, and resets. */
enum rtg_stage {
  RTG_STAGE_COLORDECONV = 0, /* k_colordeconv_vec (o1+o2)                  */
  RTG_STAGE_RECON = 1,       /* IWPP reconstruction (o3)                  */
  RTG_STAGE_FILL_HOLES = 2,  /* candidate threshold + IWPP fill (o4)      */
  RTG_STAGE_AREA = 3,        /* union-find CCL + area filter (o5)         */
  RTG_STAGE_EDT = 4,         /* exact EDT (o6)                            */
  RTG_STAGE_MARKERS = 5,     /* HMAX + regional-maxima IWPP (o6)          */
  RTG_STAGE_WATERSHED = 6,   /* arrows, marker CCL, plateaus, basins (o7) */
  RTG_STAGE_LABEL = 7,       /* final CCL + canonical relabel (o8)        */
  RTG_STAGE_FEATURES = 8,    /* two-step features (o9)                    */
  RTG_STAGE_TEXTURE = 9,     /* Canny + texture columns (params->texture)  */
  RTG_NUM_STAGES = 10
};
int rtg_ctx_profile(rtg_ctx* ctx, int enable);
int rtg_ctx_profile_read(rtg_ctx* ctx, double ms[RTG_NUM_STAGES],
                         int64_t calls[RTG_NUM_STAGES]);
/* Kernels launched through this ctx since creation (host-side counter). */
int rtg_ctx_launches(rtg_ctx* ctx, int64_t* out);

/* Implementation choices that do not change results (all bit-identical). */
enum rtg_option {
  /* FillHoles: 0 = union-find labelling of the 4-connected background
   * (default), 1 = IWPP binary reconstruction from the border on the tile
   * queue. */
  RTG_OPT_FILL_HOLES_IMPL = 0,
  /* rtg_process_tile_dev replays a cached CUDA graph of the whole stage per
   * distinct argument tuple (1, default) or launches kernel by kernel (0). */
  RTG_OPT_USE_GRAPHS = 1,
  /* ReconToNuclei inside the stage: 0 = threshold decomposition (default:
   * the stage only consumes recon >= nuc_thresh, which equals the union-find
   * components of {H >= nuc_thresh} holding a pixel with H >= nuc_thresh +
   * recon_h), 1 = full grayscale IWPP reconstruction then threshold.  The
   * per-operator rtg_recon_*_dev entry points are always the grayscale IWPP. */
  RTG_OPT_RECON_IMPL = 2,
  /* PreWatershed + watershed (stage and rtg_watershed_dev): 0 = tiled
   * whole-tile passes (EDT, HMAX, global arrows, plateau components that
   * also yield the regional maxima) (default), 1 = object-parallel: each
   * object's bounding-box region processed on-chip by one warp. */
  RTG_OPT_WATERSHED_IMPL = 3,
  /* HMAX of the distance map in the tiled watershed: 0 = sparse components
   * (default: a pixel with a neighbour at least ws_h higher keeps its value;
   * the few remaining pixels form small components, one warp each),
   * 1 = IWPP reconstruction on the tile queue. */
  RTG_OPT_HMAX_IMPL = 4,
  /* Programmatic dependent launch between the stage's kernels: 1 = each
   * kernel is scheduled while its predecessor drains (shorter single-stream
   * latency, ~5 %), 0 = plain stream order (default: with several contexts
   * sharing a GPU the waiting CTAs of early-launched kernels cost more
   * throughput than the overlap gains).  Results are identical either way. */
  RTG_OPT_PDL = 5,
  /* rtg_recon_u8_dev: 0 = choose per input (default): when marker and mask
   * hold at most 4 distinct non-zero values, one seeded union-find labelling
   * per value (reconstruction by level decomposition; a long single
   * wavefront, e.g. a maze, costs no more than a short one); otherwise the
   * IWPP tile queue.  The choice reads 64 bytes back (one stream
   * synchronisation) and is skipped under graph capture.  1 = always IWPP. */
  RTG_OPT_RECON_ENTRY_IMPL = 6,
  /* Colour deconvolution (o1+o2): 1 = one CTA per SM fed by a 4-stage ring
   * of 24 KB bulk async copies (TMA, cp.async.bulk + mbarrier) (default);
   * 0 = 128-bit streaming loads with register prefetch, two 512-thread CTAs
   * per SM.  Identical results. */
  RTG_OPT_STREAM_IMPL = 7,
  /* Stage labellings (ReconToNuclei, the joint FillHoles + AreaThreshold,
   * BWLabel): 1 = run-table form where the tile width is a multiple of 32
   * (default): each 32x32 tile keeps its row masks, a table of its runs'
   * local roots and its border pixels' roots instead of a root per pixel,
   * and a per-tile pass writes the outputs; 0 = a root per pixel.
   * Identical results. */
  RTG_OPT_LABEL_RUNS = 8
};
int rtg_ctx_set_option(rtg_ctx* ctx, int option, int64_t value);

/* Debug check of the context's scratch (no reference counterpart: test
 * infrastructure standing in for compute-sanitizer, which this GPU pool does
 * not run).  With RTG_GUARD_BYTES=N in the environment at rtg_ctx_create,
 * every scratch buffer is allocated N bytes larger and the tail filled with
 * a canary; this call synchronises the context's stream and fails with
 * RTG_ERR_INTERNAL (naming the buffer) if any canary byte changed.
 * *n_checked = the number of guarded buffers (0 without RTG_GUARD_BYTES). */
int rtg_ctx_guard_check(rtg_ctx* ctx, int32_t* n_checked);

/* Thread-local message of the last failing call on this thread. */
const char* rtg_last_error(void);

/* Pinned host memory for Chunk payloads (data_region.hpp:87-92, follow-up f1). */
int rtg_host_alloc(size_t bytes, void** out);
int rtg_host_free(void* p);

/* ---- whole tile, host buffers (synchronous) ------------------------------ */

/* Segments one RGB tile: writes the final nucleus mask (u8 0/1, h*w) and the
 * canonical labels (i32, h*w; 1..n in order of each object's minimum linear
 * pixel index, 0 = background).  Either output may be NULL. */
int rtg_segment_tile(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w,
                     int64_t pitch_bytes, const rtg_params* params,
                     uint8_t* mask_out, int32_t* labels_out,
                     int32_t* n_objects);

/* Feature table for a labelled tile: out is n_objects x RTG_NUM_FEATURES f32,
 * row k-1 describes label k. */
int rtg_features(rtg_ctx* ctx, const int32_t* labels, const uint8_t* intensity,
                 int64_t h, int64_t w, int32_t n_objects, float* out);

/* Segmentation + features in one call (the stage body).  features_out holds
 * max_rows rows of rtg_feature_columns(params) floats; *n_objects receives
 * the object count (RTG_ERR_OVERFLOW when it exceeds max_rows).  mask_out /
 * labels_out / hema_out may be NULL. */
int rtg_process_tile(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w,
                     int64_t pitch_bytes, const rtg_params* params,
                     uint8_t* mask_out, int32_t* labels_out, uint8_t* hema_out,
                     float* features_out, int32_t max_rows,
                     int32_t* n_objects);

/* Batch of tiles of one shape (the stage body applied to a bag of tiles).
 * The upload of tile i+1 overlaps the processing of tile i (two device RGB
 * buffers, a copy stream, events); returns when every tile is done.
 * features_out[i] holds max_rows rows (NULL entries skip the table),
 * n_objects[i] receives tile i's object count; RTG_ERR_OVERFLOW when a tile
 * exceeds max_rows (its first max_rows rows are still written).  Host RGB and
 * feature buffers from rtg_host_alloc give full copy/compute overlap. */
int rtg_process_tiles(rtg_ctx* ctx, int32_t count, const uint8_t* const* rgb, int64_t h,
                      int64_t w, int64_t pitch_bytes, const rtg_params* params,
                      float* const* features_out, int32_t max_rows, int32_t* n_objects);

/* ---- whole tile, host buffers, asynchronous (3-phase pipeline) ----------- */

/* The stage body as the paper's upload / compute / download pipeline
 * (the reference models it only in virtual time,
 * src/wrm.cpp:385-415 prefetch_pipeline and src/sim.cpp:672-684).  Enqueues
 * the H2D copy of `rgb`, the stage and the D2H copies of the requested
 * outputs (any of mask_out / labels_out / hema_out / features_out may be
 * NULL) and returns at once with a ticket.  Each context keeps
 * RTG_ASYNC_SLOTS tiles in flight, each with its own device buffers: the
 * upload of tile t+1 overlaps the stage of tile t and the download of tile
 * t-1.  When every slot is busy the call first waits for the oldest ticket
 * (whose result stays available to rtg_ticket_wait).  Host buffers must stay
 * valid, and outputs unread, until the ticket is waited.  Host memory from
 * rtg_host_alloc gives full overlap; pageable outputs make the call block
 * until their copies finish.  features_out holds max_rows rows. */
#define RTG_ASYNC_SLOTS 3
int rtg_process_tile_async(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w,
                           int64_t pitch_bytes, const rtg_params* params,
                           uint8_t* mask_out, int32_t* labels_out, uint8_t* hema_out,
                           float* features_out, int32_t max_rows, uint64_t* ticket);
/* Waits for a ticket's outputs; *n_objects receives the tile's object count.
 * RTG_ERR_OVERFLOW when it exceeds max_rows or the context's max_objects (the
 * first rows are still written); RTG_ERR_NOT_FOUND for an unknown ticket or
 * one already waited. */
int rtg_ticket_wait(rtg_ctx* ctx, uint64_t ticket, int32_t* n_objects);
/* *done = 1 once the ticket's outputs are in host memory (does not block). */
int rtg_ticket_query(rtg_ctx* ctx, uint64_t ticket, int* done);

/* ---- whole tile, device buffers (asynchronous on the ctx stream) --------- */

/* d_rgb: device RGB (pitch_bytes >= 3*w).  d_mask (u8), d_labels (i32),
 * d_hema (u8) may be NULL.  d_features: max_objects x
 * rtg_feature_columns(params) f32 (ctx capacity), d_n_objects: one device
 * int32. */
int rtg_process_tile_dev(rtg_ctx* ctx, const uint8_t* d_rgb, int64_t h,
                         int64_t w, int64_t pitch_bytes,
                         const rtg_params* params, uint8_t* d_mask,
                         int32_t* d_labels, uint8_t* d_hema,
                         float* d_features, int32_t* d_n_objects);

/* ---- per-operator entry points, device buffers (asynchronous) ------------ */

/* o1+o2: hematoxylin plane, HMAX marker max(H - recon_h, 0), tissue mask. */
int rtg_colordeconv_dev(rtg_ctx* ctx, const uint8_t* d_rgb, int64_t h,
                        int64_t w, int64_t pitch_bytes,
                        const rtg_params* params, uint8_t* d_hema,
                        uint8_t* d_marker, uint8_t* d_tissue);
/* o3: grayscale reconstruction by dilation (marker <= mask enforced), 4/8-conn.
 * d_out may alias d_marker.  Algorithm per RTG_OPT_RECON_ENTRY_IMPL. */
int rtg_recon_u8_dev(rtg_ctx* ctx, const uint8_t* d_marker,
                     const uint8_t* d_mask, int64_t h, int64_t w, int conn,
                     uint8_t* d_out);
int rtg_recon_u16_dev(rtg_ctx* ctx, const uint16_t* d_marker,
                      const uint16_t* d_mask, int64_t h, int64_t w, int conn,
                      uint16_t* d_out);
/* o4: binary hole filling (holes = background not 4-connected to the border). */
int rtg_fill_holes_dev(rtg_ctx* ctx, const uint8_t* d_in, int64_t h,
                       int64_t w, uint8_t* d_out);
/* o8: canonical connected-component labels (conn 4/8), *d_n = count. */
int rtg_bwlabel_dev(rtg_ctx* ctx, const uint8_t* d_mask, int64_t h, int64_t w,
                    int conn, int32_t* d_labels, int32_t* d_n);
/* o5: keep conn-connected objects with min_area <= area <= max_area. */
int rtg_area_threshold_dev(rtg_ctx* ctx, const uint8_t* d_mask, int64_t h,
                           int64_t w, int conn, int32_t min_area,
                           int32_t max_area, uint8_t* d_out);
/* o6: exact squared Euclidean distance to the nearest zero pixel of the tile
 * (INT32_MAX when the tile has none). */
int rtg_edt_dev(rtg_ctx* ctx, const uint8_t* d_mask, int64_t h, int64_t w,
                int32_t* d_dist2);
/* o6+o7: PreWatershed + marker watershed on a binary mask.  Writes the
 * separated mask (u8) and, if d_basin != NULL, the per-pixel basin id
 * (1 + linear index of the basin marker's first pixel, 0 = background). */
int rtg_watershed_dev(rtg_ctx* ctx, const uint8_t* d_mask, int64_t h,
                      int64_t w, int32_t ws_h, uint8_t* d_sep_mask,
                      int32_t* d_basin);
/* o9: per-object features for canonical labels 1..*d_n (device count). */
int rtg_features_dev(rtg_ctx* ctx, const int32_t* d_labels,
                     const uint8_t* d_intensity, int64_t h, int64_t w,
                     const int32_t* d_n, float* d_features);

/* Texture table (RTG_NUM_TEXTURE columns) for canonical labels 1..n: one
 * warp per object bounding box builds the histogram + co-occurrence
 * intermediates, one thread per object turns them into the row. */
int rtg_texture_features_dev(rtg_ctx* ctx, const int32_t* d_labels,
                             const uint8_t* d_intensity, int64_t h, int64_t w,
                             const int32_t* d_n, float* d_texture);
/* Canny edges of an intensity plane: 5x5 binomial smoothing ((sum + 128) >>
 * 8), Sobel, squared magnitude m2 = gx^2 + gy^2, non-maximum suppression
 * along the quantised gradient direction (keep m2 > m2(prev) && m2 >=
 * m2(next); outside pixels are 0), then hysteresis: a kept pixel with m2 >
 * low^2 is an edge iff its 8-connected component of such pixels holds one
 * with m2 > high^2 (replicate borders throughout).  d_edges: u8 0/1. */
int rtg_canny_dev(rtg_ctx* ctx, const uint8_t* d_intensity, int64_t h, int64_t w,
                  int32_t low, int32_t high, uint8_t* d_edges);
/* Host-buffer variant: out is n_objects x RTG_NUM_TEXTURE f32. */
int rtg_texture_features(rtg_ctx* ctx, const int32_t* labels,
                         const uint8_t* intensity, int64_t h, int64_t w,
                         int32_t n_objects, float* out);

/* ---- synthetic H&E tiles (deterministic, splitmix64 as src/sim.cpp:33-44) */

/* tile seed = splitmix64(global_seed ^ (tile_row << 32 | tile_col)). */
int rtg_synth_tile_host(uint64_t global_seed, int64_t tile_row,
                        int64_t tile_col, int64_t h, int64_t w, uint8_t* rgb);
int rtg_synth_tile_dev(rtg_ctx* ctx, uint64_t global_seed, int64_t tile_row,
                       int64_t tile_col, int64_t h, int64_t w, uint8_t* d_rgb);

#ifdef __cplusplus
}
#endif

#endif /* RTG_H */
