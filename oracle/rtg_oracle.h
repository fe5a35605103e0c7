/*
 * rtg_oracle.h — CPU ORACLE for the per-tile segmentation + feature stage.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline — never as the product path.
 *
 * Parity status: the reference (/root/reference) ships NO image-analysis
 * arithmetic (SPEC.md:15 puts every operator out of scope; the compute slot is
 * a constant fill, src/sim.cpp:557-582).  This oracle is therefore a
 * sequential restatement of the operator pipeline the paper describes
 * with the exact semantics fixed
 * in DESIGN.md §3.  It is pinned against independent implementations in this
 * container (scipy.ndimage 1.18.1, OpenCV 4.13) through golden vectors
 * committed under tests/golden/ (generator: tests/golden/make_golden.py):
 * reconstruction (iterated grey dilation), binary_fill_holes, label,
 * distance_transform_edt, and the feature moments.  The watershed has no
 * third-party twin with identical tie rules; it is pinned by a brute-force
 * restatement in the golden script plus order-independence properties.
 *
 * Algorithms deliberately differ from the CUDA ones (sequential Vincent
 * hybrid reconstruction, BFS flood labelling, Meijster EDT, BFS plateau
 * distances) so agreement is evidence, not a shared bug.
 */
#ifndef RTG_ORACLE_H
#define RTG_ORACLE_H

#include <stdint.h>

#include "../include/rtg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Optional intermediate planes of orc_process_tile (each may be NULL). */
typedef struct orc_planes {
  uint8_t* hema;      /* o1 hematoxylin u8 */
  uint8_t* marker;    /* o1 HMAX marker max(H - recon_h, 0) */
  uint8_t* tissue;    /* o2 */
  uint8_t* recon;     /* o3 reconstruction of marker under H */
  uint8_t* cand;      /* o3 candidate mask */
  uint8_t* filled;    /* o4 */
  uint8_t* area;      /* o5 */
  int32_t* dist2;     /* o6 squared EDT */
  uint16_t* dq;       /* o6 floor(4*EDT) */
  uint16_t* fw;       /* o6 fg ? HMAX(dq)+1 : 0 */
  uint8_t* rmax;      /* o6 regional maxima (markers) */
  int32_t* basin;     /* o7 1 + marker root index */
  uint8_t* sep;       /* o7 separated mask */
} orc_planes;

void orc_hema_lut(const rtg_params* p, int32_t lut[3][256]);
void orc_colordeconv(const uint8_t* rgb, int64_t h, int64_t w, int64_t pitch,
                     const rtg_params* p, uint8_t* hema, uint8_t* marker,
                     uint8_t* tissue);
/* Grayscale reconstruction by dilation, Vincent (1993) hybrid algorithm. */
void orc_recon_u8(const uint8_t* marker, const uint8_t* mask, int64_t h,
                  int64_t w, int conn, uint8_t* out);
void orc_recon_u16(const uint16_t* marker, const uint16_t* mask, int64_t h,
                   int64_t w, int conn, uint16_t* out);
void orc_fill_holes(const uint8_t* in, int64_t h, int64_t w, uint8_t* out);
/* Canonical labels 1..n by first pixel in raster order; returns n. */
int32_t orc_bwlabel(const uint8_t* mask, int64_t h, int64_t w, int conn,
                    int32_t* labels);
void orc_area_threshold(const uint8_t* in, int64_t h, int64_t w, int conn,
                        int32_t min_area, int32_t max_area, uint8_t* out);
void orc_edt_sq(const uint8_t* mask, int64_t h, int64_t w, int32_t* dist2);
uint32_t orc_isqrt(uint64_t x);
/* PreWatershed + watershed on a binary mask: sep mask and basin ids. */
void orc_watershed(const uint8_t* mask, int64_t h, int64_t w, int32_t ws_h,
                   uint8_t* sep, int32_t* basin, orc_planes* planes);
/* Features for labels 1..n; out = n x RTG_NUM_FEATURES. */
void orc_features(const int32_t* labels, const uint8_t* intensity, int64_t h,
                  int64_t w, int32_t n, float* out);
/* Texture table for labels 1..n; out = n x RTG_NUM_TEXTURE (rtg.h enum
 * rtg_texture_feature).  orc_texture_row turns one object's integer
 * intermediates (16-bin histogram, 8x8 symmetric GLCM, intensity moments
 * sum v^1..v^4) into the row; the GPU finalizer mirrors it term by term. */
void orc_texture(const int32_t* labels, const uint8_t* intensity, int64_t h, int64_t w,
                 int32_t n, float* out);
void orc_texture_row(const uint32_t hist[16], const uint32_t glcm[64], const int64_t mom[4],
                     uint32_t edge_px, float* out);
/* Canny edges (rtg.h rtg_canny_dev): BFS hysteresis from the strong pixels. */
void orc_canny(const uint8_t* I, int64_t h, int64_t w, int32_t low, int32_t high,
               uint8_t* edges);
/* Full stage.  Returns object count (features written for min(n, max_rows)). */
/* features: max_rows rows of RTG_NUM_FEATURES (+ RTG_NUM_TEXTURE when
 * p->texture) floats. */
int32_t orc_process_tile(const uint8_t* rgb, int64_t h, int64_t w,
                         int64_t pitch, const rtg_params* p, uint8_t* mask,
                         int32_t* labels, float* features, int32_t max_rows,
                         orc_planes* planes);
/* Same default parameters as rtg_params_default (restated independently). */
void orc_params_default(rtg_params* p);

#ifdef __cplusplus
}
#endif

#endif
