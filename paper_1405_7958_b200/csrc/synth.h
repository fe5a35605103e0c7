/* Synthetic H&E-like tiles: deterministic shape list + integer rasteriser.
 *
 * Seeding follows the reference simulator's portable PRNG (splitmix64,
 * /root/reference/proj/src/sim.cpp:33-44): tile seed =
 * splitmix64(global_seed ^ (tile_row << 32 | tile_col)).  The shape list is
 * generated once on the host; the host rasteriser (rtg_synth_tile_host) and
 * the device rasteriser (k_synth_* in synth_dev.cu) consume the same integer
 * shapes and the same per-pixel noise hash, so they are byte-identical.
 */
#ifndef RTG_SYNTH_H
#define RTG_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { RTG_CLASS_STROMA = 0, RTG_CLASS_GLASS = 1, RTG_CLASS_RBC = 2,
       RTG_CLASS_NUCLEUS = 3 };

typedef struct rtg_shape {
  int32_t cy, cx;          /* centre, tile-local (may lie outside the tile) */
  int32_t y0, x0, y1, x1;  /* inclusive bounding box, unclipped */
  int64_t A, B, C, K;      /* inside iff A dx^2 + B dx dy + C dy^2 <= K */
  uint32_t key;            /* (class << 24) | index in the shape array */
  int32_t tint;            /* added to every channel of covered pixels */
} rtg_shape;

#define RTG_DEFAULT_SEED 1405795800ULL

static inline uint64_t rtg_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

static inline uint64_t rtg_tile_seed(uint64_t global_seed, int64_t tile_row,
                                     int64_t tile_col) {
  return rtg_splitmix64(global_seed ^ (((uint64_t)tile_row << 32) |
                                       (uint64_t)(uint32_t)tile_col));
}

/* Upper bound on the number of shapes for an h x w tile. */
int64_t rtg_synth_max_shapes(int64_t h, int64_t w);
/* Fills `out` (capacity >= rtg_synth_max_shapes) and returns the count. */
int64_t rtg_synth_shapes(uint64_t tile_seed, int64_t h, int64_t w,
                         rtg_shape* out);

/* Base colour of a class, channel c. */
static inline int rtg_synth_base(int cls, int c) {
  static const unsigned char base[4][3] = {
      {230, 160, 200}, /* stroma: eosin pink */
      {242, 238, 242}, /* slide glass */
      {205, 70, 80},   /* red blood cell */
      {95, 70, 155}};  /* nucleus: hematoxylin */
  return base[cls][c];
}

#ifdef __cplusplus
}
#endif

#endif /* RTG_SYNTH_H */
