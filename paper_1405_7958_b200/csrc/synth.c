/* Host side of the synthetic tile generator (see synth.h). */
#include "synth.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "rtg.h"

/* Uniform [0, 1) draw number i of the tile's stream (53-bit, as
 * sim.cpp:42-44 unit_draw). */
static double draw(uint64_t seed, uint64_t* i) {
  return (double)(rtg_splitmix64(seed + (*i)++) >> 11) * 0x1.0p-53;
}

static int64_t scaled_count(double per_full_tile, int64_t h, int64_t w) {
  return (int64_t)floor(per_full_tile * (double)(h * w) / (4096.0 * 4096.0) +
                        0.5);
}

int64_t rtg_synth_max_shapes(int64_t h, int64_t w) {
  return 4 * scaled_count(15500.0, h, w) + scaled_count(450.0, h, w) + 8;
}

static void make_ellipse(rtg_shape* s, double cy, double cx, double a,
                         double b, double theta, uint32_t key, int32_t tint) {
  const double S = 1048576.0; /* 2^20 fixed point */
  const double c = cos(theta), sn = sin(theta);
  const double ia = 1.0 / (a * a), ib = 1.0 / (b * b);
  s->cy = (int32_t)floor(cy);
  s->cx = (int32_t)floor(cx);
  s->A = llround(S * (c * c * ia + sn * sn * ib));
  s->B = llround(S * 2.0 * c * sn * (ia - ib));
  s->C = llround(S * (sn * sn * ia + c * c * ib));
  s->K = (int64_t)S;
  const int32_t r = (int32_t)ceil(a > b ? a : b) + 1;
  s->y0 = s->cy - r;
  s->y1 = s->cy + r;
  s->x0 = s->cx - r;
  s->x1 = s->cx + r;
  s->key = key;
  s->tint = tint;
}

int64_t rtg_synth_shapes(uint64_t seed, int64_t h, int64_t w,
                         rtg_shape* out) {
  uint64_t i = 0;
  int64_t n = 0;
  const double pi = 3.14159265358979323846;
  /* Slide-glass patches: up to two large ellipses per full tile. */
  const int64_t n_glass = scaled_count(2.0 * draw(seed, &i), h, w);
  for (int64_t g = 0; g < n_glass; ++g) {
    const double cy = draw(seed, &i) * (double)h;
    const double cx = draw(seed, &i) * (double)w;
    const double a = 150.0 + 350.0 * draw(seed, &i);
    const double b = a * (0.5 + 0.5 * draw(seed, &i));
    const double th = pi * draw(seed, &i);
    make_ellipse(&out[n], cy, cx, a, b, th,
                 ((uint32_t)RTG_CLASS_GLASS << 24) | (uint32_t)n, 0);
    ++n;
  }
  /* Red blood cells. */
  const int64_t n_rbc = scaled_count(450.0, h, w);
  for (int64_t k = 0; k < n_rbc; ++k) {
    const double cy = draw(seed, &i) * (double)h;
    const double cx = draw(seed, &i) * (double)w;
    const double a = 3.0 + 3.0 * draw(seed, &i);
    const double b = a * (0.7 + 0.3 * draw(seed, &i));
    const double th = pi * draw(seed, &i);
    const int32_t tint = (int32_t)floor(draw(seed, &i) * 21.0) - 10;
    make_ellipse(&out[n], cy, cx, a, b, th,
                 ((uint32_t)RTG_CLASS_RBC << 24) | (uint32_t)n, tint);
    ++n;
  }
  /* Nuclei, placed in clusters of 1-4 so a good fraction touch or overlap
   * (drives the watershed split). */
  const int64_t n_clusters = scaled_count(15500.0, h, w);
  for (int64_t k = 0; k < n_clusters; ++k) {
    const double u = draw(seed, &i);
    const int members = u < 0.55 ? 1 : u < 0.85 ? 2 : u < 0.95 ? 3 : 4;
    double cy = draw(seed, &i) * (double)h;
    double cx = draw(seed, &i) * (double)w;
    double prev_a = 0.0;
    for (int m = 0; m < members; ++m) {
      const double a = 4.0 + 5.0 * draw(seed, &i);
      const double b = a * (0.6 + 0.4 * draw(seed, &i));
      const double th = pi * draw(seed, &i);
      const int32_t tint = (int32_t)floor(draw(seed, &i) * 41.0) - 20;
      if (m > 0) {
        const double dir = 2.0 * pi * draw(seed, &i);
        const double dist = (prev_a + a) * (0.75 + 0.3 * draw(seed, &i));
        cy += dist * sin(dir);
        cx += dist * cos(dir);
      }
      make_ellipse(&out[n], cy, cx, a, b, th,
                   ((uint32_t)RTG_CLASS_NUCLEUS << 24) | (uint32_t)n, tint);
      ++n;
      prev_a = a;
    }
  }
  return n;
}

/* Per-pixel colour from the winning shape key and the noise hash; shared
 * formula with the device kernel k_synth_colour (synth_dev.cu). */
static void colour_pixel(uint64_t seed, const rtg_shape* shapes, uint32_t key,
                         int64_t idx, uint8_t* px) {
  const int cls = key ? (int)(key >> 24) : RTG_CLASS_STROMA;
  const int32_t tint = key ? shapes[key & 0xFFFFFFu].tint : 0;
  const uint64_t z = rtg_splitmix64(seed ^ 0xd1b54a32d192ed03ULL ^
                                    (uint64_t)idx);
  for (int c = 0; c < 3; ++c) {
    const int a = (int)((z >> (16 * c)) & 0xFF);
    const int b = (int)((z >> (16 * c + 8)) & 0xFF);
    int v = rtg_synth_base(cls, c) + tint + ((a + b) >> 4) - 16;
    px[c] = (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
  }
}

int rtg_synth_raster_host(uint64_t seed, const rtg_shape* shapes, int64_t n,
                          int64_t h, int64_t w, uint8_t* rgb) {
  uint32_t* key = (uint32_t*)calloc((size_t)(h * w), sizeof(uint32_t));
  if (!key) return RTG_ERR_OUT_OF_MEMORY;
  for (int64_t s = 0; s < n; ++s) {
    const rtg_shape* sh = &shapes[s];
    const int64_t y0 = sh->y0 < 0 ? 0 : sh->y0;
    const int64_t y1 = sh->y1 >= h ? h - 1 : sh->y1;
    const int64_t x0 = sh->x0 < 0 ? 0 : sh->x0;
    const int64_t x1 = sh->x1 >= w ? w - 1 : sh->x1;
    for (int64_t y = y0; y <= y1; ++y) {
      const int64_t dy = y - sh->cy;
      for (int64_t x = x0; x <= x1; ++x) {
        const int64_t dx = x - sh->cx;
        if (sh->A * dx * dx + sh->B * dx * dy + sh->C * dy * dy <= sh->K) {
          /* shape keys carry class >= 1 in the top byte, so 0 = no shape */
          uint32_t* k = &key[y * w + x];
          if (sh->key > *k) *k = sh->key;
        }
      }
    }
  }
  for (int64_t p = 0; p < h * w; ++p) colour_pixel(seed, shapes, key[p], p, &rgb[3 * p]);
  free(key);
  return RTG_OK;
}

int rtg_synth_tile_host(uint64_t global_seed, int64_t tile_row,
                        int64_t tile_col, int64_t h, int64_t w, uint8_t* rgb) {
  if (!rgb || h <= 0 || w <= 0) return RTG_ERR_INVALID_ARG;
  const uint64_t seed = rtg_tile_seed(global_seed, tile_row, tile_col);
  rtg_shape* shapes =
      (rtg_shape*)malloc(sizeof(rtg_shape) * (size_t)rtg_synth_max_shapes(h, w));
  if (!shapes) return RTG_ERR_OUT_OF_MEMORY;
  const int64_t n = rtg_synth_shapes(seed, h, w, shapes);
  const int st = rtg_synth_raster_host(seed, shapes, n, h, w, rgb);
  free(shapes);
  return st;
}
