/*
 * rtg_oracle.c — sequential CPU restatement of the segmentation + feature
 * stage.  TEST INFRASTRUCTURE ONLY (see rtg_oracle.h for the usage rule and
 * the parity-pinning story).
 *
 * Paper anchors (the reference has no code for these operators):
 *   colour deconvolution + thresholds
 *   ReconToNuclei / FillHoles / PreWatershed (IWPP)
 *   Watershed (Koerbes arrowing)
 *   BWLabel (union-find)
 *   AreaThreshold
 *   Feature computation (two-step)
 * Exact semantics: DESIGN.md §3.
 */
#include "rtg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

void orc_params_default(rtg_params* p) {
  memset(p, 0, sizeof(*p));
  /* column 0 of inv(normalised Ruifrok-Johnston H&E stain matrix) */
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
}

/* ---- neighbourhoods ------------------------------------------------------ */

static const int DY8[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
static const int DX8[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
static const int DY4[4] = {-1, 0, 0, 1};
static const int DX4[4] = {0, -1, 1, 0};

/* ---- o1/o2 ---------------------------------------------------------------- */

void orc_hema_lut(const rtg_params* p, int32_t lut[3][256]) {
  const double scale255 = 255.0 / p->h_scale;
  for (int c = 0; c < 3; ++c) {
    for (int v = 0; v < 256; ++v) {
      const double od = -log10((double)(v + 1) / 256.0);
      lut[c][v] = (int32_t)llround(p->h_coef[c] * od * scale255 * 65536.0);
    }
  }
}

void orc_colordeconv(const uint8_t* rgb, int64_t h, int64_t w, int64_t pitch,
                     const rtg_params* p, uint8_t* hema, uint8_t* marker,
                     uint8_t* tissue) {
  int32_t lut[3][256];
  orc_hema_lut(p, lut);
  for (int64_t y = 0; y < h; ++y) {
    for (int64_t x = 0; x < w; ++x) {
      const uint8_t* px = rgb + y * pitch + 3 * x;
      const int r = px[0], g = px[1], b = px[2];
      const int32_t s = lut[0][r] + lut[1][g] + lut[2][b];
      int hv = 0;
      if (s > 0) {
        hv = (s + 32768) >> 16;
        if (hv > 255) hv = 255;
      }
      const int64_t i = y * w + x;
      if (hema) hema[i] = (uint8_t)hv;
      if (marker) marker[i] = (uint8_t)(hv > p->recon_h ? hv - p->recon_h : 0);
      if (tissue) {
        const int bg = r > p->bg_thresh && g > p->bg_thresh && b > p->bg_thresh;
        const int rbc = 10 * r > p->rbc_rg10 * g && 10 * r > p->rbc_rb10 * b;
        tissue[i] = (uint8_t)(!bg && !rbc);
      }
    }
  }
}

/* ---- o3: Vincent hybrid reconstruction on int32 planes ------------------- */

typedef struct {
  int64_t* v;
  int64_t head, tail, cap;
} fifo;

static void fifo_init(fifo* q, int64_t cap) {
  q->v = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  q->head = q->tail = 0;
  q->cap = cap;
}
static void fifo_push(fifo* q, int64_t x) {
  if (q->tail == q->cap) { /* compact or grow */
    if (q->head > 0) {
      memmove(q->v, q->v + q->head, sizeof(int64_t) * (size_t)(q->tail - q->head));
      q->tail -= q->head;
      q->head = 0;
    } else {
      q->cap *= 2;
      q->v = (int64_t*)realloc(q->v, sizeof(int64_t) * (size_t)q->cap);
    }
  }
  q->v[q->tail++] = x;
}

static void recon_i32(int32_t* J, const int32_t* I, int64_t h, int64_t w,
                      int conn) {
  const int64_t n = h * w;
  for (int64_t i = 0; i < n; ++i) if (J[i] > I[i]) J[i] = I[i];
  /* raster scan over N+ (already visited neighbours) */
  for (int64_t y = 0; y < h; ++y) {
    for (int64_t x = 0; x < w; ++x) {
      const int64_t i = y * w + x;
      int32_t m = J[i];
      if (x > 0 && J[i - 1] > m) m = J[i - 1];
      if (y > 0) {
        if (J[i - w] > m) m = J[i - w];
        if (conn == 8) {
          if (x > 0 && J[i - w - 1] > m) m = J[i - w - 1];
          if (x + 1 < w && J[i - w + 1] > m) m = J[i - w + 1];
        }
      }
      J[i] = m < I[i] ? m : I[i];
    }
  }
  /* anti-raster scan over N-, seeding the FIFO */
  fifo q;
  fifo_init(&q, 1024);
  for (int64_t y = h - 1; y >= 0; --y) {
    for (int64_t x = w - 1; x >= 0; --x) {
      const int64_t i = y * w + x;
      int32_t m = J[i];
      if (x + 1 < w && J[i + 1] > m) m = J[i + 1];
      if (y + 1 < h) {
        if (J[i + w] > m) m = J[i + w];
        if (conn == 8) {
          if (x + 1 < w && J[i + w + 1] > m) m = J[i + w + 1];
          if (x > 0 && J[i + w - 1] > m) m = J[i + w - 1];
        }
      }
      J[i] = m < I[i] ? m : I[i];
      /* push p if some N- neighbour can still grow from it */
      int push = 0;
#define ORC_CHK(cond, j) \
  if (!push && (cond) && J[j] < J[i] && J[j] < I[j]) push = 1;
      ORC_CHK(x + 1 < w, i + 1);
      ORC_CHK(y + 1 < h, i + w);
      if (conn == 8) {
        ORC_CHK(y + 1 < h && x + 1 < w, i + w + 1);
        ORC_CHK(y + 1 < h && x > 0, i + w - 1);
      }
#undef ORC_CHK
      if (push) fifo_push(&q, i);
    }
  }
  const int nn = conn == 8 ? 8 : 4;
  const int* dy = conn == 8 ? DY8 : DY4;
  const int* dx = conn == 8 ? DX8 : DX4;
  while (q.head < q.tail) {
    const int64_t i = q.v[q.head++];
    const int64_t y = i / w, x = i % w;
    for (int k = 0; k < nn; ++k) {
      const int64_t yy = y + dy[k], xx = x + dx[k];
      if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
      const int64_t j = yy * w + xx;
      if (J[j] < J[i] && I[j] != J[j]) {
        J[j] = J[i] < I[j] ? J[i] : I[j];
        fifo_push(&q, j);
      }
    }
  }
  free(q.v);
}

void orc_recon_u8(const uint8_t* marker, const uint8_t* mask, int64_t h,
                  int64_t w, int conn, uint8_t* out) {
  const int64_t n = h * w;
  int32_t* J = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t* I = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  for (int64_t i = 0; i < n; ++i) { J[i] = marker[i]; I[i] = mask[i]; }
  recon_i32(J, I, h, w, conn);
  for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)J[i];
  free(J);
  free(I);
}

void orc_recon_u16(const uint16_t* marker, const uint16_t* mask, int64_t h,
                   int64_t w, int conn, uint16_t* out) {
  const int64_t n = h * w;
  int32_t* J = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t* I = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  for (int64_t i = 0; i < n; ++i) { J[i] = marker[i]; I[i] = mask[i]; }
  recon_i32(J, I, h, w, conn);
  for (int64_t i = 0; i < n; ++i) out[i] = (uint16_t)J[i];
  free(J);
  free(I);
}

/* ---- o4: fill holes (background flood from the border, 4-connected) ------ */

void orc_fill_holes(const uint8_t* in, int64_t h, int64_t w, uint8_t* out) {
  const int64_t n = h * w;
  uint8_t* reach = (uint8_t*)calloc((size_t)n, 1);
  fifo q;
  fifo_init(&q, 1024);
  for (int64_t y = 0; y < h; ++y) {
    for (int64_t x = 0; x < w; ++x) {
      if (y != 0 && y != h - 1 && x != 0 && x != w - 1) continue;
      const int64_t i = y * w + x;
      if (!in[i] && !reach[i]) { reach[i] = 1; fifo_push(&q, i); }
    }
  }
  while (q.head < q.tail) {
    const int64_t i = q.v[q.head++];
    const int64_t y = i / w, x = i % w;
    for (int k = 0; k < 4; ++k) {
      const int64_t yy = y + DY4[k], xx = x + DX4[k];
      if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
      const int64_t j = yy * w + xx;
      if (!in[j] && !reach[j]) { reach[j] = 1; fifo_push(&q, j); }
    }
  }
  for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)(in[i] || !reach[i]);
  free(q.v);
  free(reach);
}

/* ---- o8: canonical labelling by raster-order BFS flood -------------------- */

int32_t orc_bwlabel(const uint8_t* mask, int64_t h, int64_t w, int conn,
                    int32_t* labels) {
  const int64_t n = h * w;
  memset(labels, 0, sizeof(int32_t) * (size_t)n);
  const int nn = conn == 8 ? 8 : 4;
  const int* dy = conn == 8 ? DY8 : DY4;
  const int* dx = conn == 8 ? DX8 : DX4;
  fifo q;
  fifo_init(&q, 1024);
  int32_t next = 0;
  for (int64_t s = 0; s < n; ++s) {
    if (!mask[s] || labels[s]) continue;
    ++next;
    labels[s] = next;
    q.head = q.tail = 0;
    fifo_push(&q, s);
    while (q.head < q.tail) {
      const int64_t i = q.v[q.head++];
      const int64_t y = i / w, x = i % w;
      for (int k = 0; k < nn; ++k) {
        const int64_t yy = y + dy[k], xx = x + dx[k];
        if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
        const int64_t j = yy * w + xx;
        if (mask[j] && !labels[j]) { labels[j] = next; fifo_push(&q, j); }
      }
    }
  }
  free(q.v);
  return next;
}

/* ---- o5 ------------------------------------------------------------------- */

void orc_area_threshold(const uint8_t* in, int64_t h, int64_t w, int conn,
                        int32_t min_area, int32_t max_area, uint8_t* out) {
  const int64_t n = h * w;
  int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  const int32_t k = orc_bwlabel(in, h, w, conn, lab);
  int64_t* area = (int64_t*)calloc((size_t)k + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) area[lab[i]]++;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t l = lab[i];
    out[i] = (uint8_t)(l > 0 && area[l] >= min_area && area[l] <= max_area);
  }
  free(area);
  free(lab);
}

/* ---- o6: Meijster exact squared EDT -------------------------------------- */

static int64_t floordiv(int64_t a, int64_t b) { /* b > 0 */
  int64_t q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}

void orc_edt_sq(const uint8_t* mask, int64_t h, int64_t w, int32_t* dist2) {
  const int64_t n = h * w;
  const int64_t INF = h + w + 1;
  int64_t* g = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int any_zero = 0;
  for (int64_t x = 0; x < w; ++x) {
    int64_t run = INF;
    for (int64_t y = 0; y < h; ++y) {
      const int64_t i = y * w + x;
      if (!mask[i]) { run = 0; any_zero = 1; }
      else if (run < INF) ++run;
      g[i] = run;
    }
    run = INF;
    for (int64_t y = h - 1; y >= 0; --y) {
      const int64_t i = y * w + x;
      if (!mask[i]) run = 0;
      else if (run < INF) ++run;
      if (run < g[i]) g[i] = run;
    }
  }
  if (!any_zero) {
    for (int64_t i = 0; i < n; ++i) dist2[i] = INT32_MAX;
    free(g);
    return;
  }
  int64_t* s = (int64_t*)malloc(sizeof(int64_t) * (size_t)w);
  int64_t* t = (int64_t*)malloc(sizeof(int64_t) * (size_t)w);
  for (int64_t y = 0; y < h; ++y) {
    const int64_t* gr = g + y * w;
#define F(xx, ii) (((xx) - (ii)) * ((xx) - (ii)) + gr[ii] * gr[ii])
    int64_t q = 0;
    s[0] = 0;
    t[0] = 0;
    for (int64_t u = 1; u < w; ++u) {
      while (q >= 0 && F(t[q], s[q]) > F(t[q], u)) --q;
      if (q < 0) {
        q = 0;
        s[0] = u;
      } else {
        const int64_t i = s[q];
        const int64_t sep = floordiv(u * u - i * i + gr[u] * gr[u] - gr[i] * gr[i],
                                     2 * (u - i));
        const int64_t ww = 1 + sep;
        if (ww < w) {
          ++q;
          s[q] = u;
          t[q] = ww;
        }
      }
    }
    for (int64_t u = w - 1; u >= 0; --u) {
      dist2[y * w + u] = (int32_t)F(u, s[q]);
      if (u == t[q]) --q;
    }
#undef F
  }
  free(s);
  free(t);
  free(g);
}

uint32_t orc_isqrt(uint64_t x) {
  uint64_t r = (uint64_t)sqrt((double)x);
  while (r * r > x) --r;
  while ((r + 1) * (r + 1) <= x) ++r;
  return (uint32_t)r;
}

/* ---- o6 + o7: PreWatershed markers and arrowing watershed ---------------- */

void orc_watershed(const uint8_t* mask, int64_t h, int64_t w, int32_t ws_h,
                   uint8_t* sep, int32_t* basin, orc_planes* planes) {
  const int64_t n = h * w;
  int32_t* d2 = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  orc_edt_sq(mask, h, w, d2);
  uint16_t* dq = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
  uint16_t* mk = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    uint32_t v = d2[i] == INT32_MAX ? 65535u : orc_isqrt(16ull * (uint64_t)d2[i]);
    if (v > 65534u) v = 65534u;
    dq[i] = (uint16_t)v;
    mk[i] = (uint16_t)(v > (uint32_t)ws_h ? v - (uint32_t)ws_h : 0u);
  }
  uint16_t* F = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
  orc_recon_u16(mk, dq, h, w, 8, F);
  /* Fw = fg ? HMAX + 1 : 0 keeps every relation inside the foreground */
  for (int64_t i = 0; i < n; ++i) F[i] = mask[i] ? (uint16_t)(F[i] + 1) : 0;
  /* regional maxima: Fw > recon(Fw - 1, Fw) */
  for (int64_t i = 0; i < n; ++i) mk[i] = F[i] ? (uint16_t)(F[i] - 1) : 0;
  uint16_t* G = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
  orc_recon_u16(mk, F, h, w, 8, G);
  uint8_t* rm = (uint8_t*)malloc((size_t)n);
  for (int64_t i = 0; i < n; ++i) rm[i] = (uint8_t)(F[i] > G[i]);
  /* marker ids: 1 + minimum linear index of each 8-connected marker */
  int32_t* mlab = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  const int32_t nm = orc_bwlabel(rm, h, w, 8, mlab);
  int64_t* first = (int64_t*)malloc(sizeof(int64_t) * ((size_t)nm + 1));
  for (int32_t k = 0; k <= nm; ++k) first[k] = -1;
  for (int64_t i = 0; i < n; ++i)
    if (mlab[i] && first[mlab[i]] < 0) first[mlab[i]] = i;
  /* arrows: steepest ascent (max Fw, then min index) for pixels with a
   * higher foreground neighbour; plateau pixels descend the BFS distance
   * delta to the plateau's exits (min index among delta-1 neighbours). */
  int64_t* ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int32_t* delta = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  fifo q;
  fifo_init(&q, 1024);
  for (int64_t i = 0; i < n; ++i) {
    ptr[i] = -1;
    delta[i] = -1;
    if (!F[i]) continue;
    if (rm[i]) { ptr[i] = i; continue; }
    const int64_t y = i / w, x = i % w;
    uint16_t best = F[i];
    int64_t arg = -1;
    for (int k = 0; k < 8; ++k) {
      const int64_t yy = y + DY8[k], xx = x + DX8[k];
      if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
      const int64_t j = yy * w + xx;
      /* neighbours are visited in increasing linear index, so the first
       * strict maximum is the minimum-index one */
      if (F[j] > best) {
        best = F[j];
        arg = j;
      }
    }
    if (arg >= 0) {
      ptr[i] = arg;
      delta[i] = 0;
      fifo_push(&q, i);
    }
  }
  /* BFS over same-level flat pixels (8-connected) */
  while (q.head < q.tail) {
    const int64_t i = q.v[q.head++];
    const int64_t y = i / w, x = i % w;
    for (int k = 0; k < 8; ++k) {
      const int64_t yy = y + DY8[k], xx = x + DX8[k];
      if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
      const int64_t j = yy * w + xx;
      if (F[j] == F[i] && !rm[j] && delta[j] < 0) {
        delta[j] = delta[i] + 1;
        fifo_push(&q, j);
      }
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    if (!F[i] || rm[i] || delta[i] <= 0) continue;
    const int64_t y = i / w, x = i % w;
    int64_t arg = -1;
    for (int k = 0; k < 8; ++k) {
      const int64_t yy = y + DY8[k], xx = x + DX8[k];
      if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
      const int64_t j = yy * w + xx;
      if (F[j] == F[i] && !rm[j] && delta[j] == delta[i] - 1 &&
          (arg < 0 || j < arg))
        arg = j;
    }
    ptr[i] = arg;
  }
  /* follow arrows to a marker (memoised) */
  for (int64_t i = 0; i < n; ++i) basin[i] = F[i] ? -1 : 0;
  for (int64_t i = 0; i < n; ++i) {
    if (basin[i] >= 0) continue;
    int64_t j = i;
    while (basin[j] < 0 && !rm[j] && ptr[j] >= 0) j = ptr[j];
    int32_t b = 0; /* unreachable (no exit): cannot happen for rm-defined plateaus */
    if (basin[j] >= 0) b = basin[j];
    else if (rm[j]) b = (int32_t)(first[mlab[j]] + 1);
    j = i;
    while (basin[j] < 0) {
      basin[j] = b;
      if (rm[j] || ptr[j] < 0) break;
      j = ptr[j];
    }
  }
  /* separation: drop pixels with a higher-id foreground 8-neighbour */
  for (int64_t i = 0; i < n; ++i) {
    uint8_t keep = (uint8_t)(basin[i] > 0);
    if (keep) {
      const int64_t y = i / w, x = i % w;
      for (int k = 0; k < 8 && keep; ++k) {
        const int64_t yy = y + DY8[k], xx = x + DX8[k];
        if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
        if (basin[yy * w + xx] > basin[i]) keep = 0;
      }
    }
    sep[i] = keep;
  }
  if (planes) {
    if (planes->dist2) memcpy(planes->dist2, d2, sizeof(int32_t) * (size_t)n);
    if (planes->dq) memcpy(planes->dq, dq, sizeof(uint16_t) * (size_t)n);
    if (planes->fw) memcpy(planes->fw, F, sizeof(uint16_t) * (size_t)n);
    if (planes->rmax) memcpy(planes->rmax, rm, (size_t)n);
  }
  free(q.v);
  free(delta);
  free(ptr);
  free(first);
  free(mlab);
  free(rm);
  free(G);
  free(F);
  free(mk);
  free(dq);
  free(d2);
}

/* ---- f4: Canny edges ------------------------------------------------------------ */

static int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : v > hi ? hi : v; }

void orc_canny(const uint8_t* I, int64_t h, int64_t w, int32_t low, int32_t high,
               uint8_t* edges) {
  static const int K[5] = {1, 4, 6, 4, 1};
  const int64_t n = h * w;
  uint8_t* S = (uint8_t*)malloc((size_t)n + 1);
  int32_t* M = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* G = (int32_t*)malloc(sizeof(int32_t) * 2 * ((size_t)n + 1));
  uint8_t* C = (uint8_t*)calloc((size_t)n + 1, 1);
  for (int64_t y = 0; y < h; ++y)
    for (int64_t x = 0; x < w; ++x) {
      int32_t acc = 0;
      for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx)
          acc += K[dy + 2] * K[dx + 2] * I[clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)];
      S[y * w + x] = (uint8_t)((acc + 128) >> 8);
    }
  for (int64_t y = 0; y < h; ++y)
    for (int64_t x = 0; x < w; ++x) {
      const int64_t ym = clampi(y - 1, 0, h - 1), yp = clampi(y + 1, 0, h - 1);
      const int64_t xm = clampi(x - 1, 0, w - 1), xp = clampi(x + 1, 0, w - 1);
      const int32_t gx = (S[ym * w + xp] + 2 * S[y * w + xp] + S[yp * w + xp]) -
                         (S[ym * w + xm] + 2 * S[y * w + xm] + S[yp * w + xm]);
      const int32_t gy = (S[yp * w + xm] + 2 * S[yp * w + x] + S[yp * w + xp]) -
                         (S[ym * w + xm] + 2 * S[ym * w + x] + S[ym * w + xp]);
      G[2 * (y * w + x)] = gx;
      G[2 * (y * w + x) + 1] = gy;
      M[y * w + x] = gx * gx + gy * gy;
    }
  const int64_t lo2 = (int64_t)low * low, hi2 = (int64_t)high * high;
  for (int64_t y = 0; y < h; ++y)
    for (int64_t x = 0; x < w; ++x) {
      const int32_t gx = G[2 * (y * w + x)], gy = G[2 * (y * w + x) + 1];
      const int64_t ax = gx < 0 ? -gx : gx, ay = gy < 0 ? -gy : gy;
      const int64_t t22 = ax * 13573, ay15 = ay << 15;  /* tan(22.5) * 2^15 */
      int64_t ya, xa, yb, xb;
      if (ay15 < t22) { ya = y; xa = x - 1; yb = y; xb = x + 1; }
      else if (ay15 > t22 + (ax << 16)) { ya = y - 1; xa = x; yb = y + 1; xb = x; }
      else {
        const int64_t s = ((gx ^ gy) < 0) ? -1 : 1;
        ya = y - 1; xa = x - s; yb = y + 1; xb = x + s;
      }
      const int64_t m = M[y * w + x];
      const int64_t ma = (ya >= 0 && ya < h && xa >= 0 && xa < w) ? M[ya * w + xa] : 0;
      const int64_t mb = (yb >= 0 && yb < h && xb >= 0 && xb < w) ? M[yb * w + xb] : 0;
      if (m > ma && m >= mb) C[y * w + x] = m > hi2 ? 2 : (m > lo2 ? 1 : 0);
    }
  /* hysteresis: BFS from strong pixels through weak ones (8-connected) */
  memset(edges, 0, (size_t)n);
  int64_t* q = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  int64_t qh = 0, qt = 0;
  for (int64_t i = 0; i < n; ++i)
    if (C[i] == 2) { edges[i] = 1; q[qt++] = i; }
  while (qh < qt) {
    const int64_t i = q[qh++], y = i / w, x = i % w;
    for (int k = 0; k < 8; ++k) {
      const int64_t yy = y + DY8[k], xx = x + DX8[k];
      if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
      const int64_t j = yy * w + xx;
      if (C[j] && !edges[j]) { edges[j] = 1; q[qt++] = j; }
    }
  }
  free(q);
  free(S);
  free(M);
  free(G);
  free(C);
}

/* ---- f4: texture features ---------------------------------------------------- */

void orc_texture_row(const uint32_t hist[16], const uint32_t glcm[64], const int64_t mom[4],
                     uint32_t edge_px, float* out) {
  for (int k = 0; k < RTG_NUM_TEXTURE; ++k) out[k] = 0.f;
  int64_t nn = 0;
  for (int b = 0; b < 16; ++b) nn += hist[b];
  if (nn == 0) return;
  const double N = (double)nn;
  double hent = 0.0, hen = 0.0;
  for (int b = 0; b < 16; ++b) {
    if (!hist[b]) continue;
    const double p = (double)hist[b] / N;
    hent -= p * log2(p);
    hen += p * p;
  }
  const double mu = (double)mom[0] / N, e2 = (double)mom[1] / N;
  const double e3 = (double)mom[2] / N, e4 = (double)mom[3] / N;
  const double var = e2 - mu * mu;
  double skew = 0.0, kurt = 0.0;
  if (var > 0.0) {
    const double sd = sqrt(var);
    skew = (e3 - 3.0 * mu * e2 + 2.0 * mu * mu * mu) / (var * sd);
    kurt = (e4 - 4.0 * mu * e3 + 6.0 * mu * mu * e2 - 3.0 * mu * mu * mu * mu) / (var * var) - 3.0;
  }
  out[RTG_T_HIST_ENTROPY] = (float)hent;
  out[RTG_T_HIST_ENERGY] = (float)hen;
  out[RTG_T_SKEWNESS] = (float)skew;
  out[RTG_T_KURTOSIS] = (float)kurt;
  out[RTG_T_EDGE_PIXELS] = (float)edge_px;
  out[RTG_T_EDGE_DENSITY] = (float)((double)edge_px / N);
  int64_t tt = 0;
  for (int k = 0; k < 64; ++k) tt += glcm[k];
  if (tt == 0) return;
  const double T = (double)tt;
  double asm_ = 0.0, con = 0.0, hom = 0.0, ent = 0.0, mui = 0.0, dis = 0.0, mx = 0.0;
  for (int i = 0; i < 8; ++i) {
    for (int j = 0; j < 8; ++j) {
      const uint32_t c = glcm[i * 8 + j];
      if (!c) continue;
      const double P = (double)c / T;
      const int d = i - j;
      asm_ += P * P;
      con += (double)(d * d) * P;
      hom += P / (1.0 + (double)(d * d));
      ent -= P * log2(P);
      mui += (double)i * P;
      dis += (double)(d < 0 ? -d : d) * P;
      if (P > mx) mx = P;
    }
  }
  double vari = 0.0, sij = 0.0, shade = 0.0;
  for (int i = 0; i < 8; ++i) {
    for (int j = 0; j < 8; ++j) {
      const uint32_t c = glcm[i * 8 + j];
      if (!c) continue;
      const double P = (double)c / T;
      const double di = (double)i - mui;
      const double t = (double)(i + j) - 2.0 * mui;
      vari += di * di * P;
      sij += (double)(i * j) * P;
      shade += t * t * t * P;
    }
  }
  out[RTG_T_GLCM_ASM] = (float)asm_;
  out[RTG_T_GLCM_CONTRAST] = (float)con;
  out[RTG_T_GLCM_HOMOGENEITY] = (float)hom;
  out[RTG_T_GLCM_ENTROPY] = (float)ent;
  out[RTG_T_GLCM_CORRELATION] = (float)(vari > 0.0 ? (sij - mui * mui) / vari : 0.0);
  out[RTG_T_GLCM_DISSIMILARITY] = (float)dis;
  out[RTG_T_GLCM_MAX_PROB] = (float)mx;
  out[RTG_T_GLCM_CLUSTER_SHADE] = (float)shade;
}

void orc_texture(const int32_t* labels, const uint8_t* I, int64_t h, int64_t w, int32_t n,
                 float* out) {
  uint32_t* hist = (uint32_t*)calloc((size_t)n * 16 + 1, sizeof(uint32_t));
  uint32_t* glcm = (uint32_t*)calloc((size_t)n * 64 + 1, sizeof(uint32_t));
  int64_t* mom = (int64_t*)calloc((size_t)n * 4 + 1, sizeof(int64_t));
  uint32_t* edge = (uint32_t*)calloc((size_t)n + 1, sizeof(uint32_t));
  uint8_t* E = (uint8_t*)malloc((size_t)(h * w) + 1);
  orc_canny(I, h, w, RTG_CANNY_LOW, RTG_CANNY_HIGH, E);
  /* forward offsets: right, down, down-right, down-left */
  static const int ODY[4] = {0, 1, 1, 1}, ODX[4] = {1, 0, 1, -1};
  for (int64_t y = 0; y < h; ++y) {
    for (int64_t x = 0; x < w; ++x) {
      const int32_t l = labels[y * w + x];
      if (l <= 0 || l > n) continue;
      const int64_t k = l - 1;
      const int64_t v = I[y * w + x];
      hist[k * 16 + (v >> 4)]++;
      edge[k] += E[y * w + x];
      mom[k * 4 + 0] += v;
      mom[k * 4 + 1] += v * v;
      mom[k * 4 + 2] += v * v * v;
      mom[k * 4 + 3] += v * v * v * v;
      const int q = (int)(v >> 5);
      for (int o = 0; o < 4; ++o) {
        const int64_t yy = y + ODY[o], xx = x + ODX[o];
        if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
        if (labels[yy * w + xx] != l) continue;
        const int q2 = I[yy * w + xx] >> 5;
        glcm[k * 64 + q * 8 + q2]++;
        glcm[k * 64 + q2 * 8 + q]++;
      }
    }
  }
  for (int32_t k = 0; k < n; ++k)
    orc_texture_row(hist + (size_t)k * 16, glcm + (size_t)k * 64, mom + (size_t)k * 4, edge[k],
                    out + (size_t)k * RTG_NUM_TEXTURE);
  free(edge);
  free(E);
  free(hist);
  free(glcm);
  free(mom);
}

/* ---- o9: features ----------------------------------------------------------- */

typedef struct {
  int64_t area, sy, sx, syy, sxx, sxy, si, sii, sg, sgg, perim;
  int32_t mini, maxi, y0, x0, y1, x1;
} orc_acc;

void orc_features(const int32_t* labels, const uint8_t* I, int64_t h,
                  int64_t w, int32_t n, float* out) {
  orc_acc* a = (orc_acc*)calloc((size_t)n + 1, sizeof(orc_acc));
  for (int32_t k = 0; k <= n; ++k) {
    a[k].mini = 255;
    a[k].maxi = 0;
    a[k].y0 = a[k].x0 = INT32_MAX;
    a[k].y1 = a[k].x1 = -1;
  }
  for (int64_t y = 0; y < h; ++y) {
    for (int64_t x = 0; x < w; ++x) {
      const int32_t l = labels[y * w + x];
      if (l <= 0 || l > n) continue;
      orc_acc* c = &a[l];
      const int64_t v = I[y * w + x];
      /* Sobel with replicated border */
      const int64_t ym = y > 0 ? y - 1 : 0, yp = y + 1 < h ? y + 1 : h - 1;
      const int64_t xm = x > 0 ? x - 1 : 0, xp = x + 1 < w ? x + 1 : w - 1;
#define P(yy, xx) ((int64_t)I[(yy) * w + (xx)])
      const int64_t gx = (P(ym, xp) + 2 * P(y, xp) + P(yp, xp)) -
                         (P(ym, xm) + 2 * P(y, xm) + P(yp, xm));
      const int64_t gy = (P(yp, xm) + 2 * P(yp, x) + P(yp, xp)) -
                         (P(ym, xm) + 2 * P(ym, x) + P(ym, xp));
#undef P
      const int64_t gq = orc_isqrt((uint64_t)(16 * (gx * gx + gy * gy)));
      int perim = 0;
      perim += (y == 0 || labels[(y - 1) * w + x] != l);
      perim += (y == h - 1 || labels[(y + 1) * w + x] != l);
      perim += (x == 0 || labels[y * w + x - 1] != l);
      perim += (x == w - 1 || labels[y * w + x + 1] != l);
      c->area += 1;
      c->sy += y;
      c->sx += x;
      c->syy += y * y;
      c->sxx += x * x;
      c->sxy += x * y;
      c->si += v;
      c->sii += v * v;
      c->sg += gq;
      c->sgg += gq * gq;
      c->perim += perim;
      if (v < c->mini) c->mini = (int32_t)v;
      if (v > c->maxi) c->maxi = (int32_t)v;
      if (y < c->y0) c->y0 = (int32_t)y;
      if (y > c->y1) c->y1 = (int32_t)y;
      if (x < c->x0) c->x0 = (int32_t)x;
      if (x > c->x1) c->x1 = (int32_t)x;
    }
  }
  for (int32_t l = 1; l <= n; ++l) {
    const orc_acc* c = &a[l];
    float* f = out + (size_t)(l - 1) * RTG_NUM_FEATURES;
    if (c->area == 0) {
      memset(f, 0, sizeof(float) * RTG_NUM_FEATURES);
      continue;
    }
    const double A = (double)c->area;
    const double cy = (double)c->sy / A, cx = (double)c->sx / A;
    const double mi = (double)c->si / A;
    const double vi = (double)c->sii / A - mi * mi;
    const double mg = (double)c->sg / (4.0 * A);
    const double vg = (double)c->sgg / (16.0 * A) - mg * mg;
    const double mxx = (double)c->sxx / A - cx * cx + 1.0 / 12.0;
    const double myy = (double)c->syy / A - cy * cy + 1.0 / 12.0;
    const double mxy = (double)c->sxy / A - cx * cy;
    const double half = 0.5 * (mxx + myy);
    const double dd = 0.5 * (mxx - myy);
    const double root = sqrt(dd * dd + mxy * mxy);
    const double l1 = half + root;
    double l2 = half - root;
    if (l2 < 0.0) l2 = 0.0;
    const double P = (double)c->perim;
    f[RTG_F_AREA] = (float)A;
    f[RTG_F_PERIMETER] = (float)P;
    f[RTG_F_BBOX_Y0] = (float)c->y0;
    f[RTG_F_BBOX_X0] = (float)c->x0;
    f[RTG_F_BBOX_Y1] = (float)c->y1;
    f[RTG_F_BBOX_X1] = (float)c->x1;
    f[RTG_F_CENTROID_Y] = (float)cy;
    f[RTG_F_CENTROID_X] = (float)cx;
    f[RTG_F_MEAN_I] = (float)mi;
    f[RTG_F_STD_I] = (float)sqrt(vi > 0.0 ? vi : 0.0);
    f[RTG_F_MIN_I] = (float)c->mini;
    f[RTG_F_MAX_I] = (float)c->maxi;
    f[RTG_F_MEAN_GRAD] = (float)mg;
    f[RTG_F_STD_GRAD] = (float)sqrt(vg > 0.0 ? vg : 0.0);
    f[RTG_F_MAJOR_AXIS] = (float)(4.0 * sqrt(l1));
    f[RTG_F_MINOR_AXIS] = (float)(4.0 * sqrt(l2));
    f[RTG_F_ECCENTRICITY] = (float)(l1 > 0.0 ? sqrt(1.0 - l2 / l1) : 0.0);
    f[RTG_F_ORIENTATION] = (float)(0.5 * atan2(2.0 * mxy, mxx - myy));
    f[RTG_F_CIRCULARITY] = (float)(4.0 * 3.14159265358979323846 * A / (P * P));
    f[RTG_F_EXTENT] =
        (float)(A / ((double)(c->y1 - c->y0 + 1) * (double)(c->x1 - c->x0 + 1)));
  }
  free(a);
}

/* ---- the whole stage -------------------------------------------------------- */

int32_t orc_process_tile(const uint8_t* rgb, int64_t h, int64_t w,
                         int64_t pitch, const rtg_params* p, uint8_t* mask,
                         int32_t* labels, float* features, int32_t max_rows,
                         orc_planes* planes) {
  const int64_t n = h * w;
  uint8_t* hema = (uint8_t*)malloc((size_t)n);
  uint8_t* mk = (uint8_t*)malloc((size_t)n);
  uint8_t* tis = (uint8_t*)malloc((size_t)n);
  uint8_t* rec = (uint8_t*)malloc((size_t)n);
  uint8_t* m1 = (uint8_t*)malloc((size_t)n);
  uint8_t* m2 = (uint8_t*)malloc((size_t)n);
  uint8_t* m3 = (uint8_t*)malloc((size_t)n);
  uint8_t* m4 = (uint8_t*)malloc((size_t)n);
  int32_t* basin = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* lab = labels ? labels : (int32_t*)malloc(sizeof(int32_t) * (size_t)n);

  orc_colordeconv(rgb, h, w, pitch, p, hema, mk, tis);
  orc_recon_u8(mk, hema, h, w, p->recon_conn, rec);
  for (int64_t i = 0; i < n; ++i) m1[i] = (uint8_t)(rec[i] >= p->nuc_thresh && tis[i]);
  orc_fill_holes(m1, h, w, m2);
  orc_area_threshold(m2, h, w, 8, p->min_area, p->max_area, m3);
  orc_watershed(m3, h, w, p->ws_h, m4, basin, planes);
  const int32_t nobj = orc_bwlabel(m4, h, w, 8, lab);
  if (features) {
    /* rows of RTG_NUM_FEATURES shape / intensity columns, followed by the
     * RTG_NUM_TEXTURE texture columns when p->texture is set */
    const int cols = RTG_NUM_FEATURES + (p->texture ? RTG_NUM_TEXTURE : 0);
    float* tmp = (float*)malloc(sizeof(float) * RTG_NUM_FEATURES * ((size_t)nobj + 1));
    float* tex = p->texture ? (float*)malloc(sizeof(float) * RTG_NUM_TEXTURE * ((size_t)nobj + 1))
                            : NULL;
    orc_features(lab, hema, h, w, nobj, tmp);
    if (tex) orc_texture(lab, hema, h, w, nobj, tex);
    const int32_t rows = nobj < max_rows ? nobj : max_rows;
    for (int32_t k = 0; k < rows; ++k) {
      memcpy(features + (size_t)k * cols, tmp + (size_t)k * RTG_NUM_FEATURES,
             sizeof(float) * RTG_NUM_FEATURES);
      if (tex)
        memcpy(features + (size_t)k * cols + RTG_NUM_FEATURES, tex + (size_t)k * RTG_NUM_TEXTURE,
               sizeof(float) * RTG_NUM_TEXTURE);
    }
    free(tmp);
    free(tex);
  }
  if (mask) memcpy(mask, m4, (size_t)n);
  if (planes) {
    if (planes->hema) memcpy(planes->hema, hema, (size_t)n);
    if (planes->marker) memcpy(planes->marker, mk, (size_t)n);
    if (planes->tissue) memcpy(planes->tissue, tis, (size_t)n);
    if (planes->recon) memcpy(planes->recon, rec, (size_t)n);
    if (planes->cand) memcpy(planes->cand, m1, (size_t)n);
    if (planes->filled) memcpy(planes->filled, m2, (size_t)n);
    if (planes->area) memcpy(planes->area, m3, (size_t)n);
    if (planes->basin) memcpy(planes->basin, basin, sizeof(int32_t) * (size_t)n);
    if (planes->sep) memcpy(planes->sep, m4, (size_t)n);
  }
  if (!labels) free(lab);
  free(basin);
  free(m4);
  free(m3);
  free(m2);
  free(m1);
  free(rec);
  free(tis);
  free(mk);
  free(hema);
  return nobj;
}
