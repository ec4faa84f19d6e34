/* TEST ORACLE -- plain-C restatement of the reference's hot path.
 *
 * Test infrastructure only (see amrx_oracle.h).  Pinned against the
 * reference library compiled in place (oracle/_ref) and against the golden
 * vectors under tests/golden/ by tests/test_oracle.py.
 *
 * Compiled with -ffp-contract=off like the reference (proj/CMakeLists.txt:
 * 11-12) so the FP64 interpolation below rounds exactly as contour.cpp's. */
#include "amrx_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mc_tables_oracle.inc"

#define MAX_LEVEL 30 /* proj/include/amriso/core.hpp:28 */

struct orc_index {
  uint64_t n;
  int32_t *cells; /* 4 per cell: i j k level, sorted (i,j,k,level) */
  double *scalars;
  int32_t levels[MAX_LEVEL + 1]; /* present levels, finest first */
  int nlevels;
  int32_t max_level;
  int64_t lo[3], hi[3];
};

static _Thread_local char g_err[256];

const char *orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------ core.hpp */
/* anchor_mask: x & ~(2^l - 1), rounds toward -inf (core.hpp:98-103) */
static int64_t anchor_mask(int64_t x, int32_t level)
{
  return x & ~((((int64_t)1) << level) - 1);
}

/* lexicographic (i,j,k,level) -- the defaulted <=> of CellCoord
 * (core.hpp:82-88) */
static int cmp_cell(const int32_t *a, const int32_t *b)
{
  for (int c = 0; c < 4; c++) {
    if (a[c] < b[c]) return -1;
    if (a[c] > b[c]) return 1;
  }
  return 0;
}

/* ------------------------------------------------------- build_index */
typedef struct {
  int32_t c[4];
  uint32_t idx;
} sort_rec;

/* sort by key, ties by input index (locator.cpp:52-60) */
static int cmp_rec(const void *pa, const void *pb)
{
  const sort_rec *a = (const sort_rec *)pa, *b = (const sort_rec *)pb;
  const int o = cmp_cell(a->c, b->c);
  if (o) return o;
  return (a->idx > b->idx) - (a->idx < b->idx);
}

orc_index *orc_build_index(const int32_t *cells4, const double *scalars,
                           uint64_t n, uint64_t n_scalars)
{
  /* locator.cpp:29-50 */
  if (n == 0) {
    snprintf(g_err, sizeof g_err, "dataset is empty");
    return NULL;
  }
  if (n != n_scalars) {
    snprintf(g_err, sizeof g_err,
             "cell count %llu does not match scalar count %llu",
             (unsigned long long)n, (unsigned long long)n_scalars);
    return NULL;
  }
  if (n > 0xffffffffull) {
    snprintf(g_err, sizeof g_err, "dataset too large for 32-bit cell ids");
    return NULL;
  }
  for (uint64_t r = 0; r < n; r++) {
    const int32_t *c = cells4 + 4 * r;
    if (c[3] < 0 || c[3] > MAX_LEVEL) {
      snprintf(g_err, sizeof g_err, "record %llu: level %d out of range [0,%d]",
               (unsigned long long)r, c[3], MAX_LEVEL);
      return NULL;
    }
    if (anchor_mask(c[0], c[3]) != c[0] || anchor_mask(c[1], c[3]) != c[1] ||
        anchor_mask(c[2], c[3]) != c[2]) {
      snprintf(g_err, sizeof g_err,
               "record %llu: anchor (%d %d %d) is not a multiple of the "
               "level-%d cell width",
               (unsigned long long)r, c[0], c[1], c[2], c[3]);
      return NULL;
    }
  }

  orc_index *idx = (orc_index *)calloc(1, sizeof(orc_index));
  idx->n = n;
  idx->cells = (int32_t *)malloc(n * 16);
  idx->scalars = (double *)malloc(n * 8);

  /* already in (key, input position) order: the stable sort is the
   * identity, skip it (lets tests hold 10^8..10^9-cell indices) */
  int sorted = 1;
  for (uint64_t r = 1; r < n && sorted; r++)
    if (cmp_cell(cells4 + 4 * (r - 1), cells4 + 4 * r) > 0) sorted = 0;
  if (sorted) {
    memcpy(idx->cells, cells4, n * 16);
    memcpy(idx->scalars, scalars, n * 8);
  } else {
    sort_rec *recs = (sort_rec *)malloc(n * sizeof(sort_rec));
    for (uint64_t r = 0; r < n; r++) {
      memcpy(recs[r].c, cells4 + 4 * r, 16);
      recs[r].idx = (uint32_t)r;
    }
    qsort(recs, n, sizeof(sort_rec), cmp_rec);
    for (uint64_t r = 0; r < n; r++) {
      memcpy(idx->cells + 4 * r, recs[r].c, 16);
      idx->scalars[r] = scalars[recs[r].idx];
    }
    free(recs);
  }

  /* bounds, max level, distinct levels finest first (locator.cpp:70-89) */
  int present[MAX_LEVEL + 1] = {0};
  for (int a = 0; a < 3; a++) {
    idx->lo[a] = INT64_MAX;
    idx->hi[a] = INT64_MIN;
  }
  idx->max_level = 0;
  for (uint64_t r = 0; r < n; r++) {
    const int32_t *c = idx->cells + 4 * r;
    const int64_t w = ((int64_t)1) << c[3];
    if (c[3] > idx->max_level) idx->max_level = c[3];
    present[c[3]] = 1;
    for (int a = 0; a < 3; a++) {
      if (c[a] < idx->lo[a]) idx->lo[a] = c[a];
      if (c[a] + w > idx->hi[a]) idx->hi[a] = c[a] + w;
    }
  }
  for (int l = 0; l <= idx->max_level; l++)
    if (present[l]) idx->levels[idx->nlevels++] = l;
  return idx;
}

void orc_index_free(orc_index *idx)
{
  if (!idx) return;
  free(idx->cells);
  free(idx->scalars);
  free(idx);
}

uint64_t orc_index_size(const orc_index *idx) { return idx->n; }

void orc_index_get(const orc_index *idx, int32_t *cells4, double *scalars)
{
  memcpy(cells4, idx->cells, idx->n * 16);
  memcpy(scalars, idx->scalars, idx->n * 8);
}

int orc_index_levels(const orc_index *idx, int32_t *out)
{
  memcpy(out, idx->levels, sizeof(int32_t) * idx->nlevels);
  return idx->nlevels;
}

void orc_index_bounds(const orc_index *idx, int64_t *out7)
{
  for (int a = 0; a < 3; a++) {
    out7[a] = idx->lo[a];
    out7[3 + a] = idx->hi[a];
  }
  out7[6] = idx->max_level;
}

/* -------------------------------------------------- find_exact / snap */
/* std::lower_bound + equality (locator.cpp:94-101) */
int64_t orc_find_exact(const orc_index *idx, const int32_t *c4)
{
  uint64_t lo = 0, count = idx->n;
  while (count > 0) {
    const uint64_t step = count / 2, mid = lo + step;
    if (cmp_cell(idx->cells + 4 * mid, c4) < 0) {
      lo = mid + 1;
      count -= step + 1;
    } else {
      count = step;
    }
  }
  if (lo == idx->n || cmp_cell(idx->cells + 4 * lo, c4) != 0) return -1;
  return (int64_t)lo;
}

/* snap_on_level: mask, int32 range guard, exact lookup (locator.cpp:107-119) */
static int64_t snap_on_level(const orc_index *idx, const int64_t *p,
                             int32_t level)
{
  int32_t key[4];
  for (int a = 0; a < 3; a++) {
    const int64_t m = anchor_mask(p[a], level);
    if (m < INT32_MIN || m > INT32_MAX) return -1;
    key[a] = (int32_t)m;
  }
  key[3] = level;
  return orc_find_exact(idx, key);
}

/* hint level first, then present levels finest->coarsest skipping the hint
 * (locator.cpp:122-134) */
int64_t orc_snap(const orc_index *idx, const int64_t *p3, int32_t hint)
{
  if (hint >= 0 && hint <= MAX_LEVEL) {
    const int64_t hit = snap_on_level(idx, p3, hint);
    if (hit >= 0) return hit;
  }
  for (int n = 0; n < idx->nlevels; n++) {
    if (idx->levels[n] == hint) continue;
    const int64_t hit = snap_on_level(idx, p3, idx->levels[n]);
    if (hit >= 0) return hit;
  }
  return -1;
}

/* ------------------------------------------------------ try_build_dual */
/* corners d=0..7 (dx fastest) snapped with hint = owner level; rules
 * #1 missing, #2 finer, #3 same level with lower id; first failing corner
 * decides (dual.cpp:41-72) */
int orc_try_build_dual(const orc_index *idx, const int64_t *base3,
                       int32_t level, uint32_t self, uint32_t *corners8)
{
  const int64_t w = ((int64_t)1) << level;
  for (int d = 0; d < 8; d++) {
    const int64_t corner[3] = {base3[0] + ((d & 1) ? w : 0),
                               base3[1] + ((d & 2) ? w : 0),
                               base3[2] + ((d & 4) ? w : 0)};
    const int64_t hit = orc_snap(idx, corner, level);
    if (hit < 0) return ORC_MISSING;
    const int32_t hit_level = idx->cells[4 * hit + 3];
    if (hit_level < level) return ORC_FINER;
    if (hit_level == level && (uint32_t)hit < self) return ORC_LOWER_KEY;
    if (corners8) corners8[d] = (uint32_t)hit;
  }
  return ORC_ACCEPTED;
}

/* base(delta) = anchor - w*(1-bit) per axis, bit0 = x (dual.hpp:61-67) */
static void dual_base_of(const int32_t *c, int delta, int64_t *base)
{
  const int64_t w = ((int64_t)1) << c[3];
  base[0] = c[0] - ((delta & 1) ? 0 : w);
  base[1] = c[1] - ((delta & 2) ? 0 : w);
  base[2] = c[2] - ((delta & 4) ? 0 : w);
}

/* --------------------------------------------------------- contour_hex */
/* mc::to_table_case (mc_tables.cpp:324-330) */
static int to_table_case(int slot_mask)
{
  int row = 0;
  for (int c = 0; c < 8; c++)
    if (slot_mask & (1 << ORACLE_TABLE_CORNER[c])) row |= 1 << c;
  return row;
}

/* lower CellId first, t=(iso-a)/(b-a), p=a+t*(b-a) (contour.cpp:30-50) */
static void interpolate_edge(uint32_t a_cell, uint32_t b_cell,
                             const double *a_pos, const double *b_pos,
                             double a_val, double b_val, double iso,
                             double *out)
{
  if (b_cell < a_cell) {
    interpolate_edge(b_cell, a_cell, b_pos, a_pos, b_val, a_val, iso, out);
    return;
  }
  const double t = (iso - a_val) / (b_val - a_val);
  for (int a = 0; a < 3; a++) out[a] = a_pos[a] + t * (b_pos[a] - a_pos[a]);
}

static int same3(const double *a, const double *b)
{
  return a[0] == b[0] && a[1] == b[1] && a[2] == b[2];
}

int orc_contour_hex(const uint32_t *cells8, const double *pos24,
                    const double *value8, double iso, double *out45)
{
  int mask = 0; /* strict value > iso (contour.cpp:22-28) */
  for (int d = 0; d < 8; d++)
    if (value8[d] > iso) mask |= 1 << d;
  const signed char *entry = ORACLE_TRI[to_table_case(mask)];
  if (entry[0] < 0) return 0;

  double on_edge[12][3];
  int have[12] = {0};
  for (int n = 0; n < 16 && entry[n] >= 0; n++) {
    const int e = entry[n];
    if (have[e]) continue;
    const int u = ORACLE_EDGE_CORNER[e][0], v = ORACLE_EDGE_CORNER[e][1];
    if (cells8[u] == cells8[v]) {
      snprintf(g_err, sizeof g_err,
               "contour_hex: case table selected a collapsed edge");
      return -1;
    }
    if ((value8[u] > iso) == (value8[v] > iso)) {
      snprintf(g_err, sizeof g_err,
               "interpolate_edge: no crossing on this edge");
      return -1;
    }
    interpolate_edge(cells8[u], cells8[v], pos24 + 3 * u, pos24 + 3 * v,
                     value8[u], value8[v], iso, on_edge[e]);
    have[e] = 1;
  }
  int count = 0;
  for (int n = 0; n < 16 && entry[n] >= 0; n += 3) {
    const double *p0 = on_edge[entry[n]], *p1 = on_edge[entry[n + 1]],
                 *p2 = on_edge[entry[n + 2]];
    if (same3(p0, p1) || same3(p1, p2) || same3(p0, p2)) continue;
    if (out45) {
      memcpy(out45 + 9 * count + 0, p0, 24);
      memcpy(out45 + 9 * count + 3, p1, 24);
      memcpy(out45 + 9 * count + 6, p2, 24);
    }
    count++;
  }
  return count;
}

/* make_hex_input: centre = anchor + w/2 in double (contour.cpp:89-99,
 * core.hpp:113-118) */
static void hex_input(const orc_index *idx, const uint32_t *corners8,
                      double *pos24, double *value8)
{
  for (int d = 0; d < 8; d++) {
    const int32_t *c = idx->cells + 4 * (uint64_t)corners8[d];
    const double half = 0.5 * (double)(((int64_t)1) << c[3]);
    pos24[3 * d + 0] = (double)c[0] + half;
    pos24[3 * d + 1] = (double)c[1] + half;
    pos24[3 * d + 2] = (double)c[2] + half;
    value8[d] = idx->scalars[corners8[d]];
  }
}

/* ----------------------------------------------------------- pipeline */
/* task t -> cell t>>3, delta t&7, candidate order (pipeline.cpp:40-57) */
uint64_t orc_extract_dual(const orc_index *idx, uint32_t *corners8,
                          uint32_t *owner, int64_t *base3, int32_t *level,
                          uint64_t cap, uint64_t *counters4)
{
  return orc_extract_dual_range(idx, 0, idx->n, corners8, owner, base3, level,
                                cap, counters4);
}

uint64_t orc_extract_dual_range(const orc_index *idx, uint64_t cell_begin,
                                uint64_t cell_end, uint32_t *corners8,
                                uint32_t *owner, int64_t *base3, int32_t *level,
                                uint64_t cap, uint64_t *counters4)
{
  uint64_t count = 0, cnt[4] = {0};
  for (uint64_t cell = cell_begin; cell < cell_end && cell < idx->n; cell++) {
    const int32_t *c = idx->cells + 4 * cell;
    for (int delta = 0; delta < 8; delta++) {
      int64_t base[3];
      uint32_t corners[8];
      dual_base_of(c, delta, base);
      const int r = orc_try_build_dual(idx, base, c[3], (uint32_t)cell, corners);
      cnt[r]++;
      if (r != ORC_ACCEPTED) continue;
      if (count < cap) {
        if (corners8) memcpy(corners8 + 8 * count, corners, 32);
        if (owner) owner[count] = (uint32_t)cell;
        if (base3) memcpy(base3 + 3 * count, base, 24);
        if (level) level[count] = c[3];
      }
      count++;
    }
  }
  if (counters4) memcpy(counters4, cnt, sizeof cnt);
  return count;
}

uint64_t orc_extract_iso_range(const orc_index *idx, double iso,
                               uint64_t cell_begin, uint64_t cell_end,
                               double *xyz9, uint64_t cap,
                               uint64_t *counters4)
{
  uint64_t count = 0, cnt[4] = {0};
  for (uint64_t cell = cell_begin; cell < cell_end && cell < idx->n; cell++) {
    const int32_t *c = idx->cells + 4 * cell;
    for (int delta = 0; delta < 8; delta++) {
      int64_t base[3];
      uint32_t corners[8];
      dual_base_of(c, delta, base);
      const int r = orc_try_build_dual(idx, base, c[3], (uint32_t)cell, corners);
      cnt[r]++;
      if (r != ORC_ACCEPTED) continue;
      double pos[24], val[8], tris[45];
      hex_input(idx, corners, pos, val);
      const int k = orc_contour_hex(corners, pos, val, iso, tris);
      if (k < 0) return UINT64_MAX;
      for (int t = 0; t < k; t++, count++)
        if (count < cap && xyz9) memcpy(xyz9 + 9 * count, tris + 9 * t, 72);
    }
  }
  if (counters4) memcpy(counters4, cnt, sizeof cnt);
  return count;
}

uint64_t orc_extract_iso(const orc_index *idx, double iso, double *xyz9,
                         uint64_t cap, uint64_t *counters4)
{
  return orc_extract_iso_range(idx, iso, 0, idx->n, xyz9, cap, counters4);
}

/* --------------------------------------------------------------- weld */
typedef struct {
  double p[3];
  uint64_t tag;
} tagged;

/* (x,y,z,tag) order (weld.cpp:44-51) */
static int cmp_tagged(const void *pa, const void *pb)
{
  const tagged *a = (const tagged *)pa, *b = (const tagged *)pb;
  for (int c = 0; c < 3; c++)
    if (a->p[c] != b->p[c]) return a->p[c] < b->p[c] ? -1 : 1;
  return (a->tag > b->tag) - (a->tag < b->tag);
}

uint64_t orc_weld(const double *xyz9, uint64_t n_tris, double *verts3,
                  uint32_t *tris3)
{
  if (n_tris == 0) return 0;
  tagged *t = (tagged *)malloc(3 * n_tris * sizeof(tagged));
  for (uint64_t n = 0; n < 3 * n_tris; n++) {
    memcpy(t[n].p, xyz9 + 3 * n, 24);
    t[n].tag = n;
  }
  qsort(t, 3 * n_tris, sizeof(tagged), cmp_tagged);
  uint64_t nv = 0;
  for (uint64_t n = 0; n < 3 * n_tris; n++) {
    if (n == 0 || !same3(t[n].p, t[n - 1].p)) {
      if (verts3) memcpy(verts3 + 3 * nv, t[n].p, 24);
      nv++;
    }
    if (tris3) tris3[t[n].tag] = (uint32_t)(nv - 1);
  }
  free(t);
  return nv;
}
