// Wide keys (KeyGeom::wide): datasets whose packed (i,j,k,level) key needs
// more than 64 bits -- fine cells spread over most of the int32 range, which
// the reference accepts (proj/include/amriso/core.hpp:82-88,
// proj/src/locator.cpp:26-50; its boundary test test_locator.cpp:137-153).
// The key is the 128-bit integer with the 64-bit layout's fields (pack128),
// stored as (lo, hi) words, so its order is still the reference's order and
// a sorted position is still a CellId.  Such key spaces are sparse by
// construction, so lookups go through an exact-key hash table, and snap is
// the reference's probe sequence itself (locator.cpp:107-134): the hint
// level, then the present levels finest first, one exact lookup each.
#pragma once

#include "common.cuh"

namespace amrx {

struct WideCtx {
  const ulonglong2 *keys;  // sorted (lo, hi)
  const ulonglong4 *tab;   // entry {lo, hi, id + 1 (0 = empty), 0}
  uint64_t mask;           // table entries - 1
  uint64_t n;
  int64_t id_base;         // always 0 (no distributed wide indexes)
};

__device__ __forceinline__ u128 wide_key(const ulonglong2 *keys, uint64_t i)
{
  const ulonglong2 k = __ldg(keys + i);
  return u128(k.x) | (u128(k.y) << 64);
}

__host__ __device__ inline uint64_t wide_home(u128 key, uint64_t mask)
{
  const uint64_t lo = uint64_t(key), hi = uint64_t(key >> 64);
  uint32_t x = uint32_t(lo) * 0x9E3779B1u ^ uint32_t(lo >> 32) * 0x85EBCA77u ^
               uint32_t(hi) * 0xC2B2AE3Du ^ uint32_t(hi >> 32) * 0x27D4EB2Fu;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  return uint64_t(x) & mask;
}

/// the first position holding the exact key, or -1 (find_exact's
/// lower_bound + equality, locator.cpp:94-101)
__device__ __forceinline__ int64_t wide_find(const WideCtx &w, u128 key)
{
  uint64_t h = wide_home(key, w.mask);
  for (;;) {
    const ulonglong4 e = ldg_bucket(w.tab + h);
    if (e.z == 0) return -1;
    if (e.x == uint64_t(key) && e.y == uint64_t(key >> 64)) return int64_t(e.z - 1);
    h = (h + 1) & w.mask;
  }
}

/// snap_on_level (locator.cpp:107-119): mask to the level, range guard, exact lookup
__device__ __forceinline__ int64_t wide_on_level(const WideCtx &w, const KeyGeom &g, int64_t px,
                                                 int64_t py, int64_t pz, int32_t level)
{
  if (!level_present(g, level)) return -1;
  const int64_t ax = anchor_mask(px, level), ay = anchor_mask(py, level),
                az = anchor_mask(pz, level);
  if (ax < g.mn[0] || ax > g.mx[0] || ay < g.mn[1] || ay > g.mx[1] || az < g.mn[2] ||
      az > g.mx[2])
    return -1;
  return wide_find(w, pack128(g, ax, ay, az, level));
}

/// snap (locator.cpp:122-134): the hint level if it is a level, then the
/// present levels finest first, skipping the hint; *lev = the hit's level
__device__ inline int64_t wide_snap(const WideCtx &w, const KeyGeom &g, int64_t px, int64_t py,
                                    int64_t pz, int32_t hint, int &lev)
{
  if (hint >= 0 && hint <= kMaxLevel) {
    const int64_t id = wide_on_level(w, g, px, py, pz, hint);
    if (id >= 0) {
      lev = hint;
      return id;
    }
  }
  for (int t = 0; t < g.nlevels; t++) {
    const int L = g.levels[t];
    if (L == hint) continue;
    const int64_t id = wide_on_level(w, g, px, py, pz, L);
    if (id >= 0) {
      lev = L;
      return id;
    }
  }
  return -1;
}

/*! try_build_dual (dual.cpp:41-72) for candidate delta of cell `self`:
    corners d = 0..7 at base + w bits(d), snapped with the owner level as
    hint; the first failing corner decides: 1 missing, 2 finer, 3 lower key;
    0 = accepted with ids/levels filled */
__device__ inline uint32_t wide_try(const WideCtx &w, const KeyGeom &g, const Cell &c,
                                    uint64_t self, int delta, uint32_t (&ids)[8],
                                    uint8_t (&lev)[8])
{
  const int64_t cw = int64_t(1) << c.level;
  const int64_t bx = c.i - ((delta & 1) ? 0 : cw);
  const int64_t by = c.j - ((delta & 2) ? 0 : cw);
  const int64_t bz = c.k - ((delta & 4) ? 0 : cw);
  for (int d = 0; d < 8; d++) {
    int l = 0;
    const int64_t hit = wide_snap(w, g, bx + ((d & 1) ? cw : 0), by + ((d & 2) ? cw : 0),
                                  bz + ((d & 4) ? cw : 0), c.level, l);
    if (hit < 0) return 1;
    if (l < c.level) return 2;
    if (l == c.level && uint64_t(hit) < self) return 3;
    ids[d] = uint32_t(hit);
    lev[d] = uint8_t(l);
  }
  return 0;
}

}  // namespace amrx
