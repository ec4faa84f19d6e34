// Device-side building blocks shared by the amrx kernels (sm_100a).
//
// Key geometry: a cell (i,j,k,level) packs into one u64 whose integer order
// IS the reference's CellCoord order -- lexicographic (i,j,k,level), the
// defaulted operator<=> of proj/include/amriso/core.hpp:82-88.  Per axis the
// anchor is biased by the dataset minimum and shifted right by the finest
// level present (every anchor is a multiple of 2^finest, core.hpp:98-110), and
// the level field is level-finest.  Field widths come from the data, so a
// sorted position is a CellId exactly as in locator.hpp:25-33.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace amrx {

constexpr int kMaxLevel = 30;  // core.hpp:28

// Checked builds (make CHECK=1 TAG=chk; compute-sanitizer is closed on the
// GPU pool): a violated bound sets bit `code` of this translation unit's
// check word and the access is skipped; the C ABI reads every word after
// each call and fails with AMRX_ERR_INTERNAL.  Free in normal builds.
#ifndef AMRX_CHECKED
#define AMRX_CHECKED 0
#endif
#if AMRX_CHECKED
static __device__ unsigned int g_amrx_check;
#define AMRX_BOUND(cond, code) ((cond) || (atomicOr(&g_amrx_check, 1u << (code)), false))
#else
#define AMRX_BOUND(cond, code) true
#endif
enum CheckCode : int {
  kChkKey = 0,     // a sorted-key load past n + padding
  kChkRecord = 1,  // a dense record outside the built range
  kChkHash = 2,    // a hash table bucket outside the table
  kChkStage = 3,   // a staging read/write outside its arena
  kChkSort = 4,    // a radix scatter outside [0, n)
  kChkPerm = 5,    // a permutation entry outside [0, n)
  kChkSmem = 6,    // a stencil point index outside 0..26
  kChkJob = 7,     // a marching-cubes job outside the job buffer
};

/// this translation unit's check word, cleared (host; 0 in normal builds)
static inline unsigned int take_check_word()
{
#if AMRX_CHECKED
  unsigned int w = 0, z = 0;
  cudaMemcpyFromSymbol(&w, g_amrx_check, sizeof w);
  cudaMemcpyToSymbol(g_amrx_check, &z, sizeof z);
  return w;
#else
  return 0;
#endif
}
constexpr int kWin = 128;      // keys per warp search window (1 KB of smem)
constexpr int kKeyPad = 256;   // u64 sentinel padding after the key array
constexpr uint32_t kFull = 0xffffffffu;

struct KeyGeom {
  int64_t mn[3];        // min anchor per axis
  int64_t mx[3];        // max anchor per axis
  int32_t shift;        // finest level present
  int32_t bits[3];      // field width per axis
  int32_t lbits;        // width of the level field
  int32_t total;        // key bits in use
  int32_t sh[3];        // left shift of the x/y/z fields
  uint64_t umax[3];     // largest field value per axis ((mx - mn) >> shift)
  int32_t dir_bits;     // directory has 2^dir_bits + 1 entries
  int32_t dir_shift;    // bucket = key >> dir_shift
  uint32_t level_mask;  // bit l set iff level l present
  int32_t nlevels;
  int8_t levels[32];    // present levels, finest first (locator.cpp:85-89)
  // occupancy records: buckets are 32 consecutive key values (dir_shift
  // = 5, or one bucket when total <= 5); record b = {first position of the
  // bucket, bit v set iff key (b << 5) + v is stored}, so a lookup is one
  // 8-byte load and a popcount.  occ = kOccDense: a record for every
  // bucket of the key space; kOccHash: records of the occupied buckets only,
  // in an open-addressed table (sparse or deep key spaces); kOccNone: the
  // bucket directory + binary search (duplicate keys, or forced)
  int32_t occ;
  // wide = 1: the key needs more than 64 bits (extents spanning most of the
  // int32 range at a fine level): two-word keys through the wide path
  // (wide.cu) -- exact-key hashing, per-level probes
  int32_t wide;
  // packed-space coarsening: when every min anchor is aligned to the
  // coarsest level present (aligned = 1), anchor_mask(p, L) of an in-range
  // point p is its packed key with the low L-shift bits of each coordinate
  // field cleared: key_L = (key & cmask[L]) | (L - shift)
  int32_t aligned;
  uint64_t cmask[32];
};

constexpr int kOccShift = 5;  // key values per occupancy record = 2^5
enum : int32_t { kOccNone = 0, kOccDense = 1, kOccHash = 2 };

/*! Hashed occupancy records: entry = {u64 tag = bucket + 1 (0 = empty),
    u32 start, u32 bits}; two entries per 32-byte table bucket, which a
    lookup reads with ONE 256-bit load (ld.global.nc.v4.u64).  Linear
    probing over table buckets from hash_home; a table bucket with a free
    entry ends a probe (buckets only ever fill up).  Record buckets b and
    b^1 (the two halves of an aligned 64-value range) share a home, b
    preferring entry b & 1, so neighbouring records of a dense region come
    in one load and the extraction's fast path reads 16 bytes.  The table has at least
    twelve entries per occupied record bucket (api.cu); the build reports the longest
    probe (in table buckets). */
/// home table bucket of record bucket b (mask = table buckets - 1, at most
/// 2^32 buckets): a 32-bit multiply-xorshift hash of the pair id, cheap in
/// the lookup loops (a 64-bit multiply is four IMADs)
__host__ __device__ inline uint64_t hash_home(uint64_t bucket, uint64_t mask)
{
  const uint64_t p = bucket >> 1;
  uint32_t x = uint32_t(p) * 0x9E3779B1u ^ uint32_t(p >> 32) * 0x85EBCA77u;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  return uint64_t(x) & mask;
}

__host__ __device__ inline int64_t anchor_mask(int64_t x, int32_t level)
{
  return x & ~((int64_t(1) << level) - 1);  // core.hpp:98-103
}

__host__ __device__ inline bool level_present(const KeyGeom &g, int32_t l)
{
  return l >= 0 && l <= kMaxLevel && ((g.level_mask >> l) & 1u);
}

/// pack an aligned anchor on a present level (caller has range-checked)
__host__ __device__ inline uint64_t pack_unchecked(const KeyGeom &g, int64_t i,
                                                   int64_t j, int64_t k,
                                                   int32_t level)
{
  uint64_t key = uint64_t(level - g.shift);
  if (g.bits[0]) key |= uint64_t((i - g.mn[0]) >> g.shift) << g.sh[0];
  if (g.bits[1]) key |= uint64_t((j - g.mn[1]) >> g.shift) << g.sh[1];
  if (g.bits[2]) key |= uint64_t((k - g.mn[2]) >> g.shift) << g.sh[2];
  return key;
}

/*! snap_on_level's key (locator.cpp:107-119): mask the point to the level,
    reject anchors outside the stored range (which also covers the int32
    guard: the stored range is int32), pack.  false = cannot exist. */
__host__ __device__ inline bool query_key(const KeyGeom &g, int64_t px,
                                          int64_t py, int64_t pz,
                                          int32_t level, uint64_t &key)
{
  if (!level_present(g, level)) return false;
  const int64_t ax = anchor_mask(px, level);
  const int64_t ay = anchor_mask(py, level);
  const int64_t az = anchor_mask(pz, level);
  if (ax < g.mn[0] || ax > g.mx[0] || ay < g.mn[1] || ay > g.mx[1] ||
      az < g.mn[2] || az > g.mx[2])
    return false;
  key = pack_unchecked(g, ax, ay, az, level);
  return true;
}

struct Cell {
  int64_t i, j, k;
  int32_t level;
};

// ---------------------------------------------------------------- wide keys
// A two-word key (lo, hi) = the 128-bit integer with the same field layout
// as the 64-bit key (KeyGeom::sh, bits, lbits), so its order is again the
// reference's (i,j,k,level) order (core.hpp:82-88).
typedef unsigned __int128 u128;

__host__ __device__ inline u128 pack128(const KeyGeom &g, int64_t i, int64_t j, int64_t k,
                                        int32_t level)
{
  u128 key = u128(uint64_t(level - g.shift));
  if (g.bits[0]) key |= u128(uint64_t((i - g.mn[0]) >> g.shift)) << g.sh[0];
  if (g.bits[1]) key |= u128(uint64_t((j - g.mn[1]) >> g.shift)) << g.sh[1];
  if (g.bits[2]) key |= u128(uint64_t((k - g.mn[2]) >> g.shift)) << g.sh[2];
  return key;
}

__host__ __device__ inline Cell unpack128(const KeyGeom &g, u128 key)
{
  Cell c;
  c.level = int32_t(uint64_t(key) & ((uint64_t(1) << g.lbits) - 1)) + g.shift;
  const auto field = [&](int a) -> int64_t {
    if (!g.bits[a]) return g.mn[a];
    const uint64_t u = uint64_t(key >> g.sh[a]) & ((uint64_t(1) << g.bits[a]) - 1);
    return g.mn[a] + int64_t(u << g.shift);
  };
  c.i = field(0);
  c.j = field(1);
  c.k = field(2);
  return c;
}

__host__ __device__ inline Cell unpack(const KeyGeom &g, uint64_t key)
{
  Cell c;
  c.level = int32_t(key & ((uint64_t(1) << g.lbits) - 1)) + g.shift;
  const auto field = [&](int a) -> int64_t {
    if (!g.bits[a]) return g.mn[a];
    const uint64_t u = (key >> g.sh[a]) & ((uint64_t(1) << g.bits[a]) - 1);
    return g.mn[a] + int64_t(u << g.shift);
  };
  c.i = field(0);
  c.j = field(1);
  c.k = field(2);
  return c;
}

/*! the 27-point stencil {-w,0,w}^3 of one cell at its own level, in packed
    key space: a stencil point p = (ox+1) + 3(oy+1) + 9(oz+1) is its own
    anchor at the cell's level, so its key is the cell's key plus packed
    per-axis steps -- valid exactly when the point lies in the stored
    anchor range (bit p of `inrange`). */
struct Stencil {
  uint64_t k0;          // key of the cell itself
  uint64_t sx, sy, sz;  // packed +w per axis (0 for a constant axis)
  uint32_t inrange;     // bit p: point p's anchor is inside [mn, mx]^3
};

__host__ __device__ inline Stencil make_stencil(const KeyGeom &g, uint64_t key, int level)
{
  Stencil s;
  s.k0 = key;
  const uint64_t wu = uint64_t(1) << (level - g.shift);  // w in packed units
  uint32_t out = 0;
  // points with o_axis = -1 / +1, for axis x, y, z (p%3, p/3%3, p/9)
  const uint32_t m_minus[3] = {0x1249249u, 0x1C0E07u, 0x1FFu};
  const uint32_t m_plus[3] = {0x4924924u, 0x70381C0u, 0x7FC0000u};
  uint64_t *step[3] = {&s.sx, &s.sy, &s.sz};
  for (int a = 0; a < 3; a++) {
    if (!g.bits[a]) {
      *step[a] = 0;
      out |= m_minus[a] | m_plus[a];  // a constant axis has no neighbours
      continue;
    }
    const uint64_t u = (key >> g.sh[a]) & ((uint64_t(1) << g.bits[a]) - 1);
    const uint64_t umax = g.umax[a];
    *step[a] = wu << g.sh[a];
    if (u < wu) out |= m_minus[a];
    if (u + wu > umax) out |= m_plus[a];
  }
  s.inrange = ~out & 0x7FFFFFFu;
  return s;
}

/// key of stencil point p (meaningful when bit p of inrange is set)
template <bool DIGITS = false>
__host__ __device__ inline uint64_t stencil_key(const Stencil &s, int p)
{
  // p < 27: p / 3 == (p * 11) >> 5 (exact for p < 32), then signed offsets
  // times the packed steps (mod 2^64: the point's key when it is in range)
  const uint32_t up = uint32_t(p), q1 = (up * 11u) >> 5, q2 = (q1 * 11u) >> 5;
  if (DIGITS)  // unsigned digits 0..2: per axis one 32x64 wide multiply-add
    return (s.k0 - s.sx - s.sy - s.sz) + uint64_t(up - 3u * q1) * s.sx +
           uint64_t(q1 - 3u * q2) * s.sy + uint64_t(q2) * s.sz;
  return s.k0 + uint64_t(int64_t(int32_t(up - 3u * q1) - 1)) * s.sx +
         uint64_t(int64_t(int32_t(q1 - 3u * q2) - 1)) * s.sy +
         uint64_t(int64_t(int32_t(q2) - 1)) * s.sz;
}

// ------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ uint32_t lane_id()
{
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t ldg_u64(const uint64_t *p)
{
  return __ldg(reinterpret_cast<const unsigned long long *>(p));
}

__device__ __forceinline__ ulonglong2 ldg_u64x2(const uint64_t *p)
{
  return __ldg(reinterpret_cast<const ulonglong2 *>(p));
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src,
                                             uint32_t mask = kFull)
{
  return __shfl_sync(mask, (unsigned long long)v, src);
}

/// lower_bound over a sorted u64 span in shared memory
__device__ __forceinline__ int smem_lower_bound(const uint64_t *a, int n,
                                                uint64_t q)
{
  int lo = 0;
  while (n > 0) {
    const int half = n >> 1;
    if (a[lo + half] < q) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}

/// lower_bound over [lo, hi) of the global key array
__device__ __forceinline__ uint64_t global_lower_bound(const uint64_t *keys,
                                                       uint64_t lo,
                                                       uint64_t hi,
                                                       uint64_t q)
{
  uint64_t n = hi - lo;
  while (n > 0) {
    const uint64_t half = n >> 1;
    if (ldg_u64(keys + lo + half) < q) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}

struct SearchCtx {
  const uint64_t *keys;  // sorted packed keys, kKeyPad sentinels after n
  const uint32_t *dir;   // 2^dir_bits + 1 bucket starts
  uint64_t n;
  int32_t dir_shift;
  int32_t shift;         // finest level present (level field offset)
  uint64_t lmask;        // mask of the level field
  unsigned long long *dbg;  // optional event counters (AMRX_DEBUG_COUNTERS)
  // occupancy records (KeyGeom::occ), or null: set only for an index
  // without duplicate keys, where position = rec[b].x + popcount; then the
  // plain directory `dir` is not built (null).  A partition's index holds
  // the records of its key range only: `rec` is offset so rec[b] is still
  // indexed by the global bucket (only in-range buckets are ever read)
  const uint2 *rec;
  uint64_t rec_lo, rec_cnt;  // the built records: buckets [rec_lo, rec_lo + rec_cnt)
  // hashed occupancy records (KeyGeom::occ == kOccHash), or null: 2^k
  // 32-byte table buckets (two entries each), hmask = 2^k - 1
  const ulonglong4 *htab;
  uint64_t hmask;
  // global CellId of local position 0 (a partition of a distributed index;
  // 0 otherwise): added to every id a query or an extraction reports
  int64_t id_base;
};

/// debug event counters, one atomic per warp-level event, lane 0 only
enum DbgEvent {
  kDbgTiles = 0,   // extraction tiles
  kDbgFastNeed,    // stencil points the compile-time fast batches were asked for
  kDbgFastPend,    // of those, left to the runtime loop
  kDbgRuntime,     // points through the runtime loop (batch_find + finer)
  kDbgCoarser,     // probe_coarser calls
  kDbgHashExtra,   // hashed-record probes past the home table bucket
  kDbgFindCalls, kDbgFindRounds, kDbgNarrow, kDbgFallback, kDbgQueries,
  kDbgCount
};

// counters are compiled in only for a diagnostic build (make DBG=1): the
// atomics otherwise bloat the hot loop past the instruction cache
#ifndef AMRX_DBG
#define AMRX_DBG 0
#endif

__device__ __forceinline__ void dbg_add(const SearchCtx &s, int ev,
                                        unsigned long long v = 1)
{
#if AMRX_DBG
  if (s.dbg && (threadIdx.x & 31) == 0) atomicAdd(s.dbg + ev, v);
#endif
}

/// sum of a per-lane count over the warp (all lanes call it)
__device__ __forceinline__ void dbg_sum(const SearchCtx &s, int ev, uint32_t v)
{
#if AMRX_DBG
  v = __reduce_add_sync(0xffffffffu, v);
  if (s.dbg && (threadIdx.x & 31) == 0 && v) atomicAdd(s.dbg + ev, (unsigned long long)v);
#endif
}

/// one event of this lane (divergent code)
__device__ __forceinline__ void dbg_lane(const SearchCtx &s, int ev)
{
#if AMRX_DBG
  if (s.dbg) atomicAdd(s.dbg + ev, 1ull);
#endif
}

/*! lookup through an occupancy record r = rec[q >> 5]: the exact key, or
    under FINER the first stored key with q's anchor and a lower level
    field -- the finest cell at that anchor, which sorts first -- exactly
    what the bucket search returns for unique keys (the level field is the
    key's low part and 32 is a multiple of 2^lbits, lbits <= 5, so an
    anchor's keys share one record). */
template <bool FINER>
__device__ __forceinline__ int64_t occ_resolve(uint64_t q, uint2 r, uint32_t lmask, int &rl)
{
  const uint32_t bit = uint32_t(q) & 31u;
  const uint32_t below = r.y & ((1u << bit) - 1u);
  rl = int(uint32_t(q) & lmask);
  if ((r.y >> bit) & 1u) return int64_t(r.x + uint32_t(__popc(below)));
  if (FINER) {
    const uint32_t grp = bit & ~lmask;  // first value of q's anchor
    const uint32_t m = below & ~((1u << grp) - 1u);
    if (m) {
      const uint32_t f = uint32_t(__ffs(int(m))) - 1u;
      rl = int(f & lmask);
      return int64_t(r.x + uint32_t(__popc(r.y & ((1u << f) - 1u))));
    }
  }
  return -1;
}

__device__ __forceinline__ uint2 ldg_rec(const SearchCtx &s, uint64_t q)
{
  const uint64_t b = q >> kOccShift;  // (KeyGeom::dir_shift is kOccShift for records)
  if (!AMRX_BOUND(b - s.rec_lo < s.rec_cnt, kChkRecord)) return make_uint2(0, 0);
  return __ldg(s.rec + b);
}

/// one table bucket (two entries) in a single 256-bit read-only load
__device__ __forceinline__ ulonglong4 ldg_bucket(const ulonglong4 *p)
{
  ulonglong4 v;
  asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
      : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w)
      : "l"(p));
  return v;
}

/// the record of bucket b in table bucket e (loaded from slot h); found =
/// false with more = true when the probe must go on
__device__ __forceinline__ uint2 bucket_match(ulonglong4 e, uint64_t b, bool &more)
{
  more = false;
  if (e.x == b + 1) return make_uint2(uint32_t(e.y), uint32_t(e.y >> 32));
  if (e.z == b + 1) return make_uint2(uint32_t(e.w), uint32_t(e.w >> 32));
  more = e.x != 0 && e.z != 0;
  return make_uint2(0, 0);
}

/// the hashed record of bucket b, continuing a probe at table bucket h
/// whose content e was already loaded; {0, 0} (no bits) when b is empty
__device__ __forceinline__ uint2 hash_probe(const SearchCtx &s, uint64_t b, uint64_t h,
                                            ulonglong4 e)
{
  for (;;) {
    bool more;
    const uint2 r = bucket_match(e, b, more);
    if (!more) return r;
    h = (h + 1) & s.hmask;
    dbg_lane(s, kDbgHashExtra);
    if (!AMRX_BOUND(h <= s.hmask, kChkHash)) return make_uint2(0, 0);
    e = ldg_bucket(s.htab + h);
  }
}

/// batch_find through the hashed records: the K home slots are loaded
/// together, the (rare) displaced entries probed afterwards
template <int K, bool FINER>
__device__ __forceinline__ void hash_find(const SearchCtx &s, const uint64_t (&q)[K],
                                          const bool (&valid)[K], int64_t (&out)[K],
                                          int (&lvl)[K])
{
  ulonglong4 e[K];
  uint64_t h[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    h[k] = hash_home(q[k] >> s.dir_shift, s.hmask);
    e[k] = valid[k] ? ldg_bucket(s.htab + h[k]) : make_ulonglong4(0, 0, 0, 0);
  }
#pragma unroll
  for (int k = 0; k < K; k++)
    if (valid[k]) {
      const uint2 r = hash_probe(s, q[k] >> s.dir_shift, h[k], e[k]);
      int rl;
      out[k] = occ_resolve<FINER>(q[k], r, uint32_t(s.lmask), rl);
      lvl[k] = rl + s.shift;
    }
}


/*! global-memory path of warp_find for one query: lower_bound over the
    bucket range [lo, hi), then (finer) the run of same-anchor keys before
    it.  Returns the CellId or -1; level receives the hit's level. */
static __device__ __noinline__ int64_t find_in_bucket(const SearchCtx &s, uint64_t lo,
                                               uint64_t hi, uint64_t q,
                                               bool finer, int &level)
{
  const uint64_t p = global_lower_bound(s.keys, lo, hi, q);
  int64_t res = -1;
  int rl = 0;
  if (p < hi && ldg_u64(s.keys + p) == q) {
    res = int64_t(p);
    rl = int(q & s.lmask);
  } else if (finer) {
    const uint64_t anchor = q & ~s.lmask;
    uint64_t x = p;
    while (x > lo && (ldg_u64(s.keys + x - 1) & ~s.lmask) == anchor) x--;
    if (x < p) {
      res = int64_t(x);
      rl = int(ldg_u64(s.keys + x) & s.lmask);
    }
  }
  level = rl + s.shift;
  return res;
}

/// batch_find through the occupancy records only (s.rec must be set)
template <int K, bool FINER>
__device__ __forceinline__ void occ_find(const SearchCtx &s, const uint64_t (&q)[K],
                                         const bool (&valid)[K], int64_t (&out)[K],
                                         int (&lvl)[K])
{
  uint2 r[K];
#pragma unroll
  for (int k = 0; k < K; k++) r[k] = valid[k] ? ldg_rec(s, q[k]) : make_uint2(0, 0);
#pragma unroll
  for (int k = 0; k < K; k++)
    if (valid[k]) {
      int rl;
      out[k] = occ_resolve<FINER>(q[k], r[k], uint32_t(s.lmask), rl);
      lvl[k] = rl + s.shift;
    }
}

/*! K independent lookups per lane advanced in lock-step: the directory
    loads of all K go out together, then every binary-search step issues up
    to K independent key loads, so the dependent-latency chain is that of
    ONE search instead of K.  Same contract as warp_find. */
template <int K, bool FINER>
__device__ __forceinline__ void batch_find(const SearchCtx &s, const uint64_t (&q)[K],
                                           const bool (&valid)[K], int64_t (&out)[K],
                                           int (&lvl)[K])
{
  if (s.rec) {  // occupancy records: no search at all
    occ_find<K, FINER>(s, q, valid, out, lvl);
    return;
  }
  if (s.htab) {
    hash_find<K, FINER>(s, q, valid, out, lvl);
    return;
  }
  uint32_t lo[K], n[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    lo[k] = 0;
    n[k] = 0;
    if (valid[k]) {
      const uint64_t b0 = (FINER ? (q[k] & ~s.lmask) : q[k]) >> s.dir_shift;
      lo[k] = __ldg(s.dir + b0);
      n[k] = __ldg(s.dir + (q[k] >> s.dir_shift) + 1) - lo[k];
    }
  }
  uint32_t first[K];  // bucket start: the FINER scan-back floor
#pragma unroll
  for (int k = 0; k < K; k++) first[k] = lo[k];
  bool more = true;
  while (more) {
    more = false;
#pragma unroll
    for (int k = 0; k < K; k++)
      if (n[k] > 0) {
        const uint32_t half = n[k] >> 1;
        if (ldg_u64(s.keys + lo[k] + half) < q[k]) {
          lo[k] += half + 1;
          n[k] -= half + 1;
        } else {
          n[k] = half;
        }
        more |= n[k] > 0;
      }
  }
  uint64_t at[K], before[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    at[k] = valid[k] ? ldg_u64(s.keys + lo[k]) : 0;  // padded: lo <= n
    before[k] = (valid[k] && FINER && lo[k] > first[k]) ? ldg_u64(s.keys + lo[k] - 1) : ~0ull;
  }
#pragma unroll
  for (int k = 0; k < K; k++) {
    if (!valid[k]) continue;
    int64_t res = -1;
    int rl = 0;
    if (at[k] == q[k]) {
      res = int64_t(lo[k]);
      rl = int(q[k] & s.lmask);
    } else if (FINER && (before[k] & ~s.lmask) == (q[k] & ~s.lmask)) {
      // same anchor, lower level: walk to the first of the run (rarely >1)
      uint32_t x = lo[k] - 1;
      while (x > first[k] && (ldg_u64(s.keys + x - 1) & ~s.lmask) == (q[k] & ~s.lmask)) x--;
      res = int64_t(x);
      rl = int(ldg_u64(s.keys + x) & s.lmask);
    }
    out[k] = res;
    lvl[k] = rl + s.shift;
  }
}

/// lower_bound of q in win[from, cnt), galloping from `from`
__device__ __forceinline__ int gallop_lower_bound(const uint64_t *win, int from,
                                                  int cnt, uint64_t q)
{
  int lo = from, n;
  if (from == 0) {
    n = cnt;  // first query of the window: plain binary search
  } else {
    int step = 1;
    while (lo + step - 1 < cnt && win[lo + step - 1] < q) {
      lo += step;
      step <<= 1;
    }
    n = (lo + step - 1 < cnt ? lo + step - 1 : cnt) - lo;
  }
  while (n > 0) {
    const int half = n >> 1;
    if (win[lo + half] < q) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}

/*! Warp-cooperative exact lookup of up to NQ keys per lane (find_exact,
    locator.cpp:94-101: the FIRST position holding the key, or miss).

    1. Each lane reads the directory bucket bounds of its smallest and
       largest query: every key of the bucket range lies in [lo, hi).
    2. The warp takes the lowest pending lane as leader, narrows the
       leader's range with a 32-ary search (one coalesced probe of 32 keys
       per step) until it fits one window, and stages that window of kWin
       keys in shared memory with 16-byte vector loads.
    3. Every pending lane resolves each query it can prove from the window
       (found, or absent because the window brackets it); the rest go
       round again with the next leader, then fall back to a per-lane
       binary search of their own bucket.  A lane's queries are searched in
       order, galloping from the previous one's position (the callers pass
       them ascending).

    FINER: when the exact key is absent, also report the first stored key
    with the same anchor and a lower level.  Keys differ from the query
    only in the level field then, so they sit directly before its
    lower_bound: for a stencil point p (a multiple of the owner width w)
    every finer cell containing p is anchored exactly at p, so this is
    snap's "remaining levels finest first" probe over the finer levels
    (locator.cpp:125-133) answered from the same window.

    out[t] = CellId or -1, lvl[t] = level field of the hit (FINER hits
    report their own level).  Inactive queries are left untouched.  All 32
    lanes must call this together. */
template <int NQ, bool FINER>
__device__ void warp_find(const SearchCtx &s, const uint64_t (&q)[NQ],
                          const bool (&valid)[NQ], int64_t (&out)[NQ],
                          int (&lvl)[NQ], uint64_t *win)
{
  if (s.rec) {  // occupancy records: per lane, no search (warp-uniform branch)
    occ_find<NQ, FINER>(s, q, valid, out, lvl);
    return;
  }
  if (s.htab) {
    hash_find<NQ, FINER>(s, q, valid, out, lvl);
    return;
  }
  const uint32_t lane = lane_id();
  const uint64_t amask = FINER ? ~s.lmask : ~0ull;
  bool any = false;
  uint64_t qmin = ~0ull, qmax = 0;
#pragma unroll
  for (int t = 0; t < NQ; t++)
    if (valid[t]) {
      any = true;
      const uint64_t lowest = q[t] & amask;  // same anchor, any level
      qmin = lowest < qmin ? lowest : qmin;
      qmax = q[t] > qmax ? q[t] : qmax;
    }
  uint64_t lo = 0, hi = 0;
  if (any) {
    lo = __ldg(s.dir + (qmin >> s.dir_shift));
    hi = __ldg(s.dir + (qmax >> s.dir_shift) + 1);
  }
  uint32_t unresolved = 0;  // bit t: query t still open
#pragma unroll
  for (int t = 0; t < NQ; t++)
    if (valid[t]) {
      if (lo == hi)
        out[t] = -1;  // empty bucket range: absent
      else
        unresolved |= 1u << t;
    }

  if (AMRX_DBG && s.dbg) {
    int nv = 0;
#pragma unroll
    for (int t = 0; t < NQ; t++) nv += valid[t];
    dbg_add(s, kDbgFindCalls);
    dbg_add(s, kDbgQueries, __reduce_add_sync(kFull, nv));
  }
  for (int round = 0; round < 3; round++) {
    const uint32_t pend = __ballot_sync(kFull, unresolved != 0);
    if (!pend) break;
    dbg_add(s, kDbgFindRounds);
    const int leader = __ffs(pend) - 1;
    // leader's smallest open query (anchor-lowest under FINER)
    uint64_t lq = ~0ull;
#pragma unroll
    for (int t = 0; t < NQ; t++)
      if ((unresolved >> t) & 1) {
        const uint64_t v = q[t] & amask;
        lq = v < lq ? v : lq;
      }
    lq = shfl_u64(lq, leader);
    uint64_t L = shfl_u64(lo, leader);
    uint64_t H = shfl_u64(hi, leader);
    // 32-ary narrowing of [L, H) around lower_bound(lq); 4 keys of slack
    // so the window below brackets it
    while (H - L > uint64_t(kWin - 4)) {
      const uint64_t step = (H - L + 31) >> 5;
      const uint64_t pos = L + lane * step;
      const bool below = pos < H && ldg_u64(s.keys + pos) < lq;
      const int c = __popc(__ballot_sync(kFull, below));
      const uint64_t nl = c > 0 ? L + uint64_t(c - 1) * step + 1 : L;
      const uint64_t pc = L + uint64_t(c) * step;
      const uint64_t nh = (c < 32 && pc < H) ? pc + 1 : H;
      L = nl;
      H = nh;
      dbg_add(s, kDbgNarrow);
    }
    // stage the window [ws, ws + kWin): 16-byte aligned, starting at or
    // before L-1 so the leader's key[L-1] < lq proof lies inside it
    const uint64_t ws = L >= 1 ? ((L - 1) & ~1ull) : 0;
    __syncwarp();
#pragma unroll
    for (int v = 0; v < kWin / 64; v++) {
      const uint64_t at = ws + 2 * lane + 64 * v;
      const ulonglong2 kv = ldg_u64x2(s.keys + at);  // padded: never OOB
      reinterpret_cast<ulonglong2 *>(win)[lane + 32 * v] = kv;
    }
    __syncwarp();
    const uint64_t wend = ws + kWin < s.n ? ws + kWin : s.n;
    const int cnt = int(wend - ws);
    int from = 0;
    uint64_t prev = 0;
#pragma unroll
    for (int t = 0; t < NQ; t++) {
      if (!((unresolved >> t) & 1)) continue;
      if (q[t] < prev) from = 0;
      const int p = gallop_lower_bound(win, from, cnt, q[t]);
      from = p;
      prev = q[t];
      bool done = false;
      int64_t res = -1;
      int rl = 0;
      if (p < cnt && win[p] == q[t]) {
        if (p > 0 || ws <= lo) {
          done = true;
          res = int64_t(ws + p);
          rl = int(q[t] & s.lmask);
        }
      } else if (p == 0) {
        done = ws <= lo;
      } else if (p == cnt) {
        done = wend >= hi;
      } else {
        done = true;  // bracketed by two window keys, not equal
      }
      if (FINER && done && res < 0) {
        // same-anchor keys with lower levels end right before p
        int x = p - 1;
        const uint64_t anchor = q[t] & ~s.lmask;
        while (x >= 0 && (win[x] & ~s.lmask) == anchor) x--;
        if (x < 0 && ws > lo) {
          done = false;  // the run may continue before the window
        } else if (x + 1 < p) {
          res = int64_t(ws + x + 1);
          rl = int(win[x + 1] & s.lmask);
        }
      }
      if (done) {
        out[t] = res;
        lvl[t] = rl + s.shift;
        unresolved &= ~(1u << t);
      }
    }
  }
  if (AMRX_DBG && s.dbg) dbg_add(s, kDbgFallback, __reduce_add_sync(kFull, __popc(unresolved)));
  // fallback: per-lane binary search of the own bucket range (rare; out of
  // line to keep the hot loop inside the instruction cache)
#pragma unroll
  for (int t = 0; t < NQ; t++)
    if ((unresolved >> t) & 1) {
      int rl;
      out[t] = find_in_bucket(s, lo, hi, q[t], FINER, rl);
      lvl[t] = rl;
    }
}

}  // namespace amrx
