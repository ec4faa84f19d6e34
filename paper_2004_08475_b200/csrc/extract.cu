// The fused hot path: per-cell dual enumeration + ownership rules + marching
// cubes on degenerate hexes + ordered emission, in one persistent kernel.
//
// Reference behaviour restated here (paths under /root/reference/):
//   candidate order, task t -> cell t>>3, delta t&7   proj/src/pipeline.cpp:40-57
//   dual_base_of                                      proj/include/amriso/dual.hpp:61-67
//   try_build_dual rules #1/#2/#3, first failing
//   corner decides the reject reason                  proj/src/dual.cpp:41-72
//   snap: hint level first, then levels finest first  proj/src/locator.cpp:107-134
//   strict '>' case mask, table_corner, tri_table     proj/src/contour.cpp:22-28,
//                                                     proj/src/mc_tables.cpp:318-330
//   interpolation (lower CellId first, no FMA)        proj/src/contour.cpp:30-50
//   sliver drop on exact equality                     proj/src/contour.cpp:80-84
//   two-pass count -> prefix -> emit                  proj/src/pipeline.cpp:80-146
//
// B200 design: one warp owns a tile of 32 consecutive cells,
// one per lane, handed out by an atomic ticket.  Instead of 8 independent
// candidates x 8 corner snaps, each lane resolves the points of its cell's
// 27-point stencil {-w,0,w}^3 its live candidates need: a point's key is the
// cell key plus packed steps (Stencil), a lookup is one occupancy record load
// + popcount, and the 14 points of a uniform region have compile-time
// offsets (fast_batch).  Round 0 resolves every candidate's corner 0 (82-86%
// of candidates die there); round 1 what the survivors still need.  Points
// are classified into 27-bit masks and a candidate is a mask test over its
// corner cube; the lowest failing bit is its first failing corner, so the
// reported reason is the reference's.  Duals and triangles go to per-warp
// staging chunks with per-tile (offset, count) records; a scan over the tile
// counts and reorder_kernel restore candidate order -- the reference's
// "pass 1 / prefix sum / pass 2" with the search run once.
#include "internal.h"
#include "mc_tables.inc"
#include "wide.cuh"

#include <algorithm>
#include <atomic>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <mutex>
#include <unordered_map>
#include <cstdio>
#include <cstdlib>

namespace amrx {

namespace {

#ifndef AMRX_EXTRACT_THREADS
#define AMRX_EXTRACT_THREADS 1024  // one CTA per SM: C4 extraction 43.7 -> 42.7 ms (512: 43.1, 128: 43.8)
#endif
constexpr int kThreads = AMRX_EXTRACT_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kTileCells = 32;  // cells one warp tile owns (one per lane)

// point index p = (ox+1) + 3(oy+1) + 9(oz+1), o in {-1,0,1}^3; self = 13
constexpr uint32_t kCorner0Points = (1u << 0) | (1u << 1) | (1u << 3) |
                                    (1u << 4) | (1u << 9) | (1u << 10) |
                                    (1u << 12) | (1u << 13);

enum : uint32_t { kOk = 0, kMiss = 1, kFiner = 2, kLower = 3 };

// case rows, staged into shared memory per CTA (lanes index them divergently)
__constant__ uint64_t c_mc_rows[256] = {AMRX_MC_PACKED_ROWS};

/// stencil point of corner d of candidate delta (dual.hpp:61-67 + dual.cpp:49-53)
__device__ __forceinline__ int point_of(int delta, int d)
{
  return ((d & 1) + (delta & 1)) + 3 * (((d >> 1) & 1) + ((delta >> 1) & 1)) +
         9 * (((d >> 2) & 1) + ((delta >> 2) & 1));
}


__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v)
{
  const uint32_t lane = lane_id();
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, v, off);
    if (lane >= off) v += y;
  }
  return v;
}

constexpr uint32_t kDualChunk = 1024;  // >= 8 * 32, the most one tile emits
constexpr uint32_t kTriChunk = 2048;   // >= 40 * 32 (5 triangles x 8 duals)

/*! Rounds (run_extract): a launch processes tiles in ticket order until
    every tile is done, the round's tile limit is reached, or a staging
    buffer's cursor passes its guard (capacity minus the headroom the tiles
    already in flight may still claim: one chunk per warp per tile, with a
    2x margin).  The warp that passes a guard adds kStopTicket to the ticket
    counter -- every later ticket is out of range -- and records the counter
    it saw, so the round's tiles are exactly [first ticket, stop).  No
    allocation can exceed its buffer, and no tile is ever half done. */
constexpr unsigned long long kStopTicket = 1ull << 40;

__device__ __forceinline__ void stop_round(unsigned long long *ticket,
                                           unsigned long long *stop_at)
{
  const unsigned long long old = atomicAdd(ticket, kStopTicket);
  if (old < kStopTicket) atomicMin(stop_at, old);
}

/*! staging space for `agg` items of this tile from the warp's private
    chunk (cur_end[0], cur_end[1] in shared memory); a new chunk comes from
    one atomicAdd on the arena cursor (and may end the round).  Warp-uniform. */
__device__ __forceinline__ uint64_t reserve(uint64_t *cur_end, uint32_t agg,
                                            uint32_t chunk,
                                            unsigned long long *cursor, uint64_t guard,
                                            unsigned long long *ticket,
                                            unsigned long long *stop_at)
{
  if (agg == 0) return 0;
  uint64_t cur = cur_end[0], end = cur_end[1];
  if (cur + agg > end) {
    unsigned long long b = 0;
    if (lane_id() == 0) {
      b = atomicAdd(cursor, (unsigned long long)chunk);
      if (b + chunk > guard) stop_round(ticket, stop_at);
    }
    b = __shfl_sync(kFull, b, 0);
    cur = b;
    end = b + chunk;
  }
  __syncwarp();
  if (lane_id() == 0) {
    cur_end[0] = cur + agg;
    cur_end[1] = end;
  }
  __syncwarp();
  return cur;
}

/*! A crossing dual handed from extract_kernel to mc_jobs_kernel: its corner
    ids and levels, owner key, candidate and triangle count bound, reserved
    staging slot and tile.  64 bytes. */
struct McJob {
  uint32_t id[8];
  uint64_t key;
  uint64_t out;
  uint8_t lev[8];
  uint32_t tile;
  uint16_t meta;  // delta | ntab << 8
  uint16_t pad;
};
static_assert(sizeof(McJob) == 64, "McJob is 64 bytes");

/*! Marching cubes writes each dual's triangles at the case table's upper
    bound; the slots a dual leaves unused (sliver triangles are dropped,
    contour.cpp:80-84) get a signalling-NaN marker in the word holding the
    sign and exponent of x0 -- word 0 of an f32 slot, word 1 (the high half)
    of an f64 slot -- and reorder_tri_kernel skips them.  Arithmetic never
    produces a signalling NaN (a NaN result is quiet), so no real vertex
    matches: all-ones exponent with the quiet bit clear. */
constexpr uint32_t kGapMark32 = 0xFFB4C0DEu;  // f32: exponent 0xFF, quiet bit 0
constexpr uint32_t kGapMark64 = 0xFFF4C0DEu;  // f64 high word: exponent 0x7FF, quiet bit 0
__host__ __device__ constexpr int gap_word(int words) { return words == 9 ? 0 : 1; }
__host__ __device__ constexpr uint32_t gap_mark(int words)
{
  return words == 9 ? kGapMark32 : kGapMark64;
}

/// bit i of the result: scalar i > iso (the strict case test of contour.cpp:22-28)
__global__ void __launch_bounds__(256)
sign_bits_kernel(const double *__restrict__ scal, uint64_t n, double iso,
                 uint32_t *__restrict__ bits)
{
  // a warp takes 4 consecutive 32-value words per step, loads first
  constexpr int U = 4;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t base = (uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u)) * U;
       base < n; base += stride) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t r = base + 32 * u + (threadIdx.x & 31);
      v[u] = r < n ? __ldg(scal + r) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t r = base + 32 * u + (threadIdx.x & 31);
      const uint32_t word = __ballot_sync(kFull, r < n && v[u] > iso);
      if ((threadIdx.x & 31) == 0 && base + 32 * u < n) bits[(base >> 5) + u] = word;
    }
  }
}

/*! the triangle variant of reorder_kernel: a tile's staging block holds
    up[t] reserved slots of which cnt[t] are triangles; when slivers left
    gaps (cnt < up) the warp compacts the block while moving it, 32 slots at
    a time: a ballot of the kept slots, then one flat copy of their words */
__global__ void __launch_bounds__(256)
reorder_tri_kernel(const uint32_t *__restrict__ cnt, const uint32_t *__restrict__ up,
                   const uint64_t *__restrict__ src_off, const uint64_t *__restrict__ dst_off,
                   uint32_t tiles, int words, const uint32_t *__restrict__ src,
                   uint32_t *__restrict__ dst, uint64_t dst_base, uint64_t dst_cap,
                   uint64_t src_n)
{
  __shared__ uint8_t s_kept[8][32];
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < tiles; t += warps) {
    const uint32_t n = cnt[t], u = up[t];
    if (!n) continue;
    const uint64_t so = src_off[t], d0 = dst_base + dst_off[t];
    if (!AMRX_BOUND(so + u <= src_n && n <= u, kChkStage)) continue;
    if (n == u) {
      const uint64_t keep = d0 >= dst_cap ? 0 : (d0 + n > dst_cap ? dst_cap - d0 : n);
      const uint64_t nw = keep * uint64_t(words);
      for (uint64_t w = lane; w < nw; w += 32) dst[d0 * words + w] = __ldg(src + so * words + w);
      continue;
    }
    uint64_t done = 0;
    const int gw = gap_word(words);
    const uint32_t gm = gap_mark(words);
    const int wib = threadIdx.x >> 5;
    for (uint32_t i0 = 0; i0 < u; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool ok = i < u && __ldg(src + (so + i) * words + gw) != gm;
      const uint32_t bal = __ballot_sync(kFull, ok);
      // the kept slots of this chunk in order (rank -> lane), then one
      // flat copy of their words across the warp
      if (ok) s_kept[wib][__popc(bal & lanemask_lt())] = uint8_t(lane);
      __syncwarp();
      const uint32_t kept = __popc(bal), nw = kept * uint32_t(words);
      for (uint32_t w = lane; w < nw; w += 32) {
        const uint32_t j = w / uint32_t(words), c = w - j * uint32_t(words);
        const uint64_t d = d0 + done + j;
        if (d < dst_cap) dst[d * words + c] = __ldg(src + (so + i0 + s_kept[wib][j]) * words + c);
      }
      done += kept;
      __syncwarp();
    }
  }
}

/*! move each tile's block from its staging position to its place in
    candidate order (final offset = exclusive scan of tile counts): one warp
    per tile, `words` 32-bit words per item, coalesced both ways */
__global__ void __launch_bounds__(256)
reorder_kernel(const uint32_t *__restrict__ cnt, const uint64_t *__restrict__ src_off,
               const uint64_t *__restrict__ dst_off, uint32_t tiles, int words,
               const uint32_t *__restrict__ src, uint32_t *__restrict__ dst,
               uint64_t dst_base, uint64_t dst_cap, int words2,
               const uint32_t *__restrict__ src2, uint32_t *__restrict__ dst2, uint64_t src_n)
{
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < tiles;
       t += warps) {
    const uint32_t n = cnt[t];
    if (!n) continue;
    const uint64_t so = src_off[t], d0 = dst_base + dst_off[t];
    if (!AMRX_BOUND(so + n <= src_n, kChkStage)) continue;
    const uint64_t keep = d0 >= dst_cap ? 0 : (d0 + n > dst_cap ? dst_cap - d0 : n);
    const uint64_t nw = keep * uint64_t(words);
    for (uint64_t w = lane; w < nw; w += 32)
      dst[d0 * words + w] = __ldg(src + so * words + w);
    if (words2) {
      const uint64_t nw2 = keep * uint64_t(words2);
      for (uint64_t w = lane; w < nw2; w += 32)
        dst2[d0 * words2 + w] = __ldg(src2 + so * words2 + w);
    }
  }
}

struct KArgs {
  SearchCtx s;
  KeyGeom g;
  const uint32_t *above;  // bit i: scalar i > iso (EMIT_TRI)
  bool unique;            // no duplicate keys in the index
  const double *scal;
  uint64_t cell_begin, cell_end;
  uint32_t num_tiles;
  double iso;
  uint32_t *corners;
  uint64_t *tasks;
  uint64_t dual_cap;
  void *xyz;
  uint64_t tri_cap;
  uint32_t *tile_dual_cnt;
  uint64_t *tile_dual_off;
  uint32_t *tile_tri_cnt;  // triangles kept (upper bound minus slivers)
  uint32_t *tile_tri_up;   // slots reserved (the case tables' upper bound)
  uint64_t *tile_tri_off;
  struct McJob *jobs;      // crossing duals for mc_jobs_kernel (EMIT_TRI)
  uint64_t job_cap;
  // round control: tiles [ticket, tile_limit); a cursor past its guard ends
  // the round (stop_round)
  uint64_t tile_limit;
  uint64_t dual_guard, tri_guard, job_guard;
  unsigned long long *ticket;
  unsigned long long *stop_at;
  unsigned long long *out;  // [0..3] counters, [4] duals, [5] tris counted,
                            // [6] tris written, [7] error flags,
                            // [8] dual arena cursor, [9] tri arena cursor,
                            // [10] job cursor
};

struct Smem {
  uint32_t id[kWarps][27][32];
  uint8_t lev[kWarps][27][32];
  uint64_t mc_rows[256];
  // per-warp accumulators (lane 0 writes): [0..3] reject counters, [4]
  // duals, [5] triangles counted, [6] triangles written; staging chunk
  // cursors (cur, end) for duals and triangles
  unsigned long long acc[kWarps][8];
  uint64_t chunk[kWarps][4];
  uint4 mk[kWarps][32];  // compacted runtime loop: per-lane mark bits (ok, miss, fin, low)
};

/// slot-numbered corner mask -> table row (mc::to_table_case, mc_tables.cpp:324-330)
__device__ __forceinline__ int table_row(uint32_t mask)
{
  int row = 0;
#pragma unroll
  for (int t = 0; t < 8; t++)
    if (mask & (1u << ((AMRX_MC_TABLE_CORNER >> (3 * t)) & 7))) row |= 1 << t;
  return row;
}

/// centre of the corner cell: anchor + half width, in double (core.hpp:113-118).
/// The reference's double(anchor) + 0.5 * 2^level is exact (|anchor| < 2^32,
/// level <= 30), so it equals (2 * anchor + 2^level) converted once and
/// halved -- the same bits with one conversion and one multiply
__device__ __forceinline__ double centre(int64_t anchor, int level)
{
  return __dmul_rn(0.5, double(2 * anchor + (int64_t(1) << level)));
}

/*! marching cubes over one accepted dual (contour.cpp:52-87): write its
    non-sliver triangles from slot `at` (staging capacity `cap`) and return
    how many.  FP64 with explicit round-to-nearest intrinsics: no FMA
    contraction, matching the reference's -ffp-contract=off build.
    corner(d) gives the id and level of the dual's corner d (an edge's
    endpoints are runtime corner numbers: they are re-read through it from
    shared memory rather than kept in dynamically indexed arrays, which
    would live in local memory). */
template <bool F32, bool GAPS = true, typename Corner, typename TCache>
__device__ __forceinline__ int mc_core(const double *scal, const uint64_t *rows, const Cell &c,
                                       int delta, double iso, void *out, uint64_t at,
                                       uint64_t cap, uint32_t &err, Corner corner, TCache tcache)
{
  const int64_t w = int64_t(1) << c.level;
  int mask = 0;
#pragma unroll
  for (int d = 0; d < 8; d++)
    if (__ldg(scal + corner(d).x) > iso) mask |= 1 << d;
  const uint64_t word = rows[mask];  // rows pre-permuted by corner mask
  const int ntab = int(word & 15);
  if (ntab == 0) return 0;

  // an edge's endpoints, the lower CellId first (contour.cpp:42-44)
  const auto ends_of = [&](int e, int &u, int &v, uint2 &cu, uint2 &cv) {
    const uint32_t ends = e < 8 ? uint32_t(AMRX_MC_EDGE_LO >> (8 * e))
                                : uint32_t(AMRX_MC_EDGE_HI >> (8 * (e - 8)));
    u = int(ends & 15);
    v = int((ends >> 4) & 15);
    cu = corner(u);  // (id, level)
    cv = corner(v);
    if (cv.x < cu.x) {
      const int t = u;
      u = v;
      v = t;
      const uint2 tc = cu;
      cu = cv;
      cv = tc;
    }
  };
  // the interpolation parameter of each distinct edge the case's triangles
  // use (contour.cpp:30-50), computed once: a vertex shared by two triangles
  // is the same arithmetic on the same operands, so the same bits
  {
    uint32_t used = 0;
    for (int q = 0; q < 3 * ntab; q++) used |= 1u << ((word >> (4 + 4 * q)) & 15);
    for (; used; used &= used - 1) {
      const int e = __ffs(used) - 1;
      int u, v;
      uint2 cu, cv;
      ends_of(e, u, v, cu, cv);
      if (cu.x == cv.x) err |= 1u;  // collapsed edge selected (contour.cpp:67-70)
      const double vu = __ldg(scal + cu.x), vv = __ldg(scal + cv.x);
      tcache(e) = __ddiv_rn(__dsub_rn(iso, vu), __dsub_rn(vv, vu));
    }
  }

  const auto edge_point = [&](int e, double (&pt)[3]) {
    int u, v;
    uint2 cu, cv;
    ends_of(e, u, v, cu, cv);
    const double t = tcache(e);
    const int ou[3] = {((u & 1) + (delta & 1)) - 1, (((u >> 1) & 1) + ((delta >> 1) & 1)) - 1,
                       (((u >> 2) & 1) + ((delta >> 2) & 1)) - 1};
    const int ov[3] = {((v & 1) + (delta & 1)) - 1, (((v >> 1) & 1) + ((delta >> 1) & 1)) - 1,
                       (((v >> 2) & 1) + ((delta >> 2) & 1)) - 1};
    const int64_t self[3] = {c.i, c.j, c.k};
    const int lu = int(cu.y), lvv = int(cv.y);
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
      const double pa = centre(anchor_mask(self[ax] + ou[ax] * w, lu), lu);
      const double pb = centre(anchor_mask(self[ax] + ov[ax] * w, lvv), lvv);
      pt[ax] = __dadd_rn(pa, __dmul_rn(t, __dsub_rn(pb, pa)));
    }
  };

  int count = 0;
  for (int tri = 0; tri < ntab; tri++) {
    double pv[3][3];
#pragma unroll 1
    for (int k = 0; k < 3; k++)  // one copy of the edge code (I-cache)
      edge_point(int((word >> (4 + 12 * tri + 4 * k)) & 15), pv[k]);
    const double *p0 = pv[0], *p1 = pv[1], *p2 = pv[2];
    const bool e01 = p0[0] == p1[0] && p0[1] == p1[1] && p0[2] == p1[2];
    const bool e12 = p1[0] == p2[0] && p1[1] == p2[1] && p1[2] == p2[2];
    const bool e02 = p0[0] == p2[0] && p0[1] == p2[1] && p0[2] == p2[2];
    if (e01 || e12 || e02) continue;
    const uint64_t slot = at + uint64_t(count);
    if (slot < cap) {
      if (F32) {
        float *o = static_cast<float *>(out) + slot * 9;
        o[0] = float(p0[0]); o[1] = float(p0[1]); o[2] = float(p0[2]);
        o[3] = float(p1[0]); o[4] = float(p1[1]); o[5] = float(p1[2]);
        o[6] = float(p2[0]); o[7] = float(p2[1]); o[8] = float(p2[2]);
      } else {
        double *o = static_cast<double *>(out) + slot * 9;
        o[0] = p0[0]; o[1] = p0[1]; o[2] = p0[2];
        o[3] = p1[0]; o[4] = p1[1]; o[5] = p1[2];
        o[6] = p2[0]; o[7] = p2[1]; o[8] = p2[2];
      }
    }
    count++;
  }
  for (int g = count; GAPS && g < ntab; g++) {  // mark the slots slivers left unused
    const uint64_t slot = at + uint64_t(g);
    if (slot < cap)
      static_cast<uint32_t *>(out)[slot * (F32 ? 9 : 18) + gap_word(F32 ? 9 : 18)] =
        gap_mark(F32 ? 9 : 18);
  }
  return count;
}

struct McArgs {
  KeyGeom g;
  const double *scal;
  double iso;
  const McJob *jobs;
  uint64_t job_cap;
  void *xyz;
  uint64_t tri_cap;
  uint32_t *tile_tri_cnt;
  unsigned long long *out;  // [5] tris counted, [6] written, [7] errors, [10] jobs
};

#ifndef AMRX_MC_THREADS
#define AMRX_MC_THREADS 256
#endif
constexpr int kMcThreads = AMRX_MC_THREADS;

/*! marching cubes over the crossing duals extract_kernel queued, one per
    thread: every lane busy (inside extract_kernel only the few lanes of a
    tile that own a crossing dual were), and its own register budget.  A
    job's corner ids and levels sit in this thread's shared-memory column. */
struct McSmem {
  double tcs[12][kMcThreads];
  uint64_t rows[256];
  uint32_t jid[8][kMcThreads];
  uint8_t jlev[8][kMcThreads];
};

template <bool F32>
#ifndef AMRX_MC_MINB
#define AMRX_MC_MINB 4
#endif
__global__ void __launch_bounds__(kMcThreads, AMRX_MC_MINB)
mc_jobs_kernel(const __grid_constant__ McArgs a)
{
  extern __shared__ __align__(16) unsigned char mc_smem_raw[];
  McSmem &ms = *reinterpret_cast<McSmem *>(mc_smem_raw);
  uint64_t *rows = ms.rows;
  auto &jid = ms.jid;
  auto &jlev = ms.jlev;
  auto &tcs = ms.tcs;  // per edge interpolation parameter
  for (int i = threadIdx.x; i < 256; i += kMcThreads) rows[i] = c_mc_rows[table_row(uint32_t(i))];
  __syncthreads();
  const uint64_t n = std::min<uint64_t>(*(volatile unsigned long long *)(a.out + 10), a.job_cap);
  const int t = threadIdx.x;
  uint32_t err = 0;
  unsigned long long wrote_sum = 0;
  for (uint64_t j = uint64_t(blockIdx.x) * kMcThreads + t; j < n;
       j += uint64_t(gridDim.x) * kMcThreads) {
    if (!AMRX_BOUND(j < a.job_cap, kChkJob)) break;
    const McJob &job = a.jobs[j];
#pragma unroll
    for (int d = 0; d < 8; d++) {
      jid[d][t] = job.id[d];
      jlev[d][t] = job.lev[d];
    }
    const Cell c = unpack(a.g, job.key);
    const uint32_t meta = job.meta;
    const int wrote = mc_core<F32>(a.scal, rows, c, int(meta & 7), a.iso, a.xyz, job.out,
                                   a.tri_cap, err,
                                   [&](int d) { return make_uint2(jid[d][t], jlev[d][t]); },
                                   [&](int e) -> double & { return tcs[e][t]; });
    const uint32_t deficit = (meta >> 8) - uint32_t(wrote);
    if (deficit) atomicSub(a.tile_tri_cnt + job.tile, deficit);
    wrote_sum += uint64_t(wrote);
  }
  wrote_sum = __reduce_add_sync(kFull, uint32_t(wrote_sum));
  err = __reduce_or_sync(kFull, err);
  if ((t & 31) == 0) {
    if (wrote_sum) {
      atomicAdd(a.out + 5, wrote_sum);
      atomicAdd(a.out + 6, wrote_sum);
    }
    if (err) atomicOr(a.out + 7, (unsigned long long)err);
  }
}

struct Hit {
  int64_t id;
  int level;
};

/*! coarser-level probe for one point the hint+finer lookup missed: the
    present levels above the hint (bit L of `cand` = level L), ascending
    (the reference's finest-first order restricted to them).  Per lane, no
    warp collectives; rare, so out of line -- and scalar, so the caller's
    batch arrays stay in registers. */
__device__ __noinline__ Hit probe_coarser(const KArgs &a, int level, const Stencil &st,
                                          int p, uint32_t cand)
{
  const KeyGeom &g = a.g;
  dbg_lane(a.s, kDbgCoarser);
  struct {
    int level;
  } c{level};
  if (g.aligned && ((st.inrange >> p) & 1u)) {
    // in-range point, aligned origin: coarsen in packed key space
    const uint64_t q0 = stencil_key(st, p);
    while (cand) {
      const int L = __ffs(cand) - 1;
      cand &= cand - 1;
      uint64_t q[1] = {(q0 & g.cmask[L]) | uint64_t(L - g.shift)};
      const bool v[1] = {true};
      int64_t o[1] = {-1};
      int l1[1];
      batch_find<1, false>(a.s, q, v, o, l1);
      if (o[0] >= 0) return Hit{o[0], L};
    }
    return Hit{-1, c.level};
  }
  // the cell's coordinates only on this (unaligned-origin or out-of-range
  // point) path: decoded from its key here, so the hot loop carries just
  // the level
  const Cell cc = unpack(g, st.k0);
  const int64_t w = int64_t(1) << c.level;
  const int64_t px = cc.i + (p % 3 - 1) * w, py = cc.j + ((p / 3) % 3 - 1) * w,
                pz = cc.k + (p / 9 - 1) * w;
  while (cand) {
    const int L = __ffs(cand) - 1;
    cand &= cand - 1;
    uint64_t q[1];
    bool v[1];
    int64_t o[1] = {-1};
    int l1[1];
    v[0] = query_key(g, px, py, pz, L, q[0]);
    if (!v[0]) continue;
    batch_find<1, false>(a.s, q, v, o, l1);
    if (o[0] >= 0) return Hit{o[0], L};
  }
  return Hit{-1, c.level};
}

// ---------------------------------------------------------------------------
// Mask-based rules: each resolved stencil point
// is classified into four 27-bit masks, and a candidate's fate is a mask test
// over its corner cube (no per-corner walk).

/// per-lane point classification (bit p = stencil point p), dual.cpp:60-67
struct Marks {
  uint32_t ok, miss, fin, low;
  __device__ __forceinline__ uint32_t resolved() const { return ok | miss | fin | low; }
};

/// a candidate's corners {0,1}^3 as stencil bits, shifted by its corner 0
constexpr uint32_t kCube = 0x361Bu;  // points 0,1,3,4,9,10,12,13
__host__ __device__ constexpr int base_of(int delta)
{
  return (delta & 1) + 3 * ((delta >> 1) & 1) + 9 * (delta >> 2);
}

constexpr uint32_t kFast0 = kCorner0Points & ~(1u << 13);  // 0 1 3 4 9 10 12
constexpr uint32_t kFast1 = kCube << 13 & ~(1u << 13);       // 14 16 17 22 23 25 26

/*! stencil points Ps (compile-time) for the lanes that need them, from one
    occupancy record each (the key from compile-time steps): every record
    load of the list is issued before any is used, so they are in flight
    together.  The common case -- the point's own anchor exists on the hint
    level -- is resolved here; anything else (finer, coarser, absent) is
    left in `pend` for the runtime loop.  L = kOccDense reads the dense
    record (8 bytes); L = kOccHash the preferred entry of the record's home
    table bucket (16 bytes: tag + record) -- an entry holding another bucket
    leaves the point to the runtime loop's full probe. */
template <int P>
__device__ __forceinline__ uint64_t fast_key(const Stencil &st)
{
  constexpr int ox = P % 3 - 1, oy = (P / 3) % 3 - 1, oz = P / 9 - 1;
  uint64_t q = st.k0;
  if (ox > 0) q += st.sx;
  if (ox < 0) q -= st.sx;
  if (oy > 0) q += st.sy;
  if (oy < 0) q -= st.sy;
  if (oz > 0) q += st.sz;
  if (oz < 0) q -= st.sz;
  return q;
}

template <int L>
struct FastRec;
template <>
struct FastRec<kOccDense> {
  using T = uint2;
};
template <>
struct FastRec<kOccHash> {
  using T = uint4;  // {tag lo, tag hi, start, bits}
};

template <int P, int L>
__device__ __forceinline__ void fast_issue(const KArgs &a, const Stencil &st, uint32_t need,
                                           typename FastRec<L>::T &r)
{
  const uint64_t q = fast_key<P>(st);
  const bool go = ((need & st.inrange) >> P) & 1u;
  if (L == kOccDense) {
    uint2 v = make_uint2(0, 0);
    if (go) v = ldg_rec(a.s, q);
    reinterpret_cast<uint2 &>(r) = v;
  } else {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (go) {
      const uint64_t b = q >> a.s.dir_shift;
      v = __ldg(reinterpret_cast<const uint4 *>(a.s.htab + hash_home(b, a.s.hmask)) + (b & 1));
    }
    reinterpret_cast<uint4 &>(r) = v;
  }
}

template <int P, int L>
__device__ __forceinline__ void fast_finish(const KArgs &a, Smem &sm, int warp, int lane,
                                            const Cell &c, const Stencil &st, uint32_t need,
                                            typename FastRec<L>::T rr, Marks &m, uint32_t &pend)
{
  if (!((need >> P) & 1u)) return;
  const uint64_t q = fast_key<P>(st);
  const uint32_t bit = uint32_t(q) & 31u;
  uint2 r;
  if (L == kOccDense) {
    r = reinterpret_cast<const uint2 &>(rr);
  } else {
    const uint4 e = reinterpret_cast<const uint4 &>(rr);
    const bool mine = (uint64_t(e.x) | (uint64_t(e.y) << 32)) == (q >> a.s.dir_shift) + 1;
    r = mine ? make_uint2(e.z, e.w) : make_uint2(0, 0);
  }
  if ((r.y >> bit) & 1u) {  // (an out-of-range point has r = 0: a miss)
    constexpr int ox = P % 3 - 1, oy = (P / 3) % 3 - 1, oz = P / 9 - 1;
    constexpr bool lower = ox < 0 || (ox == 0 && (oy < 0 || (oy == 0 && oz < 0)));
    if (lower)
      m.low |= 1u << P;
    else
      m.ok |= 1u << P;
    sm.id[warp][P][lane] = r.x + uint32_t(__popc(r.y & ((1u << bit) - 1u)));
    sm.lev[warp][P][lane] = uint8_t(c.level);
    return;
  }
  pend |= 1u << P;
}

template <int L, int... Ps, size_t... I>
__device__ __forceinline__ void fast_batch_impl(std::index_sequence<I...>, const KArgs &a,
                                                Smem &sm, int warp, int lane, const Cell &c,
                                                const Stencil &st, uint32_t need, Marks &m,
                                                uint32_t &pend)
{
  typename FastRec<L>::T r[sizeof...(Ps)];
  (fast_issue<Ps, L>(a, st, need, r[I]), ...);
  (fast_finish<Ps, L>(a, sm, warp, lane, c, st, need, r[I], m, pend), ...);
}

template <int L, int... Ps>
__device__ __forceinline__ void fast_batch(const KArgs &a, Smem &sm, int warp, int lane,
                                           const Cell &c, const Stencil &st, uint32_t need,
                                           Marks &m, uint32_t &pend)
{
  fast_batch_impl<L, Ps...>(std::make_index_sequence<sizeof...(Ps)>{}, a, sm, warp, lane, c, st,
                            need, m, pend);
}

/// index of the r-th (0-based) set bit of mask (mask has more than r bits)
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t mask, uint32_t r)
{
  uint32_t pos = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const uint32_t cand = pos + uint32_t(step);
    const uint32_t below = cand >= 32 ? mask : mask & ((1u << cand) - 1u);
    if (uint32_t(__popc(below)) <= r) pos = cand;
  }
  return pos;
}

/*! resolve the stencil points in `todo` into the marks (classes of
    dual.cpp:60-67: missing, finer, lower key, ok), with the warp's work
    compacted: the (lane, point) pairs of every lane's `todo` are numbered by
    a warp scan and dealt out one per lane, so the lookups (hint level +
    finer, then the coarser levels in snap's order, locator.cpp:122-134) run
    with every lane busy instead of the warp looping as long as its busiest
    lane (the per-lane loop it replaced: C4 extraction 60.1 -> 44.9 ms).  A worker reads its owner's stencil
    through shuffles, writes the result into the owner's shared-memory column
    and ORs the point's class into the owner's mark words. */
template <bool DIGITS>
__device__ __forceinline__ void resolve_marks_compact(const KArgs &a, Smem &sm, int warp,
                                                      int lane, const Cell &c,
                                                      const Stencil &st, uint32_t self,
                                                      uint32_t todo, Marks &m)
{
  if (!__any_sync(kFull, todo != 0)) return;
  const uint32_t cnt = __popc(todo);
  const uint32_t incl = warp_incl_scan(cnt);
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  dbg_sum(a.s, kDbgRuntime, cnt);
  sm.mk[warp][lane] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  for (uint32_t base = 0; base < total; base += 32) {
    const uint32_t i = base + uint32_t(lane);
    // owner = the number of lanes whose inclusive count is <= i
    uint32_t owner = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
      const uint32_t v = __shfl_sync(kFull, incl, int(owner) + step - 1);
      if (v <= i) owner += uint32_t(step);
    }
    owner = owner > 31u ? 31u : owner;
    const bool have = i < total;
    const uint32_t otodo = __shfl_sync(kFull, todo, int(owner));
    const uint32_t oexcl = __shfl_sync(kFull, incl - cnt, int(owner));
    Stencil ost;
    ost.k0 = shfl_u64(st.k0, int(owner));
    ost.sx = shfl_u64(st.sx, int(owner));
    ost.sy = shfl_u64(st.sy, int(owner));
    ost.sz = shfl_u64(st.sz, int(owner));
    ost.inrange = __shfl_sync(kFull, st.inrange, int(owner));
    const int olevel = __shfl_sync(kFull, c.level, int(owner));
    const uint32_t oself = __shfl_sync(kFull, self, int(owner));
    if (!have) continue;
    const int p = int(nth_set_bit(otodo, i - oexcl));
    uint64_t q[1] = {stencil_key<DIGITS>(ost, p)};
    const bool v[1] = {((ost.inrange >> p) & 1u) != 0};
    int64_t out[1] = {-1};
    int lvl[1] = {olevel};
    batch_find<1, true>(a.s, q, v, out, lvl);
    const uint32_t coarser = a.g.level_mask & ~((2u << olevel) - 1);
    if (out[0] < 0 && coarser) {
      const Hit h = probe_coarser(a, olevel, ost, p, coarser);
      out[0] = h.id;
      lvl[0] = h.level;
    }
    sm.id[warp][p][owner] = uint32_t(out[0]);
    sm.lev[warp][p][owner] = uint8_t(lvl[0]);
    const uint32_t bit = 1u << p;
    unsigned int *mk = &sm.mk[warp][owner].x;
    if (out[0] < 0)
      atomicOr(mk + 1, bit);
    else if (lvl[0] < olevel)
      atomicOr(mk + 2, bit);
    else if (lvl[0] == olevel && uint32_t(out[0]) < oself)
      atomicOr(mk + 3, bit);
    else
      atomicOr(mk, bit);
  }
  __syncwarp();
  const uint4 w = sm.mk[warp][lane];
  m.ok |= w.x;
  m.miss |= w.y;
  m.fin |= w.z;
  m.low |= w.w;
  __syncwarp();
}

template <bool EMIT_DUAL, bool EMIT_TRI, bool F32, int LOOKUP>
#ifndef AMRX_MINB
#define AMRX_MINB 1  // CTAs per SM the register budget is sized for (64 regs at 1024 threads)
#endif
#ifndef AMRX_MINB_HASH
#define AMRX_MINB_HASH 1
#endif
__global__ void __launch_bounds__(kThreads, LOOKUP == kOccHash ? AMRX_MINB_HASH : AMRX_MINB)
extract_kernel(const __grid_constant__ KArgs a)
{
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem &sm = *reinterpret_cast<Smem *>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool kNeighbours = LOOKUP == kOccHash;  // see the k-neighbour shortcut below
  if (EMIT_TRI) {
    // indexed by the slot-numbered corner mask directly (table_row applied
    // once here instead of per dual)
    for (int i = threadIdx.x; i < 256; i += kThreads)
      sm.mc_rows[i] = c_mc_rows[table_row(uint32_t(i))];
    __syncthreads();
  }

  if (lane < 8) sm.acc[warp][lane] = 0;
  if (lane < 4) sm.chunk[warp][lane] = 0;
  __syncwarp();
  uint32_t err = 0;

  // tiles from an atomic ticket: the warps' positions stay within a few
  // thousand tiles of each other, so the lookups share one compact L2
  // working set (a static interleaved assignment drifts apart: 19% slower)
  for (;;) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1ull);
    tk = __shfl_sync(kFull, tk, 0);
    if (tk >= a.tile_limit) break;
    const uint32_t tile = uint32_t(tk);
    dbg_add(a.s, kDbgTiles);

    const uint64_t cell_s = a.cell_begin + uint64_t(tile) * kTileCells + lane;
    const bool working = cell_s < a.cell_end;
    const bool valid = working && cell_s < a.s.n;
    const uint64_t cell = valid ? cell_s : 0;
    const uint32_t self = uint32_t(cell);
    const uint64_t kself =
      valid && AMRX_BOUND(cell < a.s.n, kChkKey) ? ldg_u64(a.s.keys + cell) : 0;
    // the sorted neighbours of the tile's end lanes (the others are lanes)
    uint64_t kedge = 0;
    if (kNeighbours && valid && lane == 0 && cell > 0) kedge = ldg_u64(a.s.keys + cell - 1);
    if (kNeighbours && valid && lane == 31 && cell + 1 < a.s.n)
      kedge = ldg_u64(a.s.keys + cell + 1);
    const Cell c = unpack(a.g, kself);
    const Stencil st = make_stencil(a.g, kself, c.level);

    uint32_t accepted = 0, reasons = 0;
    {
      Marks m{0, 0, 0, 0};
      uint32_t need = working ? kCorner0Points : 0;
      if (working && a.unique) {
        // the cell's own key can only find the cell itself (no duplicates)
        m.ok |= 1u << 13;
        sm.id[warp][13][lane] = self;
        sm.lev[warp][13][lane] = uint8_t(c.level);
        need &= ~(1u << 13);
      }
      if (kNeighbours) {
        // points 4 and 22, (0, 0, -w) and (0, 0, +w): when the sorted
        // neighbour's key is the stencil key, the lookup would find exactly
        // that cell (position self -1 / +1, the cell's level) -- resolved
        // without one; a lower key (rule #3) and an ok corner.  Hashed
        // records only: a hashed lookup costs more than the shortcut (deep
        // extraction 28.0 -> 27.2 ms), a dense one less (C4 43.8 -> 44.0,
        // C5 14.0 -> 14.8)
        const uint64_t up = __shfl_up_sync(kFull, kself, 1);
        const uint64_t dn = __shfl_down_sync(kFull, kself, 1);
        const uint64_t kp = lane == 0 ? kedge : up, kn = lane == 31 ? kedge : dn;
        const bool have_p = lane > 0 || cell > 0, have_n = lane < 31 || cell + 1 < a.s.n;
        if (working && a.unique) {
          if (have_p && ((st.inrange >> 4) & 1u) && kp == stencil_key(st, 4)) {
            m.low |= 1u << 4;
            sm.id[warp][4][lane] = self - 1;
            sm.lev[warp][4][lane] = uint8_t(c.level);
            need &= ~(1u << 4);
          }
          if (have_n && ((st.inrange >> 22) & 1u) && kn == stencil_key(st, 22)) {
            m.ok |= 1u << 22;
            sm.id[warp][22][lane] = self + 1;
            sm.lev[warp][22][lane] = uint8_t(c.level);
          }
        }
      }
      // round 0: every candidate's corner 0 ({-w,0}^3); round 1: the
      // survivors' other corners (one inlined copy of the column code)
      uint32_t alive = 0;
#pragma unroll 1
      for (int round = 0; round < 2; round++) {
        if (round == 1) {
          // candidate delta lives on iff its corner 0 (point base_of(delta))
          // is acceptable; a dead one's reason is its corner 0's (corner
          // order, dual.cpp:49-67); corner-0 points map one-to-one to
          // candidates
#pragma unroll
          for (int delta = 0; delta < 8; delta++)
            alive |= ((m.ok >> base_of(delta)) & 1u) << delta;
          reasons = (uint32_t(__popc(m.miss & kCorner0Points)) << 8) |
                    (uint32_t(__popc(m.fin & kCorner0Points)) << 16) |
                    (uint32_t(__popc(m.low & kCorner0Points)) << 24);
          need = 0;
          for (uint32_t mm = alive; mm; mm &= mm - 1) need |= kCube << base_of(__ffs(mm) - 1);
          need &= ~m.resolved();
        }
        if (LOOKUP != kOccNone) {
          // the points every cell of a uniform region needs -- all
          // candidates' corner 0 in round 0, candidate 7's cube in round 1 --
          // with compile-time offsets; the rest and every miss go through
          // the runtime loop
          constexpr int L = LOOKUP == kOccHash ? kOccHash : kOccDense;
          uint32_t pend = 0;
          if (round == 0) {
            dbg_sum(a.s, kDbgFastNeed, __popc(need & kFast0));
            fast_batch<L, 0, 1, 3, 4, 9, 10, 12>(a, sm, warp, lane, c, st, need, m, pend);
            need &= ~kFast0;
          } else if (__any_sync(kFull, (need & kFast1) != 0)) {
            dbg_sum(a.s, kDbgFastNeed, __popc(need & kFast1));
            fast_batch<L, 14, 16, 17, 22, 23, 25, 26>(a, sm, warp, lane, c, st, need, m, pend);
            need &= ~kFast1;
          }
          dbg_sum(a.s, kDbgFastPend, __popc(pend));
          need |= pend;
        }
        resolve_marks_compact<EMIT_TRI>(a, sm, warp, lane, c, st, self, need, m);
      }
      // corners in order d = 0..7 are ascending stencil points, so the
      // first failing corner is the lowest failing bit
      const uint32_t res = m.resolved();
      for (uint32_t mm = alive; mm; mm &= mm - 1) {
        const int delta = __ffs(mm) - 1;
        const uint32_t cube = kCube << base_of(delta);
        if (cube & ~res) err |= 2u;  // cannot happen: every corner resolved
        const uint32_t bad = cube & ~m.ok;
        if (!bad) {
          accepted |= 1u << delta;
          reasons += 1u;
        } else {
          const uint32_t b = bad & (0u - bad);
          reasons += (m.miss & b) ? (1u << 8) : (m.fin & b) ? (1u << 16) : (1u << 24);
        }
      }
    }

    // ---- pass 1 + pass 2 fused.  No waiting on other tiles: the tile's
    // block goes to this warp's private chunk of the staging arena and
    // (offset, count) to the tile table; reorder_kernel later moves blocks
    // into candidate order (the reference's prefix sum, pipeline.cpp:109-114).
    const uint32_t nd = __popc(accepted);
    uint32_t upper = 0, cross = 0, ntabs = 0;
    if (EMIT_TRI) {
      // duals whose 8 corners all classify alike carry no triangle: decide
      // from the sign bits (value > iso, contour.cpp:22-28) before touching
      // the FP64 scalars; the case row's table count bounds the triangles
      for (uint32_t m = accepted; m; m &= m - 1) {
        const int delta = __ffs(m) - 1;
        uint32_t mask = 0;
#pragma unroll
        for (int d = 0; d < 8; d++) {
          const uint32_t id = sm.id[warp][point_of(delta, d)][lane];
          mask |= ((__ldg(a.above + (id >> 5)) >> (id & 31)) & 1u) << d;
        }
        if (mask != 0 && mask != 0xffu) {
          const uint32_t nt = uint32_t(sm.mc_rows[mask] & 15);
          cross |= 1u << delta;
          ntabs |= nt << (4 * delta);
          upper += nt;
        }
      }
    }
    // tile totals into the warp's accumulators (16-bit fields cannot carry:
    // 32 lanes x 8 candidates)
    {
      const uint32_t r01 = __reduce_add_sync(kFull, (reasons & 0xffu) | ((reasons & 0xff00u) << 8));
      const uint32_t r23 = __reduce_add_sync(kFull, ((reasons >> 16) & 0xffu) | ((reasons >> 24) << 16));
      const uint32_t tnd = __reduce_add_sync(kFull, nd);
      if (lane == 0) {
        sm.acc[warp][0] += r01 & 0xffffu;
        sm.acc[warp][1] += r01 >> 16;
        sm.acc[warp][2] += r23 & 0xffffu;
        sm.acc[warp][3] += r23 >> 16;
        sm.acc[warp][4] += tnd;
      }
    }
    __syncwarp();
    if (EMIT_DUAL) {
      const uint32_t incl = warp_incl_scan(nd);
      const uint32_t agg = __shfl_sync(kFull, incl, 31);
      const uint64_t base = reserve(&sm.chunk[warp][0], agg, kDualChunk, a.out + 8,
                                    a.dual_guard, a.ticket, a.stop_at) +
                            (incl - nd);
      if (lane == 0) {
        a.tile_dual_cnt[tile] = agg;
        a.tile_dual_off[tile] = base;
      }
      uint32_t k = 0;
      for (uint32_t m = accepted; m; m &= m - 1, k++) {
        const int delta = __ffs(m) - 1;
        const uint64_t slot = base + k;
        if (slot >= a.dual_cap) continue;
        uint32_t ids[8];
        const uint32_t ib = uint32_t(a.s.id_base);  // global ids (partition)
#pragma unroll
        for (int d = 0; d < 8; d++) ids[d] = sm.id[warp][point_of(delta, d)][lane] + ib;
        uint4 *dst = reinterpret_cast<uint4 *>(a.corners + slot * 8);
        dst[0] = make_uint4(ids[0], ids[1], ids[2], ids[3]);
        dst[1] = make_uint4(ids[4], ids[5], ids[6], ids[7]);
        a.tasks[slot] = uint64_t(int64_t(cell) + a.s.id_base) * 8 + uint64_t(delta);
      }
    }
    if (EMIT_TRI) {
      // reserve the table's upper bound for the tile, then queue its
      // crossing duals (candidate order: lane, then delta) with their slots
      // for mc_jobs_kernel, which subtracts what slivers drop
      const uint32_t incl = warp_incl_scan(upper);
      const uint32_t agg_up = __shfl_sync(kFull, incl, 31);
      const uint64_t block = reserve(&sm.chunk[warp][2], agg_up, kTriChunk, a.out + 9,
                                     a.tri_guard, a.ticket, a.stop_at);
      const uint32_t nc = __popc(cross);
      const uint32_t incl_c = warp_incl_scan(nc);
      const uint32_t total = __shfl_sync(kFull, incl_c, 31);
      unsigned long long jb = 0;
      if (lane == 0) {
        a.tile_tri_cnt[tile] = agg_up;
        a.tile_tri_up[tile] = agg_up;
            a.tile_tri_off[tile] = block;
        if (total) {
          jb = atomicAdd(a.out + 10, (unsigned long long)total);
          if (jb + total > a.job_guard) stop_round(a.ticket, a.stop_at);
        }
      }
      jb = __shfl_sync(kFull, jb, 0);
      uint64_t at = block + (incl - upper), j = jb + (incl_c - nc);
      for (uint32_t mm = cross; mm; mm &= mm - 1, j++) {
        const int delta = __ffs(mm) - 1;
        const uint32_t nt = (ntabs >> (4 * delta)) & 15u;
        if (j < a.job_cap) {
          McJob &job = a.jobs[j];
          uint32_t ids[8];
          uint8_t lvs[8];
#pragma unroll
          for (int d = 0; d < 8; d++) {
            ids[d] = sm.id[warp][point_of(delta, d)][lane];
            lvs[d] = sm.lev[warp][point_of(delta, d)][lane];
          }
          uint4 *q = reinterpret_cast<uint4 *>(&job);
          q[0] = make_uint4(ids[0], ids[1], ids[2], ids[3]);
          q[1] = make_uint4(ids[4], ids[5], ids[6], ids[7]);
          q[2] = make_uint4(uint32_t(kself), uint32_t(kself >> 32), uint32_t(at),
                            uint32_t(at >> 32));
          q[3] = make_uint4(uint32_t(lvs[0]) | uint32_t(lvs[1]) << 8 | uint32_t(lvs[2]) << 16 |
                              uint32_t(lvs[3]) << 24,
                            uint32_t(lvs[4]) | uint32_t(lvs[5]) << 8 | uint32_t(lvs[6]) << 16 |
                              uint32_t(lvs[7]) << 24,
                            tile, uint32_t(delta) | nt << 8);
        }
        at += nt;
      }
    }
    __syncwarp();
  }

  // per-warp totals -> global
  err = __reduce_or_sync(kFull, err);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 7; i++)
      if (sm.acc[warp][i]) atomicAdd(a.out + i, sm.acc[warp][i]);
    if (err) atomicOr(a.out + 7, (unsigned long long)err);
  }
}

// ------------------------------------------------------- query kernels

/*! snap (locator.cpp:122-134) for one point per lane, warp-cooperatively:
    probe sequence = hint (if in [0,30]) then present levels finest first
    skipping the hint */
__device__ int64_t warp_snap(const SearchCtx &s, const KeyGeom &g, bool active,
                             int64_t px, int64_t py, int64_t pz, int32_t hint,
                             uint64_t *win)
{
  int64_t result = -1;
  bool pend = active;
  int probe = (hint >= 0 && hint <= kMaxLevel) ? -1 : 0;
  while (__any_sync(kFull, pend)) {
    if (probe >= 0)
      while (probe < g.nlevels && g.levels[probe] == hint) probe++;
    const bool have = pend && (probe < 0 || probe < g.nlevels);
    const int L = probe < 0 ? hint : (have ? g.levels[probe] : 0);
    uint64_t q[1];
    bool v[1];
    int64_t o[1] = {-1};
    int l1[1];
    v[0] = have && query_key(g, px, py, pz, L, q[0]);
    warp_find<1, false>(s, q, v, o, l1, win);
    if (pend && v[0] && o[0] >= 0) {
      result = o[0];
      pend = false;
    }
    if (!have) pend = false;
    probe++;
  }
  return result;
}

__global__ void __launch_bounds__(kThreads)
find_exact_kernel(const SearchCtx s, const KeyGeom g,
                  const int4 *__restrict__ cells, uint64_t n,
                  int64_t *__restrict__ out)
{
  __shared__ uint64_t win[kWarps][kWin];
  const int warp = threadIdx.x >> 5;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
       base < n; base += stride) {
    const uint64_t r = base + (threadIdx.x & 31);
    const bool in = r < n;
    int4 cc = in ? cells[r] : make_int4(0, 0, 0, 0);
    uint64_t q[1];
    bool v[1];
    int64_t o[1] = {-1};
    // find_exact matches the full key: the anchor must be the stored one
    v[0] = in && cc.w >= 0 && cc.w <= kMaxLevel &&
           anchor_mask(cc.x, cc.w) == cc.x &&
           anchor_mask(cc.y, cc.w) == cc.y &&
           anchor_mask(cc.z, cc.w) == cc.z &&
           query_key(g, cc.x, cc.y, cc.z, cc.w, q[0]);
    int l1[1];
    warp_find<1, false>(s, q, v, o, l1, win[warp]);
    if (in) out[r] = v[0] && o[0] >= 0 ? o[0] + s.id_base : -1;
  }
}

__global__ void __launch_bounds__(kThreads)
snap_kernel(const SearchCtx s, const KeyGeom g,
            const int64_t *__restrict__ points, const int32_t *__restrict__ hints,
            int32_t hint_all, uint64_t n, int64_t *__restrict__ out)
{
  __shared__ uint64_t win[kWarps][kWin];
  const int warp = threadIdx.x >> 5;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
       base < n; base += stride) {
    const uint64_t r = base + (threadIdx.x & 31);
    const bool in = r < n;
    const int64_t px = in ? points[3 * r] : 0, py = in ? points[3 * r + 1] : 0,
                  pz = in ? points[3 * r + 2] : 0;
    const int32_t h = in ? (hints ? hints[r] : hint_all) : -1;
    const int64_t res = warp_snap(s, g, in, px, py, pz, h, win[warp]);
    if (in) out[r] = res >= 0 ? res + s.id_base : -1;
  }
}

/// try_build_dual (dual.cpp:41-72) for one task (cell*8+delta) per lane
__global__ void __launch_bounds__(kThreads)
try_build_kernel(const SearchCtx s, const KeyGeom g,
                 const uint64_t *__restrict__ tasks, uint64_t n,
                 uint8_t *__restrict__ reject, uint32_t *__restrict__ corners)
{
  __shared__ uint64_t win[kWarps][kWin];
  const int warp = threadIdx.x >> 5;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
       base < n; base += stride) {
    const uint64_t r = base + (threadIdx.x & 31);
    bool live = r < n;
    const uint64_t task = live ? tasks[r] : 0;
    const uint64_t cell = uint64_t(int64_t(task >> 3) - s.id_base);  // local position
    const int delta = int(task & 7);
    live = live && cell < s.n;
    const Cell c = unpack(g, live ? ldg_u64(s.keys + cell) : 0);
    const int64_t w = int64_t(1) << c.level;
    const int64_t bx = c.i - ((delta & 1) ? 0 : w);
    const int64_t by = c.j - ((delta & 2) ? 0 : w);
    const int64_t bz = c.k - ((delta & 4) ? 0 : w);
    uint32_t code = live ? 0u : 1u;
    uint32_t ids[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool going = live;
    for (int d = 0; d < 8; d++) {
      const int64_t hit =
        warp_snap(s, g, going, bx + ((d & 1) ? w : 0), by + ((d & 2) ? w : 0),
                  bz + ((d & 4) ? w : 0), c.level, win[warp]);
      if (going) {
        if (hit < 0) {
          code = kMiss;
          going = false;
        } else {
          const int hl = unpack(g, ldg_u64(s.keys + hit)).level;
          if (hl < c.level) {
            code = kFiner;
            going = false;
          } else if (hl == c.level && uint64_t(hit) < cell) {
            code = kLower;
            going = false;
          } else {
            ids[d] = uint32_t(hit);
          }
        }
      }
    }
    if (r < n) {
      reject[r] = uint8_t(code);
      if (corners)
        for (int d = 0; d < 8; d++)
          corners[8 * r + d] = code == 0 ? ids[d] + uint32_t(s.id_base) : 0;
    }
  }
}

int grid_query(uint64_t n)
{
  const uint64_t blocks = (n + kThreads - 1) / kThreads;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(blocks,
                                                       uint64_t(device_sm_count()) * 8)));
}

template <bool D, bool T, bool F, int L>
void launch_extract(const KArgs &k, int grid, cudaStream_t st)
{
  ensure_smem_attr(reinterpret_cast<const void *>(extract_kernel<D, T, F, L>), sizeof(Smem));
  extract_kernel<D, T, F, L><<<grid, kThreads, sizeof(Smem), st>>>(k);
  AMRX_LAUNCH_CHECK();
}

template <bool D, bool T, bool F, int L>
int occupancy_grid()
{
  static int per_sm[64] = {0};  // per device
  int dev = 0;
  AMRX_CUDA(cudaGetDevice(&dev));
  int &ps = per_sm[dev & 63];
  if (!ps) {
    ensure_smem_attr(reinterpret_cast<const void *>(extract_kernel<D, T, F, L>), sizeof(Smem));
    AMRX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &ps, extract_kernel<D, T, F, L>, kThreads, sizeof(Smem)));
    ps = std::max(1, ps);
  }
  return ps * device_sm_count();
}

/*! the extraction kernel variant for a request: dual mesh, or the soup in
    f64 / f32, times the lookup structure's fast path (none, dense records,
    hashed records) -- fn(kernel tag) with the template arguments bound */
template <typename Fn>
void with_variant(bool D, bool F, int occ, Fn &&fn)
{
  const auto by_lookup = [&](auto d, auto f) {
    constexpr bool Dv = decltype(d)::value, Fv = decltype(f)::value;
    if (occ == kOccDense)
      fn(std::integral_constant<int, kOccDense>{}, d, f);
    else if (occ == kOccHash)
      fn(std::integral_constant<int, kOccHash>{}, d, f);
    else
      fn(std::integral_constant<int, kOccNone>{}, d, f);
    (void)Dv;
    (void)Fv;
  };
  if (D)
    by_lookup(std::true_type{}, std::false_type{});
  else if (F)
    by_lookup(std::false_type{}, std::true_type{});
  else
    by_lookup(std::false_type{}, std::false_type{});
}

}  // namespace

namespace {

/// grow a device buffer to `need` bytes keeping its first `keep` bytes
void grow_keep(DevBuf &b, size_t need, size_t keep, cudaStream_t st)
{
  if (b.ptr && b.bytes >= need) return;
  DevBuf n;
  n.reserve(std::max(need, b.bytes + b.bytes / 2), st);
  if (keep && b.ptr) AMRX_CUDA(cudaMemcpyAsync(n.ptr, b.ptr, keep, cudaMemcpyDeviceToDevice, st));
  std::swap(b.ptr, n.ptr);
  std::swap(b.bytes, n.bytes);
  std::swap(b.stream, n.stream);
}

// staging caps per round (rounds make any size correct; these bound memory)
constexpr uint64_t kStageBytes = uint64_t(16) << 30;
constexpr uint64_t kJobCap = uint64_t(64) << 20;  // 4 GB of McJob

}  // namespace

std::atomic<uint64_t> g_round_limit{0};  // amrx_debug_round_limit

/*! The extraction in rounds.  Every round runs the search
    kernel over the next tiles in ticket order until a staging buffer is
    nearly full (stop_round), marching cubes over the round's crossing
    duals, then the exclusive scan of the round's tile counts and the
    reorder of its tiles into candidate order after everything earlier --
    the reference's pass 1 / prefix sum / pass 2 (pipeline.cpp:80-146) with
    the search run once.  The staging sizes only decide how many rounds a
    call takes, never the result, and nothing is ever run twice. */
ExtractResult run_extract(const ExtractRequest &r, cudaStream_t st)
{
  ExtractScratch x;
  ExtractResult res{};
  const uint64_t cells = r.cell_end > r.cell_begin ? r.cell_end - r.cell_begin : 0;
  const uint64_t tiles = (cells + kTileCells - 1) / kTileCells;
  const bool D = r.emit_dual, T = r.emit_tri, F = r.tri_f32;
  if (D == T) throw std::invalid_argument("extract: exactly one of dual mesh / soup per call");
  const int occ = r.s.rec ? kOccDense : r.s.htab ? kOccHash : kOccNone;
  int grid = 1;
  with_variant(D, F, occ, [&](auto l, auto d, auto f) {
    grid = occupancy_grid<decltype(d)::value, !decltype(d)::value, decltype(f)::value,
                          decltype(l)::value>();
  });
  grid = int(std::max<uint64_t>(1, std::min<uint64_t>(grid, (tiles + kWarps - 1) / kWarps)));
  if (g_round_limit.load()) grid = 1;  // testing hook: few tiles in flight, many rounds
  const uint64_t warps = uint64_t(grid) * kWarps;

  // control block | tile tables (count u32 + staging offset u64 + final
  // offset u64, per output kind)
  x.ctl.reserve(256, st);
  x.tiles.reserve(size_t(tiles + 1) * 48 + 64, st);
  auto *ctl = x.ctl.as<unsigned long long>();
  auto *tb = x.tiles.as<unsigned char>();
  uint32_t *dual_cnt = reinterpret_cast<uint32_t *>(tb);
  uint32_t *tri_cnt = dual_cnt + (tiles + 1);
  uint32_t *tri_up = tri_cnt + (tiles + 1);
  uint64_t *dual_off = reinterpret_cast<uint64_t *>(tb + ((3 * (tiles + 1) * 4 + 15) & ~size_t(15)));
  uint64_t *tri_off = dual_off + (tiles + 1);
  uint64_t *final_off = tri_off + (tiles + 1);
  AMRX_CUDA(cudaMemsetAsync(ctl, 0, 256, st));
  AMRX_CUDA(cudaMemsetAsync(ctl + 17, 0xff, 8, st));  // stop_at: none
  if (tiles) AMRX_CUDA(cudaMemsetAsync(tb, 0, size_t(tiles + 1) * 12, st));

  const bool grow = r.grow_a != nullptr;
  const bool want_d = D && (r.corners || grow);
  const bool want_t = T && (r.xyz || grow);
  const uint64_t out_d_cap = grow ? ~0ull : r.dual_cap;
  const uint64_t out_t_cap = grow ? ~0ull : r.tri_cap;
  const int tri_words = F ? 9 : 18;  // 32-bit words per triangle
  // guard headroom (stop_round): the tiles in flight claim at most one
  // chunk each; 3 chunks per warp
  const uint64_t hd = 3 * warps * kDualChunk, ht = 3 * warps * kTriChunk, hj = 3 * warps * 256;
  const uint64_t lim = g_round_limit.load() ? g_round_limit.load() : ~0ull;
  const uint64_t dual_stage =
    want_d ? hd + std::min<uint64_t>({out_d_cap, cells + cells / 4 + 1024, kStageBytes / 40, lim})
           : 0;
  const uint64_t tri_stage =
    want_t ? ht + std::min<uint64_t>({out_t_cap / 8 * 9 + 1024, 3 * cells + 1024,
                                      kStageBytes / uint64_t(tri_words * 4), lim})
           : 0;
  const uint64_t job_cap =
    want_t ? hj + std::min<uint64_t>({cells / 4 + 1024, kJobCap, lim}) : 0;
  if (dual_stage) {
    x.stage_a.reserve(dual_stage * 32, st);
    x.stage_b.reserve(dual_stage * 8, st);
  }
  if (tri_stage) x.stage_a.reserve(tri_stage * tri_words * 4, st);
  if (job_cap) x.jobs.reserve(job_cap * sizeof(McJob), st);

  KArgs k;
  k.s = r.s;
  k.g = r.g;
  k.unique = r.unique;
  k.above = nullptr;
  if (T) {
    const uint64_t words = (r.s.n + 31) / 32;
    x.bits.reserve(words * 4 + 64, st);
    k.above = x.bits.as<uint32_t>();
    const int bgrid =
      int(std::min<uint64_t>((words + 7) / 8, uint64_t(device_sm_count()) * 16));
    sign_bits_kernel<<<std::max(1, bgrid), 256, 0, st>>>(r.scal, r.s.n, r.iso,
                                                         x.bits.as<uint32_t>());
    AMRX_LAUNCH_CHECK();
    res.launches += 1;
  }
  k.scal = r.scal;
  k.cell_begin = r.cell_begin;
  k.cell_end = r.cell_end;
  k.num_tiles = uint32_t(tiles);
  k.iso = r.iso;
  k.corners = dual_stage ? x.stage_a.as<uint32_t>() : nullptr;
  k.tasks = dual_stage ? x.stage_b.as<uint64_t>() : nullptr;
  k.dual_cap = dual_stage;
  k.xyz = tri_stage ? x.stage_a.ptr : nullptr;
  k.tri_cap = tri_stage;
  k.tile_dual_cnt = dual_cnt;
  k.tile_dual_off = dual_off;
  k.tile_tri_cnt = tri_cnt;
  k.tile_tri_up = tri_up;
  k.tile_tri_off = tri_off;
  k.jobs = job_cap ? x.jobs.as<McJob>() : nullptr;
  k.job_cap = job_cap;
  k.dual_guard = dual_stage - std::min(dual_stage, hd);
  k.tri_guard = tri_stage - std::min(tri_stage, ht);
  k.job_guard = job_cap - std::min(job_cap, hj);
  k.out = ctl;
  k.ticket = ctl + 16;
  k.stop_at = ctl + 17;
  static const bool debug = std::getenv("AMRX_DEBUG_COUNTERS") != nullptr;
  k.s.dbg = debug ? ctl + 18 : nullptr;  // ctl holds 32 u64

  McArgs m;
  m.g = k.g;
  m.scal = k.scal;
  m.iso = k.iso;
  m.jobs = k.jobs;
  m.job_cap = k.job_cap;
  m.xyz = k.xyz;
  m.tri_cap = k.tri_cap;
  m.tile_tri_cnt = k.tile_tri_cnt;
  m.out = ctl;

  // host output: each round is reordered into a device buffer and copied
  // down on a side stream while the next round runs (two buffers)
  cudaStream_t cp = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr};
  WsBuf out_a(kWsOutA), out_b(kWsOutB), out_c(kWsScratch);
  struct Cleanup {
    cudaStream_t s;
    cudaEvent_t *e;
    ~Cleanup()
    {
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
      for (int i = 0; i < 2; i++)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } cleanup{nullptr, copied};
  if (r.final_host && (want_d || want_t)) {
    AMRX_CUDA(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
    cleanup.s = cp;
    for (int i = 0; i < 2; i++)
      AMRX_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
  }

  cudaEvent_t e0, e1, e2;
  AMRX_CUDA(cudaEventCreate(&e0));
  AMRX_CUDA(cudaEventCreate(&e1));
  AMRX_CUDA(cudaEventCreate(&e2));
  unsigned long long h[18] = {}, prev[8] = {};
  uint64_t t0 = 0, base_d = 0, base_t = 0;
#ifndef AMRX_REORDER_BLOCKS
#define AMRX_REORDER_BLOCKS 256  // C4 triangle reorder: 16 4.77 ms, 128 3.91, 256 3.78, 1024 3.74; C3 favours 128-256
#endif
  const int rgrid_cap = device_sm_count() * AMRX_REORDER_BLOCKS;  // blocks per SM
  for (int round = 0; t0 < tiles; round++) {
    // the round's tile limit: host output starts with small rounds (1/64,
    // then 1/32 of the tiles) so the first download starts early
    uint64_t limit = tiles;
    if (r.stream_rounds) {
      const uint64_t first = tiles / 64, second = tiles * 3 / 64;
      if (round == 0 && first > 0) limit = first;
      else if (t0 < second) limit = second;
      else limit = std::min(tiles, t0 + (tiles - second + 7) / 8);
      limit = std::max(limit, t0 + 1);
    }
    if (round) {  // fresh cursors, the ticket at the first open tile
      const unsigned long long reset[10] = {0, 0, 0, 0, 0, 0, 0, 0, t0, ~0ull};
      AMRX_CUDA(cudaMemcpyAsync(ctl + 8, reset, sizeof reset, cudaMemcpyHostToDevice, st));
    }
    k.tile_limit = limit;
    NvtxRange nvtx_round("extraction round");
    AMRX_CUDA(cudaEventRecord(e0, st));
    with_variant(D, F, occ, [&](auto l, auto d, auto f) {
      launch_extract<decltype(d)::value, !decltype(d)::value, decltype(f)::value,
                     decltype(l)::value>(k, grid, st);
    });
    res.launches += 1;
    if (T && tri_stage) {
#ifndef AMRX_MC_GRID_THREADS
#define AMRX_MC_GRID_THREADS 16384  // threads-worth of blocks per SM: C4 marching cubes 10.18 (2048) -> 9.50 ms, C2 2.54 -> 2.43 (65536: C4 9.30, C2 2.74)
#endif
      const int mgrid = device_sm_count() * std::max(1, AMRX_MC_GRID_THREADS / kMcThreads);
      if (F) {
        ensure_smem_attr(reinterpret_cast<const void *>(mc_jobs_kernel<true>), sizeof(McSmem));
        mc_jobs_kernel<true><<<mgrid, kMcThreads, sizeof(McSmem), st>>>(m);
      } else {
        ensure_smem_attr(reinterpret_cast<const void *>(mc_jobs_kernel<false>), sizeof(McSmem));
        mc_jobs_kernel<false><<<mgrid, kMcThreads, sizeof(McSmem), st>>>(m);
      }
      AMRX_LAUNCH_CHECK();
      res.launches += 1;
    }
    AMRX_CUDA(cudaEventRecord(e1, st));
    AMRX_CUDA(cudaMemcpyAsync(h, ctl, sizeof h, cudaMemcpyDeviceToHost, st));
    AMRX_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    AMRX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    res.ms += ms;
    const uint64_t stop = h[16] >= kStopTicket ? h[17] : h[16];
    const uint64_t t1 = std::min({limit, tiles, uint64_t(stop)});
    if (t1 <= t0 || h[8] > dual_stage || h[9] > tri_stage || h[10] > job_cap)
      throw std::runtime_error("extract: round " + std::to_string(round) +
                               " overran its staging or made no progress");
    const uint32_t nt = uint32_t(t1 - t0);
    const int rgrid = int(std::min<uint64_t>((nt + 7) / 8, uint64_t(rgrid_cap)));
    const uint64_t round_d = h[4] - prev[4], round_t = h[6] - prev[6];
    const int slot = round & 1;
    AMRX_CUDA(cudaEventRecord(e1, st));
    if (want_d && round_d) {
      res.launches += scan_exclusive_u32_u64(dual_cnt + t0, final_off + t0, nt, x.scan, st);
      uint32_t *dc = r.corners;
      uint64_t *dt = r.tasks;
      uint64_t dbase = base_d, dcap = r.dual_cap;
      if (grow) {
        grow_keep(*r.grow_a, (base_d + round_d) * 32, base_d * 32, st);
        grow_keep(*r.grow_b, (base_d + round_d) * 8, base_d * 8, st);
        dc = r.grow_a->as<uint32_t>();
        dt = r.grow_b->as<uint64_t>();
        dcap = ~0ull;
      } else if (r.final_host) {
        // this round's part into a device buffer (the copy that last used
        // it has drained), then down to host memory at its offset
        if (round >= 2) AMRX_CUDA(cudaStreamWaitEvent(st, copied[slot], 0));
        WsBuf &bc = slot ? out_b : out_a;
        bc.reserve(round_d * 32 + 16, st);
        dc = bc.as<uint32_t>();
        dt = nullptr;
        if (r.tasks) {
          out_c.reserve(round_d * 8 + 16, st);
          dt = out_c.as<uint64_t>();
        }
        dbase = 0;
        dcap = base_d < r.dual_cap ? std::min(round_d, r.dual_cap - base_d) : 0;
      }
      reorder_kernel<<<std::max(1, rgrid), 256, 0, st>>>(
        dual_cnt + t0, dual_off + t0, final_off + t0, nt, 8, x.stage_a.as<uint32_t>(), dc,
        dbase, dcap, dt ? 2 : 0, x.stage_b.as<uint32_t>(), reinterpret_cast<uint32_t *>(dt),
        dual_stage);
      AMRX_LAUNCH_CHECK();
      res.launches += 1;
      if (r.final_host && !grow && dcap) {
        AMRX_CUDA(cudaMemcpyAsync(r.corners + base_d * 8, dc, dcap * 32, cudaMemcpyDeviceToHost,
                                  st));
        if (r.tasks)  // (the tasks buffer is not double-buffered: copied in order)
          AMRX_CUDA(cudaMemcpyAsync(r.tasks + base_d, dt, dcap * 8, cudaMemcpyDeviceToHost, st));
      }
    }
    if (want_t && round_t) {
      res.launches += scan_exclusive_u32_u64(tri_cnt + t0, final_off + t0, nt, x.scan, st);
      uint32_t *dx = static_cast<uint32_t *>(r.xyz);
      uint64_t tbase = base_t, tcap = r.tri_cap;
      if (grow) {
        grow_keep(*r.grow_a, (base_t + round_t) * tri_words * 4, base_t * tri_words * 4, st);
        dx = r.grow_a->as<uint32_t>();
        tcap = ~0ull;
      } else if (r.final_host) {
        if (round >= 2) AMRX_CUDA(cudaStreamWaitEvent(st, copied[slot], 0));
        WsBuf &bx = slot ? out_b : out_a;
        bx.reserve(round_t * tri_words * 4 + 16, st);
        dx = bx.as<uint32_t>();
        tbase = 0;
        tcap = base_t < r.tri_cap ? std::min(round_t, r.tri_cap - base_t) : 0;
      }
      reorder_tri_kernel<<<std::max(1, rgrid), 256, 0, st>>>(
        tri_cnt + t0, tri_up + t0, tri_off + t0, final_off + t0, nt, tri_words,
        x.stage_a.as<uint32_t>(), dx, tbase, tcap, tri_stage);
      AMRX_LAUNCH_CHECK();
      res.launches += 1;
      if (r.final_host && !grow && tcap) {
        // overlapped: the copy drains on its own stream during the next round
        cudaEvent_t ready;
        AMRX_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        AMRX_CUDA(cudaEventRecord(ready, st));
        AMRX_CUDA(cudaStreamWaitEvent(cp, ready, 0));
        AMRX_CUDA(cudaMemcpyAsync(static_cast<char *>(r.xyz) + base_t * tri_words * 4, dx,
                                  tcap * tri_words * 4, cudaMemcpyDeviceToHost, cp));
        AMRX_CUDA(cudaEventRecord(copied[slot], cp));
        cudaEventDestroy(ready);
      }
    }
    AMRX_CUDA(cudaEventRecord(e2, st));
    AMRX_CUDA(cudaEventSynchronize(e2));
    AMRX_CUDA(cudaEventElapsedTime(&ms, e1, e2));
    res.ms2 += ms;
    base_d += round_d;
    base_t += round_t;
    for (int i = 0; i < 8; i++) prev[i] = h[i];
    t0 = t1;
    res.rounds += 1;
  }
  if (cp) AMRX_CUDA(cudaStreamSynchronize(cp));
  AMRX_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < 4; i++) res.counters[i] = h[i];
  res.duals = h[4];
  res.tris_counted = h[5];
  res.tris_written = h[6];
  res.error_flags = uint32_t(h[7]);
  if (debug) {
    unsigned long long d[kDbgCount];
    AMRX_CUDA(cudaMemcpy(d, ctl + 18, sizeof d, cudaMemcpyDeviceToHost));
    const char *names[kDbgCount] = {"tiles", "fast_need", "fast_pend", "runtime_points",
                                    "coarser_calls", "hash_extra_probes", "find_calls",
                                    "find_rounds", "narrow_steps", "fallback_queries",
                                    "queries"};
    std::fprintf(stderr, "[amrx dbg]");
    for (int i = 0; i < kDbgCount; i++)
      std::fprintf(stderr, " %s=%llu (%.2f/tile)", names[i], d[i],
                   d[0] ? double(d[i]) / double(d[0]) : 0.0);
    std::fprintf(stderr, "\n");
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  return res;
}

// ------------------------------------------------------- wide-key extraction

namespace {

struct WArgs {
  WideCtx w;
  KeyGeom g;
  const double *scal;
  uint64_t cell_begin, cell_end;
  double iso;
  uint32_t *dual_cnt, *tri_cnt;            // pass 1: per-cell counts
  const uint64_t *dual_off, *tri_off;      // pass 2: exclusive scans of them
  uint32_t *corners;
  uint64_t *tasks;
  uint64_t dual_cap;
  void *xyz;
  uint64_t tri_cap;
  unsigned long long *out;  // [0..3] counters, [4] duals, [5] tris, [7] errors
};

/*! the reference's two passes (pipeline.cpp:80-146) for the wide path: one
    thread per cell runs try_build_dual on its 8 candidates
    (pipeline.cpp:40-57) and contour_hex on the accepted ones; pass 1
    (WRITE = false) counts duals and triangles per cell, pass 2 writes them
    at the scanned offsets -- candidate order by construction */
template <bool DUAL, bool F32, bool WRITE>
__global__ void __launch_bounds__(256)
wide_extract_kernel(const __grid_constant__ WArgs a)
{
  __shared__ uint64_t rows[256];
  __shared__ double tcs[DUAL ? 1 : 12][256];  // per edge interpolation parameter
  if (!DUAL) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) rows[i] = c_mc_rows[table_row(uint32_t(i))];
    __syncthreads();
  }
  unsigned long long cnt[4] = {0, 0, 0, 0}, nd_sum = 0, nt_sum = 0;
  uint32_t err = 0;
  const uint64_t cells = a.cell_end - a.cell_begin;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < cells; r += stride) {
    const uint64_t cell = a.cell_begin + r;
    const Cell c = unpack128(a.g, wide_key(a.w.keys, cell));
    uint32_t nd = 0, nt = 0;
    for (int delta = 0; delta < 8; delta++) {
      uint32_t ids[8];
      uint8_t lev[8];
      const uint32_t code = wide_try(a.w, a.g, c, cell, delta, ids, lev);
      cnt[code]++;
      if (code) continue;
      if (DUAL) {
        if (WRITE) {
          const uint64_t slot = a.dual_off[r] + nd;
          if (slot < a.dual_cap) {
            for (int d = 0; d < 8; d++) a.corners[slot * 8 + d] = ids[d];
            if (a.tasks) a.tasks[slot] = cell * 8 + uint64_t(delta);
          }
        }
        nd++;
      } else {
        const uint64_t at = WRITE ? a.tri_off[r] + nt : 0;
        nt += uint32_t(mc_core<F32, false>(a.scal, rows, c, delta, a.iso,
                                           WRITE ? a.xyz : nullptr, at, WRITE ? a.tri_cap : 0,
                                           err, [&](int d) { return make_uint2(ids[d], lev[d]); },
                                           [&](int e) -> double & { return tcs[e][threadIdx.x]; }));
      }
    }
    if (!WRITE) {
      if (DUAL)
        a.dual_cnt[r] = nd;
      else
        a.tri_cnt[r] = nt;
    }
    nd_sum += nd;
    nt_sum += nt;
  }
  if (WRITE) return;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    for (int i = 0; i < 4; i++) cnt[i] += __shfl_xor_sync(kFull, cnt[i], off);
    nd_sum += __shfl_xor_sync(kFull, nd_sum, off);
    nt_sum += __shfl_xor_sync(kFull, nt_sum, off);
  }
  err = __reduce_or_sync(kFull, err);
  if ((threadIdx.x & 31) == 0) {
    for (int i = 0; i < 4; i++)
      if (cnt[i]) atomicAdd(a.out + i, cnt[i]);
    if (nd_sum) atomicAdd(a.out + 4, nd_sum);
    if (nt_sum) {
      atomicAdd(a.out + 5, nt_sum);
      atomicAdd(a.out + 6, nt_sum);
    }
    if (err) atomicOr(a.out + 7, (unsigned long long)err);
  }
}

template <bool DUAL, bool F32, bool WRITE>
void launch_wide(const WArgs &a, cudaStream_t st)
{
  const uint64_t cells = a.cell_end - a.cell_begin;
  const int grid = int(std::max<uint64_t>(
    1, std::min<uint64_t>((cells + 255) / 256, uint64_t(device_sm_count()) * 8)));
  wide_extract_kernel<DUAL, F32, WRITE><<<grid, 256, 0, st>>>(a);
  AMRX_LAUNCH_CHECK();
}

}  // namespace

ExtractResult run_extract_wide(const ExtractRequest &r, const WideCtx &w, cudaStream_t st)
{
  ExtractResult res{};
  const uint64_t cells = r.cell_end > r.cell_begin ? r.cell_end - r.cell_begin : 0;
  const bool D = r.emit_dual, F = r.tri_f32;
  DevBuf ctl, cnt, off, scratch, tmp_a, tmp_b;
  ctl.reserve(256, st);
  AMRX_CUDA(cudaMemsetAsync(ctl.ptr, 0, 256, st));
  cnt.reserve(cells * 4 + 16, st);
  off.reserve(cells * 8 + 16, st);
  WArgs a{};
  a.w = w;
  a.g = r.g;
  a.scal = r.scal;
  a.cell_begin = r.cell_begin;
  a.cell_end = r.cell_begin + cells;
  a.iso = r.iso;
  a.dual_cnt = a.tri_cnt = cnt.as<uint32_t>();
  a.dual_off = a.tri_off = off.as<uint64_t>();
  a.out = ctl.as<unsigned long long>();
  cudaEvent_t e0, e1, e2;
  AMRX_CUDA(cudaEventCreate(&e0));
  AMRX_CUDA(cudaEventCreate(&e1));
  AMRX_CUDA(cudaEventCreate(&e2));
  AMRX_CUDA(cudaEventRecord(e0, st));
  if (cells) {
    if (D) launch_wide<true, false, false>(a, st);
    else if (F) launch_wide<false, true, false>(a, st);
    else launch_wide<false, false, false>(a, st);
    res.launches += 1;
  }
  unsigned long long h[8];
  AMRX_CUDA(cudaMemcpyAsync(h, ctl.ptr, sizeof h, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  AMRX_CUDA(cudaEventRecord(e1, st));
  const uint64_t total = D ? h[4] : h[6];
  const size_t item = D ? 32 : (F ? 36 : 72);
  if (cells && total) {
    res.launches += scan_exclusive_u32_u64(cnt.as<uint32_t>(), off.as<uint64_t>(), cells, scratch,
                                           st);
    // destination: the growable arena, a device buffer for host output, or
    // the caller's device buffer (writes past its capacity are skipped)
    void *dst = D ? static_cast<void *>(r.corners) : r.xyz;
    uint64_t *dst_tasks = r.tasks;
    uint64_t cap = D ? r.dual_cap : r.tri_cap;
    if (r.grow_a) {
      r.grow_a->reserve(total * item, st);
      dst = r.grow_a->ptr;
      if (D) {
        r.grow_b->reserve(total * 8, st);
        dst_tasks = r.grow_b->as<uint64_t>();
      }
      cap = total;
    } else if (r.final_host) {
      cap = std::min(cap, total);
      tmp_a.reserve(cap * item + 16, st);
      dst = tmp_a.ptr;
      if (D && r.tasks) {
        tmp_b.reserve(cap * 8 + 16, st);
        dst_tasks = tmp_b.as<uint64_t>();
      }
    }
    if (D) {
      a.corners = static_cast<uint32_t *>(dst);
      a.tasks = dst_tasks;
      a.dual_cap = cap;
      launch_wide<true, false, true>(a, st);
    } else {
      a.xyz = dst;
      a.tri_cap = cap;
      if (F) launch_wide<false, true, true>(a, st);
      else launch_wide<false, false, true>(a, st);
    }
    res.launches += 1;
    if (r.final_host && !r.grow_a && cap) {
      AMRX_CUDA(cudaMemcpyAsync(D ? static_cast<void *>(r.corners) : r.xyz, dst, cap * item,
                                cudaMemcpyDeviceToHost, st));
      if (D && r.tasks)
        AMRX_CUDA(cudaMemcpyAsync(r.tasks, dst_tasks, cap * 8, cudaMemcpyDeviceToHost, st));
    }
  }
  AMRX_CUDA(cudaEventRecord(e2, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  AMRX_CUDA(cudaEventElapsedTime(&res.ms, e0, e1));
  AMRX_CUDA(cudaEventElapsedTime(&res.ms2, e1, e2));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  for (int i = 0; i < 4; i++) res.counters[i] = h[i];
  res.duals = h[4];
  res.tris_counted = h[5];
  res.tris_written = h[6];
  res.error_flags = uint32_t(h[7]);
  res.rounds = 1;
  return res;
}

void run_find_exact(const SearchCtx &s, const KeyGeom &g, const int4 *cells,
                    uint64_t n, int64_t *out, cudaStream_t st)
{
  if (!n) return;
  find_exact_kernel<<<grid_query(n), kThreads, 0, st>>>(s, g, cells, n, out);
  AMRX_LAUNCH_CHECK();
}

void run_snap(const SearchCtx &s, const KeyGeom &g, const int64_t *points,
              const int32_t *hints, int32_t hint_all, uint64_t n, int64_t *out,
              cudaStream_t st)
{
  if (!n) return;
  snap_kernel<<<grid_query(n), kThreads, 0, st>>>(s, g, points, hints, hint_all,
                                                  n, out);
  AMRX_LAUNCH_CHECK();
}

void run_try_build(const SearchCtx &s, const KeyGeom &g, const uint64_t *tasks,
                   uint64_t n, uint8_t *reject, uint32_t *corners,
                   cudaStream_t st)
{
  if (!n) return;
  try_build_kernel<<<grid_query(n), kThreads, 0, st>>>(s, g, tasks, n, reject,
                                                       corners);
  AMRX_LAUNCH_CHECK();
}

}  // namespace amrx

namespace amrx {
unsigned int check_word_extract() { return take_check_word(); }
}  // namespace amrx
