// Stable LSD radix sort of (u64 key, u32 or u64 value) pairs, onesweep
// style: the digit histograms of every pass up front (counted while the keys
// are packed, or by one sweep), then per 9-bit pass a single kernel that
// ranks a tile in shared memory (warp multisplit with peer masks built by
// shared-memory OR), shuffles it into digit order, obtains the tile's global
// digit offsets through a decoupled look-back over its predecessors, and
// scatters digit-sorted runs so the stores coalesce.  Replaces the std::sort
// over a permutation in build_index (proj/src/locator.cpp:52-68); stability
// keeps duplicate keys in input order exactly like its (key, input index)
// comparator.
#include "internal.h"

#include <algorithm>
#include <type_traits>
#include <vector>

namespace amrx {

namespace {

// digit width (<= 9: one thread per digit); C4: 4 passes of 9 bits 63.5 ms
// ingest vs 5 of 8 bits 64.7
constexpr int kRadixBits = kSortRadixBits;
constexpr int kDigits = 1 << kRadixBits;
#ifndef AMRX_SORT_THREADS
#define AMRX_SORT_THREADS 512
#endif
constexpr int kSortThreads = AMRX_SORT_THREADS;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef AMRX_SORT_ITEMS
#define AMRX_SORT_ITEMS 9  // C4 ingest: 8 40.4 ms, 9 38.0, 10 40.8 (spills), 12 / 16 at 1 CTA/SM 41.7 / 43.6
#endif
constexpr int kSortItems = AMRX_SORT_ITEMS;  // keys per thread
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kMaxPasses = kSortMaxPasses;

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed(
  const unsigned long long *p)
{
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(unsigned long long *p,
                                           unsigned long long v)
{
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}

/// all passes' digit histograms in one sweep over the keys
__global__ void __launch_bounds__(256)
histogram_kernel(const uint64_t *__restrict__ keys, uint64_t n, int passes,
                 unsigned int *__restrict__ hist)
{
  __shared__ unsigned int h[kMaxPasses][kDigits];
  for (int i = threadIdx.x; i < kMaxPasses * kDigits; i += blockDim.x)
    (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += stride) {
    const uint64_t k = ldg_u64(keys + r);
    for (int p = 0; p < passes; p++)
      atomicAdd(&h[p][(k >> (p * kRadixBits)) & (kDigits - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kDigits; i += blockDim.x) {
    const unsigned int v = (&h[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

/// exclusive scan of each pass's 256 bins (one block, one warp per pass)
__global__ void digit_offsets_kernel(const unsigned int *hist, int passes,
                                     unsigned long long *offs)
{
  const int lane = threadIdx.x & 31, p = threadIdx.x >> 5;
  if (p >= passes) return;
  unsigned long long run = 0;
  for (int base = 0; base < kDigits; base += 32) {
    unsigned long long v = hist[p * kDigits + base + lane];
    unsigned long long x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, x, off);
      if (lane >= off) x += y;
    }
    offs[p * kDigits + base + lane] = run + x - v;
    run += __shfl_sync(kFull, x, 31);
  }
}

#ifndef AMRX_SORT_LB
#define AMRX_SORT_LB 4  // with 9 keys per thread: 2 37.9, 3 37.6, 4 37.5, 6 37.7, 8 38.0
#endif
constexpr int kLookBack = AMRX_SORT_LB;
#ifndef AMRX_SORT_MINB
#define AMRX_SORT_MINB 2
#endif
// peer masks by shared-memory OR, not MATCH.ANY (its latency): C4 ingest 44.7 -> 43.6 ms
#ifndef AMRX_SORT_WHIST16
#define AMRX_SORT_WHIST16 1  // C4 ingest 49.9 -> 48.8 ms (u32 counts: more shared-memory traffic)
#endif
// per-warp digit counts (<= 32 x items) and their tile prefixes (< tile) fit u16
using WhistT = std::conditional_t<AMRX_SORT_WHIST16 != 0, uint16_t, uint32_t>;

template <typename V>
struct PassSmem {
  union {
    struct {
      uint64_t keys[kSortTile];
      V vals[kSortTile];
    };
    uint32_t pmasks[kSortWarps * kDigits];  // ranking's peer masks (before the shuffle)
  };
  WhistT whist[kSortWarps][kDigits];  // per-warp counts -> warp offsets
  uint32_t bexcl[kDigits];              // tile-local digit start
  uint32_t hist[kDigits];               // tile digit counts (early publish)
  uint32_t wsum[kSortWarps];            // block scan: per-warp totals
  unsigned long long gofs[kDigits];     // global start of this tile's run
  uint32_t tile;
};

/*! one LSD pass.  MODE kPassGather (the last pass): instead of the u32
    values, write gsrc[value] -- the payload the values index (the scalars
    in input order) -- so the separate gather kernel and the value round
    trip disappear; the random payload loads are issued together per thread
    in the final scatter, after the look-back.  MODE kPassInverse (the last
    pass): write vals_out[value] = sorted position (the inverse permutation,
    for scattering a payload that is still arriving). */
enum { kPassPlain = 0, kPassGather = 1, kPassInverse = 2 };
template <int MODE, typename V>
__global__ void __launch_bounds__(kSortThreads, AMRX_SORT_MINB)
onesweep_pass_kernel(const uint64_t *__restrict__ keys_in,
                     const V *__restrict__ vals_in,
                     uint64_t *__restrict__ keys_out,
                     V *__restrict__ vals_out, uint64_t n, int shift,
                     const unsigned long long *__restrict__ digit_start,
                     unsigned long long *state, unsigned int *ticket,
                     const double *__restrict__ gsrc, double *__restrict__ gdst,
                     uint32_t *__restrict__ ts, int ts_shift, uint64_t ts_tiles)
{
  static_assert(MODE == kPassPlain || sizeof(V) == 4, "gather/inverse carry u32 values");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  PassSmem<V> &sm = *reinterpret_cast<PassSmem<V> *>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the record tiles' first positions (last pass only, ts non-null): a key
  // whose smem predecessor is in its digit run knows its global
  // predecessor (dst - 1) and writes the tiles between the two exactly; a
  // run's first key only bounds its own tile (atomicMin) -- the empty tiles
  // in between are filled by tile_starts_fix_kernel
  const auto tile_start_note = [&](int pos, uint64_t kk, uint32_t d, uint64_t dst) {
    const uint64_t tcur = min((kk >> ts_shift) >> kRecTileLog, ts_tiles);
    if (pos > int(sm.bexcl[d])) {
      const uint64_t tprev = min((sm.keys[pos - 1] >> ts_shift) >> kRecTileLog, ts_tiles);
      for (uint64_t t = tprev + 1; t <= tcur; t++) ts[t] = uint32_t(dst);
    } else {
      atomicMin(ts + tcur, uint32_t(dst));
    }
  };

  if (threadIdx.x == 0) sm.tile = atomicAdd(ticket, 1u);
  // peer masks (per warp and digit) live in the key buffer's space, which
  // only the shuffle after the ranking writes (two alternating mask sets, to
  // drop one warp barrier per item, measured slower: 42.5 -> 43.0 ms)
  constexpr int kMaskWords = kSortWarps * kDigits;
  // zero the per-warp counts and the peer masks with 16-byte stores
  {
    constexpr int kW = int(sizeof(sm.whist) / 16);
    uint4 *w = reinterpret_cast<uint4 *>(&sm.whist[0][0]);
#pragma unroll
    for (int i = threadIdx.x; i < kW; i += kSortThreads) w[i] = make_uint4(0, 0, 0, 0);
    constexpr int kM = kMaskWords * 4 / 16;
    uint4 *m = reinterpret_cast<uint4 *>(sm.pmasks);
#pragma unroll
    for (int i = threadIdx.x; i < kM; i += kSortThreads) m[i] = make_uint4(0, 0, 0, 0);
  }
  for (int i = threadIdx.x; i < kDigits; i += kSortThreads) sm.hist[i] = 0;

  __syncthreads();
  const uint32_t tile = sm.tile;
  const uint64_t base = uint64_t(tile) * kSortTile;

  // warp-striped load: item t of lane l in warp w is tile position
  // w*256 + t*32 + l, so (w, t, l) order is input order
  uint64_t k[kSortItems];
  V v[kSortItems];
  uint32_t dig[kSortItems];
  uint32_t rank[kSortItems];
#pragma unroll
  for (int t = 0; t < kSortItems; t++) {
    const uint64_t r = base + uint64_t(warp) * (32 * kSortItems) + t * 32 + lane;
    const bool in = r < n;
    k[t] = in ? ldg_u64(keys_in + r) : ~0ull;
    v[t] = in ? __ldg(vals_in + r) : V(0);
    dig[t] = in ? uint32_t((k[t] >> shift) & (kDigits - 1)) : uint32_t(kDigits);
  }
  // the tile's digit counts by shared atomics, published right away so the
  // successors' look-back finds this tile's aggregate while it still ranks
#pragma unroll
  for (int t = 0; t < kSortItems; t++)
    if (dig[t] < kDigits) atomicAdd(&sm.hist[dig[t]], 1u);
  __syncthreads();
  const bool digit_thread = threadIdx.x < kDigits;
  unsigned long long *me = state + uint64_t(tile) * kDigits + threadIdx.x;
  if (digit_thread) st_relaxed(me, (tile == 0 ? kFlagPre : kFlagAgg) | sm.hist[threadIdx.x]);
  // warp multisplit: rank within (warp, digit) in input order
  const uint32_t lt = lanemask_lt();
  uint32_t *pmask = sm.pmasks + warp * kDigits;
#pragma unroll
  for (int t = 0; t < kSortItems; t++) {
    const bool valid = dig[t] < kDigits;
    uint32_t peers = 0;
    if (valid) atomicOr(pmask + dig[t], 1u << lane);
    __syncwarp();
    uint32_t before = 0;
    if (valid) {
      peers = pmask[dig[t]];
      before = sm.whist[warp][dig[t]];
    }
    rank[t] = before + __popc(peers & lt);
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == lane) {  // the digit's leader
      sm.whist[warp][dig[t]] = WhistT(before + __popc(peers));
      pmask[dig[t]] = 0;
    }
    __syncwarp();  // the clear lands before the next item's OR
  }
  __syncthreads();

  // per digit: exclusive over warps, tile total
  uint32_t total = 0;
  if (threadIdx.x < kDigits) {
    const int d = threadIdx.x;
    for (int w = 0; w < kSortWarps; w++) {
      const uint32_t c = sm.whist[w][d];
      sm.whist[w][d] = WhistT(total);
      total += c;
    }
  }
  // tile-local digit starts: block-wide exclusive scan of the totals, one
  // digit per thread (warp scans + a scan of the warp sums)
  {
    uint32_t x = total;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) sm.wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = lane < kSortWarps ? sm.wsum[lane] : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, w, off);
        if (lane >= off) w += y;
      }
      if (lane < kSortWarps) sm.wsum[lane] = w;
    }
    __syncthreads();
    if (digit_thread)
      sm.bexcl[threadIdx.x] = x - total + (warp ? sm.wsum[warp - 1] : 0u);
  }

  // the shuffle needs only tile-local offsets: done before the look-back,
  // the keys and values leave the registers before it (with the 8-wide
  // look-back: C4 ingest 49.5 -> 44.7 ms)
  __syncthreads();
  // local shuffle into digit order
#pragma unroll
  for (int t = 0; t < kSortItems; t++)
    if (dig[t] < kDigits) {
      const uint32_t pos = sm.bexcl[dig[t]] + sm.whist[warp][dig[t]] + rank[t];
      sm.keys[pos] = k[t];
      sm.vals[pos] = v[t];
    }
  // decoupled look-back per digit (the aggregate went out before the
  // ranking): sum the predecessors' until an inclusive prefix appears
  if (digit_thread) {
    const int d = threadIdx.x;
    unsigned long long excl = 0;
    if (tile != 0) {
      // AMRX_SORT_LB predecessors per round trip: the walk back to the
      // nearest inclusive prefix costs ~1/LB of the dependent L2 loads
      // (tile 0 always holds an inclusive prefix, so the walk ends there)
      int64_t j = int64_t(tile) - 1;
      for (bool done = false; !done;) {
        unsigned long long s[kLookBack];
#pragma unroll
        for (int q = 0; q < kLookBack; q++)
          s[q] = j - q >= 0 ? ld_relaxed(state + uint64_t(j - q) * kDigits + d) : 0ull;
#pragma unroll
        for (int q = 0; q < kLookBack; q++) {
          if (done || (s[q] & ~kValMask) == 0) break;  // not published yet: poll again from j
          excl += s[q] & kValMask;
          done = (s[q] & ~kValMask) == kFlagPre;
          j--;
        }
      }
      st_relaxed(me, kFlagPre | (excl + total));
    }
    sm.gofs[d] = digit_start[d] + excl;
  }
  __syncthreads();
  const uint64_t valid = n - base < uint64_t(kSortTile) ? n - base : kSortTile;
  if (MODE == kPassInverse) {
    for (int pos = threadIdx.x; pos < int(valid); pos += kSortThreads) {
      const uint64_t kk = sm.keys[pos];
      const uint32_t d = uint32_t((kk >> shift) & (kDigits - 1));
      const uint64_t dst = sm.gofs[d] + (pos - sm.bexcl[d]);
      if (!AMRX_BOUND(dst < n && uint64_t(sm.vals[pos]) < n, kChkSort)) continue;
      keys_out[dst] = kk;
      vals_out[sm.vals[pos]] = V(dst);
      if (ts) tile_start_note(pos, kk, d, dst);
    }
    return;
  }
  if (MODE == kPassGather) {
    constexpr int U = 4;  // payload loads in flight per thread
    for (int p0 = threadIdx.x; p0 < int(valid); p0 += U * kSortThreads) {
      double g[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int pos = p0 + u * kSortThreads;
        g[u] = pos < int(valid) ? __ldg(gsrc + sm.vals[pos]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int pos = p0 + u * kSortThreads;
        if (pos < int(valid)) {
          const uint64_t kk = sm.keys[pos];
          const uint32_t d = uint32_t((kk >> shift) & (kDigits - 1));
          const uint64_t dst = sm.gofs[d] + (pos - sm.bexcl[d]);
          if (!AMRX_BOUND(dst < n, kChkSort)) continue;
          keys_out[dst] = kk;
          gdst[dst] = g[u];
        }
      }
    }
    return;
  }
  for (int pos = threadIdx.x; pos < int(valid); pos += kSortThreads) {
    const uint64_t kk = sm.keys[pos];
    const uint32_t d = uint32_t((kk >> shift) & (kDigits - 1));
    const uint64_t dst = sm.gofs[d] + (pos - sm.bexcl[d]);
    if (!AMRX_BOUND(dst < n, kChkSort)) continue;
    keys_out[dst] = kk;
    vals_out[dst] = sm.vals[pos];
    if (ts) tile_start_note(pos, kk, d, dst);
  }
}

/// tile starts after the last pass: a reverse running minimum (the empty
/// tiles take the next tile's start; never-seen entries are 0xFFFFFFFF),
/// the sentinel entry is n.  Two launches over chunks of 1024 entries: the
/// chunk minima, then each chunk's reverse scan seeded with the minimum of
/// the chunks after it.
constexpr int kFixChunk = 1024;

__device__ __forceinline__ uint32_t ts_at(const uint32_t *ts, uint64_t i, uint64_t m, uint32_t n)
{
  return i >= m ? 0xFFFFFFFFu : (i == m - 1 ? min(ts[i], n) : ts[i]);
}

__global__ void __launch_bounds__(kFixChunk) tile_starts_min_kernel(const uint32_t *ts, uint64_t m,
                                                                   uint32_t n, uint32_t *cmin)
{
  __shared__ uint32_t wmin[kFixChunk / 32];
  const uint64_t i = uint64_t(blockIdx.x) * kFixChunk + threadIdx.x;
  uint32_t v = ts_at(ts, i, m, n);
  v = __reduce_min_sync(kFull, v);
  if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = __reduce_min_sync(kFull, wmin[threadIdx.x]);
    if (threadIdx.x == 0) cmin[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(kFixChunk) tile_starts_fix_kernel(uint32_t *ts, uint64_t m,
                                                                   uint32_t n, const uint32_t *cmin,
                                                                   uint32_t chunks)
{
  __shared__ uint32_t wsum[kFixChunk / 32];
  __shared__ uint32_t carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // carry: the minimum over the chunks after this one
  if (warp == 0) {
    uint32_t c = 0xFFFFFFFFu;
    for (uint32_t j = blockIdx.x + 1 + lane; j < chunks; j += 32) c = min(c, cmin[j]);
    c = __reduce_min_sync(kFull, c);
    if (lane == 0) carry_s = c;
  }
  const uint64_t i = uint64_t(blockIdx.x) * kFixChunk + threadIdx.x;
  uint32_t x = ts_at(ts, i, m, n);
  // reverse inclusive min-scan over the chunk: within the warp, then across
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_down_sync(kFull, x, off);
    if (lane + off < 32) x = min(x, y);
  }
  if (lane == 0) wsum[warp] = x;  // the warp's minimum
  __syncthreads();
  uint32_t later = carry_s;
  for (int w = warp + 1; w < kFixChunk / 32; w++) later = min(later, wsum[w]);
  if (i < m) ts[i] = min(x, later);
}

}  // namespace

size_t radix_sort_scratch_bytes(uint64_t n)
{
  const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
  return size_t(kMaxPasses) * kDigits * 12 + 256 + size_t(tiles) * kDigits * 8;
}

namespace {

/*! the pass driver for u32 or u64 values; vals_src (may differ from vals)
    is what the first executed pass reads, so a payload can enter the sort
    straight from the caller's read-only input */
template <typename V>
bool sort_impl(uint64_t *keys, const V *vals_src, V *vals, uint64_t *keys_alt, V *vals_alt,
               uint64_t n, int key_bits, void *scratch, cudaStream_t st, int *passes_run,
               const double *gsrc, double *gdst, cudaEvent_t gsrc_ready, uint32_t **rank_out,
               const unsigned int *hist_in, TileStarts *tstarts)
{
  if (tstarts) tstarts->filled = false;
  if (passes_run) *passes_run = 0;
  if (rank_out) *rank_out = nullptr;
  if (n <= 1 || key_bits <= 0) return false;
  const int passes = (key_bits + kRadixBits - 1) / kRadixBits;
  const uint64_t tiles = (n + kSortTile - 1) / kSortTile;

  // scratch: hist (passes*256 u32) | offsets (passes*256 u64) | ticket |
  // look-back state (tiles*256 u64)
  const size_t hist_bytes = size_t(kMaxPasses) * kDigits * 4;
  const size_t offs_bytes = size_t(kMaxPasses) * kDigits * 8;
  const size_t state_bytes = size_t(tiles) * kDigits * 8;
  auto *base = static_cast<unsigned char *>(scratch);
  auto *hist = reinterpret_cast<unsigned int *>(base);
  auto *offs = reinterpret_cast<unsigned long long *>(base + hist_bytes);
  auto *ticket = reinterpret_cast<unsigned int *>(base + hist_bytes + offs_bytes);
  auto *state = reinterpret_cast<unsigned long long *>(base + hist_bytes +
                                                       offs_bytes + 256);

  if (hist_in) {
    hist = const_cast<unsigned int *>(hist_in);  // counted while packing
  } else {
    AMRX_CUDA(cudaMemsetAsync(hist, 0, hist_bytes, st));
    const int hgrid = int(std::min<uint64_t>((n + 1023) / 1024,
                                             uint64_t(device_sm_count()) * 8));
    histogram_kernel<<<std::max(1, hgrid), 256, 0, st>>>(keys, n, passes, hist);
    AMRX_LAUNCH_CHECK();
  }
  digit_offsets_kernel<<<1, 32 * kMaxPasses, 0, st>>>(hist, passes, offs);
  AMRX_LAUNCH_CHECK();

  // passes whose digit is constant over all keys permute nothing: skip
  std::vector<unsigned int> h(size_t(passes) * kDigits);
  AMRX_CUDA(cudaMemcpyAsync(h.data(), hist, h.size() * 4,
                            cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));

  const size_t smem = sizeof(PassSmem<V>);
  ensure_smem_attr(reinterpret_cast<const void *>(onesweep_pass_kernel<kPassPlain, V>), smem);
  if (sizeof(V) == 4) {
    ensure_smem_attr(reinterpret_cast<const void *>(onesweep_pass_kernel<kPassGather, uint32_t>),
                     sizeof(PassSmem<uint32_t>));
    ensure_smem_attr(reinterpret_cast<const void *>(onesweep_pass_kernel<kPassInverse, uint32_t>),
                     sizeof(PassSmem<uint32_t>));
  }
  int last = -1;
  bool trivial[kMaxPasses] = {};
  for (int p = 0; p < passes; p++) {
    for (int d = 0; d < kDigits; d++)
      if (h[size_t(p) * kDigits + d] == n) trivial[p] = true;
    if (!trivial[p]) last = p;
  }
  uint64_t *kin = keys, *kout = keys_alt;
  V *vin = vals, *vout = vals_alt;
  int run = 0;
  const bool want_ts = tstarts && tstarts->starts && last >= 0 && !gsrc;
  for (int p = 0; p < passes; p++) {
    if (trivial[p]) continue;
    AMRX_CUDA(cudaMemsetAsync(state, 0, state_bytes, st));
    AMRX_CUDA(cudaMemsetAsync(ticket, 0, 4, st));
    const V *src = run == 0 ? vals_src : vin;
    uint32_t *ts = nullptr;
    int ts_shift = 0;
    uint64_t ts_tiles = 0;
    if (want_ts && p == last) {
      AMRX_CUDA(cudaMemsetAsync(tstarts->starts, 0xff, (tstarts->tiles + 1) * 4, st));
      ts = tstarts->starts;
      ts_shift = tstarts->shift;
      ts_tiles = tstarts->tiles;
    }
    if constexpr (sizeof(V) == 4) {
      if (rank_out && p == last) {
        onesweep_pass_kernel<kPassInverse, uint32_t><<<unsigned(tiles), kSortThreads, smem, st>>>(
          kin, src, kout, vout, n, p * kRadixBits, offs + size_t(p) * kDigits,
          state, ticket, nullptr, nullptr, ts, ts_shift, ts_tiles);
        *rank_out = vout;
      } else if (gsrc && p == last) {
        if (gsrc_ready) AMRX_CUDA(cudaStreamWaitEvent(st, gsrc_ready, 0));
        onesweep_pass_kernel<kPassGather, uint32_t><<<unsigned(tiles), kSortThreads, smem, st>>>(
          kin, src, kout, vout, n, p * kRadixBits, offs + size_t(p) * kDigits,
          state, ticket, gsrc, gdst, nullptr, 0, 0);
      } else {
        onesweep_pass_kernel<kPassPlain, V><<<unsigned(tiles), kSortThreads, smem, st>>>(
          kin, src, kout, vout, n, p * kRadixBits, offs + size_t(p) * kDigits,
          state, ticket, nullptr, nullptr, ts, ts_shift, ts_tiles);
      }
    } else {
      onesweep_pass_kernel<kPassPlain, V><<<unsigned(tiles), kSortThreads, smem, st>>>(
        kin, src, kout, vout, n, p * kRadixBits, offs + size_t(p) * kDigits,
        state, ticket, nullptr, nullptr, ts, ts_shift, ts_tiles);
    }
    AMRX_LAUNCH_CHECK();
    if (ts) {
      const uint64_t m = ts_tiles + 1;
      const uint32_t chunks = uint32_t((m + kFixChunk - 1) / kFixChunk);
      // the look-back state is free after the last pass: the chunk minima
      uint32_t *cmin = reinterpret_cast<uint32_t *>(state);
      tile_starts_min_kernel<<<chunks, kFixChunk, 0, st>>>(ts, m, uint32_t(n), cmin);
      AMRX_LAUNCH_CHECK();
      tile_starts_fix_kernel<<<chunks, kFixChunk, 0, st>>>(ts, m, uint32_t(n), cmin, chunks);
      AMRX_LAUNCH_CHECK();
      tstarts->filled = true;
    }
    std::swap(kin, kout);
    std::swap(vin, vout);
    run++;
  }
  if (passes_run) *passes_run = run;
  if (gsrc && !rank_out && last < 0) {  // nothing to permute: the payload in input order
    if (gsrc_ready) AMRX_CUDA(cudaStreamWaitEvent(st, gsrc_ready, 0));
    AMRX_CUDA(cudaMemcpyAsync(gdst, gsrc, n * 8, cudaMemcpyDeviceToDevice, st));
  }
  if (run == 0 && vals_src != vals)  // nothing permuted: the payload as given
    AMRX_CUDA(cudaMemcpyAsync(vals, vals_src, n * sizeof(V), cudaMemcpyDeviceToDevice, st));
  return kin != keys;  // the sorted keys (and values) are in the alt buffers
}

}  // namespace

bool radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_alt,
                      uint32_t *vals_alt, uint64_t n, int key_bits,
                      void *scratch, cudaStream_t st, int *passes_run,
                      const double *gsrc, double *gdst, cudaEvent_t gsrc_ready,
                      uint32_t **rank_out, const unsigned int *hist_in, TileStarts *ts)
{
  return sort_impl<uint32_t>(keys, vals, vals, keys_alt, vals_alt, n, key_bits, scratch, st,
                             passes_run, gsrc, gdst, gsrc_ready, rank_out, hist_in, ts);
}

bool radix_sort_pairs_u64(uint64_t *keys, const uint64_t *vals_src, uint64_t *vals,
                          uint64_t *keys_alt, uint64_t *vals_alt, uint64_t n, int key_bits,
                          void *scratch, cudaStream_t st, int *passes_run,
                          const unsigned int *hist_in, TileStarts *ts)
{
  return sort_impl<uint64_t>(keys, vals_src, vals, keys_alt, vals_alt, n, key_bits, scratch,
                             st, passes_run, nullptr, nullptr, nullptr, nullptr, hist_in, ts);
}

}  // namespace amrx

namespace amrx {
unsigned int check_word_sort() { return take_check_word(); }
}  // namespace amrx
