// Ingest kernels: validation prepass, key packing, order check, scalar
// gather, search directory, device scan.  Replaces build_index's serial
// loops (proj/src/locator.cpp:26-92) with HBM-streaming passes.
#include "internal.h"

#include <algorithm>
#include <climits>
#include <vector>

namespace amrx {

namespace {

constexpr int kThreads = 256;
#ifndef AMRX_GRID_BLOCKS
#define AMRX_GRID_BLOCKS 32
#endif

int grid_for(uint64_t n, int threads, int per_thread = 1, int blocks_per_sm = AMRX_GRID_BLOCKS)
{
  const uint64_t blocks = (n + uint64_t(threads) * per_thread - 1) /
                          (uint64_t(threads) * per_thread);
  const uint64_t cap = uint64_t(device_sm_count()) * blocks_per_sm;
  return int(std::max<uint64_t>(1, std::min(blocks, cap)));
}

struct PrepassAcc {
  unsigned long long first_bad;
  int mn[3];
  int mx[3];
  long long hi[3];
  unsigned int level_mask;
};

/*! locator.cpp:33-50 per record (level in [0,30], anchor aligned) fused
    with the bounds/level reductions of locator.cpp:70-89.  The first bad
    record in INPUT order wins (atomicMin on its position), so the host can
    name "record n" exactly like the serial loop. */
constexpr int kPrepassItems = 4;

__global__ void __launch_bounds__(kThreads)
prepass_kernel(const int4 *__restrict__ cells, uint64_t n, PrepassAcc *acc)
{
  int mn[3] = {INT_MAX, INT_MAX, INT_MAX};
  int mx[3] = {INT_MIN, INT_MIN, INT_MIN};
  long long hi[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  unsigned int mask = 0;
  unsigned long long bad = ~0ull;
  // kPrepassItems loads in flight per thread (strided by the block size)
  constexpr int U = kPrepassItems;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t r0 = uint64_t(blockIdx.x) * blockDim.x * U + threadIdx.x; r0 < n;
       r0 += stride) {
    int4 cs[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      if (r0 + u * blockDim.x < n) cs[u] = __ldg(cells + r0 + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t r = r0 + u * blockDim.x;
      if (r >= n) break;
      const int4 c = cs[u];
      const int v[3] = {c.x, c.y, c.z};
      bool ok = c.w >= 0 && c.w <= kMaxLevel;
      if (ok) {
        const int64_t w = int64_t(1) << c.w;
#pragma unroll
        for (int a = 0; a < 3; a++) {
          ok = ok && anchor_mask(v[a], c.w) == v[a];
          mn[a] = min(mn[a], v[a]);
          mx[a] = max(mx[a], v[a]);
          hi[a] = max(hi[a], (long long)(v[a] + w));
        }
        mask |= 1u << c.w;
      }
      if (!ok && r < bad) bad = r;
    }
  }
  // warp reduce, then one atomic per warp
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      mn[a] = min(mn[a], __shfl_xor_sync(kFull, mn[a], off));
      mx[a] = max(mx[a], __shfl_xor_sync(kFull, mx[a], off));
      hi[a] = max(hi[a], (long long)__shfl_xor_sync(kFull, hi[a], off));
    }
    mask |= __shfl_xor_sync(kFull, mask, off);
    const unsigned long long ob = __shfl_xor_sync(kFull, bad, off);
    bad = ob < bad ? ob : bad;
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      atomicMin(&acc->mn[a], mn[a]);
      atomicMax(&acc->mx[a], mx[a]);
      atomicMax(&acc->hi[a], hi[a]);
    }
    atomicOr(&acc->level_mask, mask);
    if (bad != ~0ull) atomicMin(&acc->first_bad, bad);
  }
}

__global__ void __launch_bounds__(kThreads)
pack_kernel(const int4 *__restrict__ cells, uint64_t n, const KeyGeom g,
            uint64_t *__restrict__ keys, uint32_t *__restrict__ idx)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += stride) {
    const int4 c = __ldg(cells + r);
    keys[r] = pack_unchecked(g, c.x, c.y, c.z, c.w);
    if (idx) idx[r] = uint32_t(r);
  }
}

/*! pack + the sort's digit histograms + the order check in one read of the
    cells: per-block shared histograms flushed once; a key's successor
    comes from the next lane (whole warps step together), or is packed again
    at a warp's last lane */
constexpr int kPackRuns = 4;

__global__ void __launch_bounds__(kThreads)
pack_hist_kernel(const int4 *__restrict__ cells, uint64_t n, const KeyGeom g,
                 uint64_t *__restrict__ keys, uint32_t *__restrict__ idx,
                 unsigned int *__restrict__ hist, int passes,
                 unsigned long long *__restrict__ order2)
{
  __shared__ unsigned int h[kSortMaxPasses][kSortDigits];
  for (int i = threadIdx.x; i < passes * kSortDigits; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned long long desc = 0, eq = 0;
  // a warp takes kPackRuns runs of 32 consecutive cells per step, all loads
  // issued first; a run's last key compares with the next run's first
  constexpr int U = kPackRuns;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
  for (uint64_t base = (uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u)) * U; base < n;
       base += stride) {
    int4 c[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t r = base + u * 32 + lane;
      if (r < n) c[u] = __ldg(cells + r);
    }
    int4 tail = make_int4(0, 0, 0, 0);
    const uint64_t after = base + U * 32;  // the first cell past the warp's runs
    if (lane == 31 && after < n) tail = __ldg(cells + after);
    uint64_t k[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t r = base + u * 32 + lane;
      k[u] = 0;
      if (r < n) {
        k[u] = pack_unchecked(g, c[u].x, c[u].y, c[u].z, c[u].w);
        keys[r] = k[u];
        if (idx) idx[r] = uint32_t(r);
#pragma unroll 1
        for (int p = 0; p < passes; p++)
          atomicAdd(&h[p][(k[u] >> (p * kSortRadixBits)) & (kSortDigits - 1)], 1u);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t r = base + u * 32 + lane;
      uint64_t nxt = __shfl_down_sync(kFull, (unsigned long long)k[u], 1);
      if (u + 1 < U) {
        const uint64_t first = __shfl_sync(kFull, (unsigned long long)k[u + 1 < U ? u + 1 : u], 0);
        if (lane == 31) nxt = first;
      } else if (lane == 31 && after < n) {
        nxt = pack_unchecked(g, tail.x, tail.y, tail.z, tail.w);
      }
      if (r + 1 < n) {
        desc += k[u] > nxt;
        eq += k[u] == nxt;
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    desc += __shfl_xor_sync(kFull, desc, off);
    eq += __shfl_xor_sync(kFull, eq, off);
  }
  if (lane == 0) {
    if (desc) atomicAdd(order2, desc);
    if (eq) atomicAdd(order2 + 1, eq);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kSortDigits; i += blockDim.x) {
    const unsigned int v = (&h[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

__global__ void __launch_bounds__(kThreads)
order_check_kernel(const uint64_t *__restrict__ keys, uint64_t n,
                   unsigned long long *out2)
{
  unsigned long long desc = 0, eq = 0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
       r + 1 < n; r += stride) {
    const uint64_t a = ldg_u64(keys + r), b = ldg_u64(keys + r + 1);
    desc += a > b;
    eq += a == b;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    desc += __shfl_xor_sync(kFull, desc, off);
    eq += __shfl_xor_sync(kFull, eq, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (desc) atomicAdd(out2, desc);
    if (eq) atomicAdd(out2 + 1, eq);
  }
}

__global__ void __launch_bounds__(kThreads)
gather_kernel(const uint32_t *__restrict__ perm, const double *__restrict__ in,
              double *__restrict__ out, uint64_t n)
{
  // four independent random loads in flight per thread (the gather is
  // bound by outstanding 32-byte sector reads, not by bandwidth)
  constexpr int U = 4;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r0 < n;
       r0 += stride * U) {
    uint32_t p[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t r = r0 + u * stride;
      p[u] = r < n ? __ldg(perm + r) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = r0 + u * stride < n ? __ldg(in + p[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; u++)
      if (r0 + u * stride < n) out[r0 + u * stride] = v[u];
  }
}

__global__ void __launch_bounds__(kThreads)
scatter_kernel(const uint32_t *__restrict__ rank, const double *__restrict__ in,
               double *__restrict__ out, uint64_t n)
{
  constexpr int U = 4;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r0 < n;
       r0 += stride * U) {
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t r = r0 + u * stride;
      if (r < n) out[__ldg(rank + r)] = __ldg(in + r);
    }
  }
}

__global__ void __launch_bounds__(kThreads)
iota_kernel(uint32_t *__restrict__ p, uint64_t n)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride)
    p[r] = uint32_t(r);
}

__global__ void pad_kernel(uint64_t *keys, uint64_t n)
{
  keys[n + threadIdx.x] = ~0ull;
}

/*! bucket histogram over sorted keys: equal buckets form runs, so each
    warp issues one atomic per distinct bucket it holds */
__global__ void __launch_bounds__(kThreads)
bucket_count_kernel(const uint64_t *__restrict__ keys, uint64_t n, int shift,
                    uint32_t *__restrict__ cnt, unsigned long long *order2)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t start = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long desc = 0, eq = 0;
  // whole warps iterate together so the match below sees all lanes
  for (uint64_t base = start - (threadIdx.x & 31); base < n; base += stride) {
    const uint64_t r = base + (threadIdx.x & 31);
    const bool in = r < n;
    const uint64_t k = in ? ldg_u64(keys + r) : 0;
    // fused order check of the sorted keys (descents must be 0; equal
    // neighbours are duplicate cells)
    if (in && r + 1 < n) {
      const uint64_t k1 = ldg_u64(keys + r + 1);
      desc += k > k1;
      eq += k == k1;
    }
    const uint64_t b = in ? (k >> shift) : ~0ull;
    const uint32_t peers = __match_any_sync(kFull, b);
    const bool leader = in && (__ffs(peers) - 1) == int(threadIdx.x & 31);
    if (leader) atomicAdd(cnt + b, __popc(peers));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    desc += __shfl_xor_sync(kFull, desc, off);
    eq += __shfl_xor_sync(kFull, eq, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (desc) atomicAdd(order2, desc);
    if (eq) atomicAdd(order2 + 1, eq);
  }
}

__global__ void __launch_bounds__(kThreads)
unpack_kernel(const uint64_t *__restrict__ keys, uint64_t n, const KeyGeom g,
              int4 *__restrict__ cells)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += stride) {
    const Cell c = unpack(g, ldg_u64(keys + r));
    cells[r] = make_int4(int(c.i), int(c.j), int(c.k), c.level);
  }
}

// --------------------------------------------------- reduce-then-scan
// T = element type, A = accumulator / output type (u32 -> u32 or u32 -> u64)
constexpr int kScanThreads = 512;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename A>
__device__ __forceinline__ A block_exclusive_sum(A v, A *smem, A *total)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  A x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const A y = __shfl_up_sync(kFull, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    A s = lane < nw ? smem[lane] : A(0);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const A y = __shfl_up_sync(kFull, s, off);
      if (lane >= off) s += y;
    }
    if (lane < nw) smem[lane] = s;
  }
  __syncthreads();
  const A warp_excl = warp ? smem[warp - 1] : A(0);
  if (total) *total = smem[(blockDim.x >> 5) - 1];
  return warp_excl + x - v;
}

template <typename T, typename A>
__global__ void __launch_bounds__(kScanThreads)
scan_reduce_kernel(const T *__restrict__ in, uint64_t n, A *__restrict__ sums)
{
  __shared__ A sm[32];
  const uint64_t base = uint64_t(blockIdx.x) * kScanTile;
  A s = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; t++) {
    const uint64_t r = base + uint64_t(t) * kScanThreads + threadIdx.x;
    if (r < n) s += A(in[r]);
  }
  A total;
  block_exclusive_sum<A>(s, sm, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

template <typename T, typename A>
__global__ void __launch_bounds__(kScanThreads)
scan_downsweep_kernel(const T *in, A *out, uint64_t n,
                      const A *__restrict__ block_offsets)
{
  __shared__ A sm[32];
  const uint64_t base = uint64_t(blockIdx.x) * kScanTile +
                        uint64_t(threadIdx.x) * kScanItems;
  A v[kScanItems];
  A s = 0;
  const bool full = base + kScanItems <= n;
  if (full && (sizeof(T) * kScanItems) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
    // a thread's items are contiguous: 16-byte vector loads
    constexpr int per = 16 / sizeof(T);
    const uint4 *src = reinterpret_cast<const uint4 *>(in + base);
#pragma unroll
    for (int q = 0; q < kScanItems / per; q++) {
      const uint4 w = src[q];
      const T *e = reinterpret_cast<const T *>(&w);
#pragma unroll
      for (int t = 0; t < per; t++) v[q * per + t] = A(e[t]);
    }
#pragma unroll
    for (int t = 0; t < kScanItems; t++) s += v[t];
  } else {
#pragma unroll
    for (int t = 0; t < kScanItems; t++) {
      const uint64_t r = base + t;
      v[t] = r < n ? A(in[r]) : A(0);
      s += v[t];
    }
  }
  A run = block_exclusive_sum<A>(s, sm, nullptr) +
          (block_offsets ? block_offsets[blockIdx.x] : A(0));
  if (full && (sizeof(A) * kScanItems) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    constexpr int per = 16 / sizeof(A);
    uint4 *dst = reinterpret_cast<uint4 *>(out + base);
#pragma unroll
    for (int q = 0; q < kScanItems / per; q++) {
      uint4 w;
      A *e = reinterpret_cast<A *>(&w);
#pragma unroll
      for (int t = 0; t < per; t++) {
        e[t] = run;
        run += v[q * per + t];
      }
      dst[q] = w;
    }
  } else {
#pragma unroll
    for (int t = 0; t < kScanItems; t++) {
      const uint64_t r = base + t;
      if (r < n) out[r] = run;
      run += v[t];
    }
  }
}

// ------------------------------------------- occupancy records, one pass
// A block owns 4096 consecutive buckets; their keys are one contiguous run
// of the sorted array, starting at tile_start[t].  The block ORs the keys'
// bits and counts them per bucket in shared memory, scans the counts and
// writes its records once: no memset, no device-wide scan, each key read
// once.  The counts (not popcounts) make rec[b].x the exact lower bound of
// bucket b even with duplicate keys, so the records double as the search
// directory (bounds rec[b].x, rec[b+1].x).

constexpr int kRecTile = 1 << kRecTileLog;
#ifndef AMRX_REC_THREADS
#define AMRX_REC_THREADS 256  // C4 ingest: 256 49.8 ms, 512 50.4, 1024 52.2
#endif
constexpr int kRecThreads = AMRX_REC_THREADS;
#ifndef AMRX_REC_UNROLL
#define AMRX_REC_UNROLL 2  // C4 records 5.85 -> 5.49 ms (4: 5.98, 8: 9.23)
#endif
constexpr int kRecUnroll = AMRX_REC_UNROLL;

/// tile_start[t] = first position whose bucket >= rec_lo + t * kRecTile,
/// t in [0, tiles]; rec_lo is a multiple of kRecTile and no key lies below it
__global__ void __launch_bounds__(kThreads)
rec_tile_start_kernel(const uint64_t *__restrict__ keys, uint64_t n, int dir_shift,
                      uint64_t rec_lo, uint64_t tiles, uint32_t *__restrict__ tile_start)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const auto tile_of = [&](uint64_t i) {
    return std::min<uint64_t>(((ldg_u64(keys + i) >> dir_shift) - rec_lo) >> kRecTileLog, tiles);
  };
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n; i += stride) {
    const uint64_t cur = i < n ? tile_of(i) : tiles;
    const uint64_t from = i > 0 ? tile_of(i - 1) + 1 : 0;
    for (uint64_t t = from; t <= cur; t++) tile_start[t] = uint32_t(i);
  }
}

__global__ void __launch_bounds__(kRecThreads)
rec_build_kernel(const uint64_t *__restrict__ keys, uint64_t n, int dir_shift,
                 uint64_t entries, const uint32_t *__restrict__ tile_start,
                 uint2 *__restrict__ rec, unsigned long long *order2)
{
  __shared__ __align__(16) uint32_t bits[kRecTile];
  __shared__ __align__(16) uint32_t cnt[kRecTile];
  __shared__ uint32_t wsum[32];
  const uint64_t t = blockIdx.x;
  const uint64_t lo = tile_start[t], hi = tile_start[t + 1];
  const uint64_t r0 = t << kRecTileLog;  // records are relative to rec_lo
  if (lo == hi) {
    // no key in these buckets (most tiles of a sparse level): every record
    // is {lo, 0}, two per 16-byte store
    const uint4 z = make_uint4(uint32_t(lo), 0u, uint32_t(lo), 0u);
    if (r0 + kRecTile <= entries) {
      uint4 *dst = reinterpret_cast<uint4 *>(rec + r0);
#pragma unroll
      for (int j = threadIdx.x; j < kRecTile / 2; j += kRecThreads) dst[j] = z;
    } else {
      for (int j = threadIdx.x; j < kRecTile; j += kRecThreads)
        if (r0 + j < entries) rec[r0 + j] = make_uint2(uint32_t(lo), 0u);
    }
    return;
  }
  {
    uint4 *zb = reinterpret_cast<uint4 *>(bits), *zc = reinterpret_cast<uint4 *>(cnt);
#pragma unroll
    for (int j = threadIdx.x; j < kRecTile / 4; j += kRecThreads) {
      zb[j] = make_uint4(0, 0, 0, 0);
      zc[j] = make_uint4(0, 0, 0, 0);
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned long long desc = 0, eq = 0;
  // whole warps step together so the match below sees all lanes;
  // kRecUnroll runs of 32 keys per warp and step, their loads issued first
  constexpr int U = kRecUnroll;
  for (uint64_t base = lo + (threadIdx.x & ~31u); base < hi; base += kRecThreads * U) {
    uint64_t kk[U], k1[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t i = base + u * kRecThreads + lane;
      kk[u] = i < hi ? ldg_u64(keys + i) : 0;
      k1[u] = i < hi && i + 1 < n ? ldg_u64(keys + i + 1) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t i = base + u * kRecThreads + lane;
      const bool in = i < hi;
      const uint64_t k = kk[u];
      if (in && i + 1 < n) {
        desc += k > k1[u];
        eq += k == k1[u];
      }
      const uint32_t b = in ? uint32_t(k >> dir_shift) & (kRecTile - 1) : 0xffffffffu;
      const uint32_t peers = __match_any_sync(kFull, b);
      uint32_t v = in ? 1u << (uint32_t(k) & 31u) : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {  // segmented OR over the run
        const uint32_t y = __shfl_down_sync(kFull, v, off);
        const uint32_t bo = __shfl_down_sync(kFull, b, off);
        if (lane + off < 32 && bo == b) v |= y;
      }
      if (in && (__ffs(peers) - 1) == lane) {
        atomicOr(&bits[b], v);
        atomicAdd(&cnt[b], uint32_t(__popc(peers)));
      }
    }
  }
  __syncthreads();
  // exclusive scan of the 4096 counts: 8 per thread
  constexpr int per = kRecTile / kRecThreads;
  uint32_t c[per], sum = 0;
#pragma unroll
  for (int j = 0; j < per; j++) {
    c[j] = cnt[threadIdx.x * per + j];
    sum += c[j];
  }
  uint32_t x = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) wsum[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t w = threadIdx.x < kRecThreads / 32 ? wsum[threadIdx.x] : 0u;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, w, off);
      if (lane >= off) w += y;
    }
    wsum[threadIdx.x] = w;
  }
  __syncthreads();
  uint32_t run = uint32_t(lo) + (x - sum) + ((threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : 0u);
#pragma unroll
  for (int j = 0; j < per; j++) {  // counts -> bucket starts, in place
    cnt[threadIdx.x * per + j] = run;
    run += c[j];
  }
  __syncthreads();
  if (r0 + kRecTile <= entries) {  // coalesced, two records per 16-byte store
    uint4 *dst = reinterpret_cast<uint4 *>(rec + r0);
#pragma unroll
    for (int j = threadIdx.x; j < kRecTile / 2; j += kRecThreads) {
      const uint2 c = reinterpret_cast<const uint2 *>(cnt)[j];
      const uint2 b = reinterpret_cast<const uint2 *>(bits)[j];
      dst[j] = make_uint4(c.x, b.x, c.y, b.y);
    }
  } else {
    for (int j = threadIdx.x; j < kRecTile; j += kRecThreads)
      if (r0 + j < entries) rec[r0 + j] = make_uint2(cnt[j], bits[j]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    desc += __shfl_xor_sync(kFull, desc, off);
    eq += __shfl_xor_sync(kFull, eq, off);
  }
  if (lane == 0) {
    if (desc) atomicAdd(order2, desc);
    if (eq) atomicAdd(order2 + 1, eq);
  }
}

// ------------------------------------------- hashed occupancy records
// For key spaces too sparse for a record per bucket (deep hierarchies, wide
// extents): one 16-byte slot per OCCUPIED bucket in an open-addressed table
// (common.cuh, hash_home).  Two passes over the sorted keys: count the
// distinct buckets (fused with the order check), then insert one slot per
// bucket, its bits ORed by the lanes holding the bucket's keys.

/// acc[0] += distinct buckets, acc[1] += descents, acc[2] += equal pairs
__global__ void __launch_bounds__(kThreads)
hash_count_kernel(const uint64_t *__restrict__ keys, uint64_t n, int dir_shift,
                  unsigned long long *acc)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  unsigned long long nb = 0, desc = 0, eq = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = ldg_u64(keys + i);
    nb += i == 0 || (ldg_u64(keys + i - 1) >> dir_shift) != (k >> dir_shift);
    if (i + 1 < n) {
      const uint64_t k1 = ldg_u64(keys + i + 1);
      desc += k > k1;
      eq += k == k1;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    nb += __shfl_xor_sync(kFull, nb, off);
    desc += __shfl_xor_sync(kFull, desc, off);
    eq += __shfl_xor_sync(kFull, eq, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (nb) atomicAdd(acc, nb);
    if (desc) atomicAdd(acc + 1, desc);
    if (eq) atomicAdd(acc + 2, eq);
  }
}

/// one entry per distinct record bucket (unique keys: a bucket holds <= 32
/// keys); the first key of a bucket inserts it with the OR of its keys' bits
/// into the first free entry of its probe sequence, the entry b & 1 of a
/// table bucket before the other (a full table bucket never empties, so a
/// probe may stop at the first table bucket with a free entry)
__global__ void __launch_bounds__(kThreads)
hash_build_kernel(const uint64_t *__restrict__ keys, uint64_t n, int dir_shift,
                  ulonglong4 *__restrict__ tab, uint64_t mask, unsigned int *max_probe)
{
  const int lane = threadIdx.x & 31;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  unsigned int longest = 0;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); base < n;
       base += stride) {
    const uint64_t i = base + lane;
    const bool in = i < n;
    const uint64_t k = in ? ldg_u64(keys + i) : 0;
    const uint64_t b = in ? k >> dir_shift : ~0ull;
    uint64_t pb = __shfl_up_sync(kFull, b, 1);
    if (lane == 0) pb = (in && i > 0) ? ldg_u64(keys + i - 1) >> dir_shift : ~0ull;
    uint32_t v = in ? 1u << (uint32_t(k) & 31u) : 0u;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {  // segmented OR toward the run's first lane
      const uint32_t y = __shfl_down_sync(kFull, v, off);
      const uint64_t bo = __shfl_down_sync(kFull, b, off);
      if (lane + off < 32 && bo == b) v |= y;
    }
    const uint64_t b31 = __shfl_sync(kFull, b, 31);
    if (in && (i == 0 || pb != b)) {
      if (b31 == b)  // the bucket continues past this warp's 32 keys
        for (uint64_t j = base + 32; j < n; j++) {
          const uint64_t kj = ldg_u64(keys + j);
          if ((kj >> dir_shift) != b) break;
          v |= 1u << (uint32_t(kj) & 31u);
        }
      uint64_t h = hash_home(b, mask);
      unsigned int probe = 0;
      unsigned long long *slot = nullptr;
      const int pref = int(b & 1);  // the preferred entry (lookups read it first)
      for (;;) {
        unsigned long long *e = reinterpret_cast<unsigned long long *>(tab + h);
        if (atomicCAS(e + 2 * pref, 0ull, (unsigned long long)(b + 1)) == 0ull) {
          slot = e + 2 * pref;
          break;
        }
        if (atomicCAS(e + 2 * (pref ^ 1), 0ull, (unsigned long long)(b + 1)) == 0ull) {
          slot = e + 2 * (pref ^ 1);
          break;
        }
        h = (h + 1) & mask;
        probe++;
      }
      slot[1] = uint64_t(uint32_t(i)) | (uint64_t(v) << 32);
      longest = probe > longest ? probe : longest;
    }
  }
  longest = __reduce_max_sync(kFull, longest);
  if (lane == 0 && longest) atomicMax(max_probe, longest);
}

/// out[t] = lower_bound of q[t] in the sorted keys (one thread per query)
__global__ void lower_bound_kernel(const uint64_t *__restrict__ keys, uint64_t n,
                                   const uint64_t *__restrict__ q, int nq, uint64_t *out)
{
  const int t = threadIdx.x;
  if (t < nq) out[t] = global_lower_bound(keys, 0, n, q[t]);
}

/*! DualCell records (dual.hpp:30-35, 64 bytes: 8 corner CellIds, the
    query base dual_base_of(owner, delta) (dual.hpp:61-67) as 3 x int64, the
    owner's level, the owner) from the extraction's corners and task ids */
template <bool WIDE>
__global__ void __launch_bounds__(kThreads)
dual_cells_kernel(const uint32_t *__restrict__ corners, const uint64_t *__restrict__ tasks,
                  uint64_t n, const void *__restrict__ keys, const KeyGeom g,
                  uint4 *__restrict__ out)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; d < n; d += stride) {
    const uint64_t t = tasks[d];
    const uint64_t owner = t >> 3;
    const int delta = int(t & 7);
    Cell c;
    if (WIDE) {
      const ulonglong2 k = __ldg(static_cast<const ulonglong2 *>(keys) + owner);
      c = unpack128(g, u128(k.x) | (u128(k.y) << 64));
    } else {
      c = unpack(g, ldg_u64(static_cast<const uint64_t *>(keys) + owner));
    }
    const int64_t w = int64_t(1) << c.level;
    const int64_t bx = c.i - ((delta & 1) ? 0 : w), by = c.j - ((delta & 2) ? 0 : w),
                  bz = c.k - ((delta & 4) ? 0 : w);
    const uint4 *src = reinterpret_cast<const uint4 *>(corners + 8 * d);
    uint4 *dst = out + 4 * d;
    dst[0] = src[0];
    dst[1] = src[1];
    dst[2] = make_uint4(uint32_t(bx), uint32_t(uint64_t(bx) >> 32), uint32_t(by),
                        uint32_t(uint64_t(by) >> 32));
    dst[3] = make_uint4(uint32_t(bz), uint32_t(uint64_t(bz) >> 32), uint32_t(c.level),
                        uint32_t(owner));
  }
}

/// recursive reduce-then-scan; block sums of each level in a pool buffer
template <typename T, typename A>
int scan_exclusive(const T *in, A *out, uint64_t n, cudaStream_t st)
{
  if (n == 0) return 0;
  const uint64_t blocks = (n + kScanTile - 1) / kScanTile;
  if (blocks == 1) {
    scan_downsweep_kernel<T, A><<<1, kScanThreads, 0, st>>>(in, out, n, nullptr);
    AMRX_LAUNCH_CHECK();
    return 1;
  }
  DevBuf sums;  // stream-ordered pool allocation: freed in stream order
  sums.reserve(size_t(blocks) * sizeof(A), st);
  scan_reduce_kernel<T, A><<<unsigned(blocks), kScanThreads, 0, st>>>(in, n, sums.as<A>());
  AMRX_LAUNCH_CHECK();
  int launches = 2 + scan_exclusive<A, A>(sums.as<A>(), sums.as<A>(), blocks, st);
  scan_downsweep_kernel<T, A><<<unsigned(blocks), kScanThreads, 0, st>>>(in, out, n,
                                                                        sums.as<A>());
  AMRX_LAUNCH_CHECK();
  return launches;
}

}  // namespace

PrepassResult ingest_prepass(const int4 *cells, uint64_t n, DevBuf &scratch,
                             cudaStream_t st)
{
  PrepassAcc init;
  init.first_bad = ~0ull;
  for (int a = 0; a < 3; a++) {
    init.mn[a] = INT_MAX;
    init.mx[a] = INT_MIN;
    init.hi[a] = LLONG_MIN;
  }
  init.level_mask = 0;
  scratch.reserve(sizeof(PrepassAcc), st);
  PrepassAcc *acc = scratch.as<PrepassAcc>();
  AMRX_CUDA(cudaMemcpyAsync(acc, &init, sizeof init, cudaMemcpyHostToDevice, st));
  prepass_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(cells, n, acc);
  AMRX_LAUNCH_CHECK();
  PrepassAcc h;
  AMRX_CUDA(cudaMemcpyAsync(&h, acc, sizeof h, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  PrepassResult r;
  r.first_bad = h.first_bad;
  for (int a = 0; a < 3; a++) {
    r.mn[a] = h.mn[a];
    r.mx[a] = h.mx[a];
    r.hi[a] = h.hi[a];
  }
  r.level_mask = h.level_mask;
  return r;
}

void ingest_pack(const int4 *cells, uint64_t n, const KeyGeom &g,
                 uint64_t *keys, uint32_t *idx, cudaStream_t st,
                 unsigned int *hist, int passes, unsigned long long *order2)
{
  if (hist) {
    AMRX_CUDA(cudaMemsetAsync(hist, 0, size_t(kSortMaxPasses) * kSortDigits * 4, st));
    AMRX_CUDA(cudaMemsetAsync(order2, 0, 16, st));
    pack_hist_kernel<<<grid_for(n, kThreads, 8), kThreads, 0, st>>>(cells, n, g, keys, idx,
                                                                   hist, passes, order2);
    AMRX_LAUNCH_CHECK();
    return;
  }
  pack_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(cells, n, g, keys,
                                                            idx);
  AMRX_LAUNCH_CHECK();
}

void ingest_order_check(const uint64_t *keys, uint64_t n, DevBuf &scratch,
                        uint64_t *descents, uint64_t *equal_pairs,
                        cudaStream_t st)
{
  scratch.reserve(16, st);
  auto *out = scratch.as<unsigned long long>();
  AMRX_CUDA(cudaMemsetAsync(out, 0, 16, st));
  order_check_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(keys, n,
                                                                   out);
  AMRX_LAUNCH_CHECK();
  unsigned long long h[2];
  AMRX_CUDA(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  *descents = h[0];
  *equal_pairs = h[1];
}

void gather_f64(const uint32_t *perm, const double *in, double *out,
                uint64_t n, cudaStream_t st)
{
  gather_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(perm, in, out,
                                                              n);
  AMRX_LAUNCH_CHECK();
}

void scatter_f64(const uint32_t *rank, const double *in, double *out, uint64_t n,
                 cudaStream_t st)
{
  if (n == 0) return;
#ifndef AMRX_SCATTER_GRID_BLOCKS
#define AMRX_SCATTER_GRID_BLOCKS 32
#endif
  scatter_kernel<<<grid_for(n, kThreads, 4, AMRX_SCATTER_GRID_BLOCKS), kThreads, 0, st>>>(rank, in,
                                                                                          out, n);
  AMRX_LAUNCH_CHECK();
}

void fill_iota(uint32_t *p, uint64_t n, cudaStream_t st)
{
  if (n == 0) return;
  iota_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(p, n);
  AMRX_LAUNCH_CHECK();
}

namespace {

/// AMRCELL1 records (io.cpp:35-37: i, j, k, level as int32 then the f64
/// scalar, 24 bytes, little-endian) into the index's input arrays; the
/// lowest record number with a non-finite scalar goes to *bad
/// (io.cpp:115-116 checks them in record order)
__global__ void __launch_bounds__(kThreads)
split_records_kernel(const uint64_t *__restrict__ rec, uint64_t n, uint64_t first,
                     int4 *__restrict__ cells, double *__restrict__ scal,
                     unsigned long long *__restrict__ bad)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint64_t a = __ldg(rec + 3 * r), b = __ldg(rec + 3 * r + 1), c = __ldg(rec + 3 * r + 2);
    cells[first + r] = make_int4(int(uint32_t(a)), int(uint32_t(a >> 32)), int(uint32_t(b)),
                                 int(uint32_t(b >> 32)));
    const double v = __longlong_as_double((long long)c);
    scal[first + r] = v;
    if (!isfinite(v)) atomicMin(bad, (unsigned long long)(first + r));
  }
}

}  // namespace

void split_records(const void *rec, uint64_t n, uint64_t first, int4 *cells, double *scal,
                   unsigned long long *bad, cudaStream_t st)
{
  if (n == 0) return;
  split_records_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(
    static_cast<const uint64_t *>(rec), n, first, cells, scal, bad);
  AMRX_LAUNCH_CHECK();
}

void pad_keys(uint64_t *keys, uint64_t n, cudaStream_t st)
{
  pad_kernel<<<1, kKeyPad, 0, st>>>(keys, n);
  AMRX_LAUNCH_CHECK();
}

void build_directory(const uint64_t *keys, uint64_t n, const KeyGeom &g,
                     uint32_t *dir, uint2 *rec, unsigned long long *order2,
                     DevBuf &scratch, cudaStream_t st, uint64_t rec_lo, uint64_t rec_n,
                     const uint32_t *tile_starts)
{
  uint64_t entries = (uint64_t(1) << g.dir_bits) + 1;
  AMRX_CUDA(cudaMemsetAsync(order2, 0, 16, st));
  if (rec) {
    if (rec_n) entries = rec_n + 1;
    const uint64_t tiles = (entries + kRecTile - 1) / kRecTile;
    DevBuf starts;
    if (!tile_starts) {  // else the sort's last pass found them (rec_lo = 0)
      starts.reserve(size_t(tiles + 1) * sizeof(uint32_t), st);
      rec_tile_start_kernel<<<grid_for(n + 1, kThreads, 4), kThreads, 0, st>>>(
        keys, n, g.dir_shift, rec_lo, tiles, starts.as<uint32_t>());
      AMRX_LAUNCH_CHECK();
      tile_starts = starts.as<uint32_t>();
    }
    rec_build_kernel<<<unsigned(tiles), kRecThreads, 0, st>>>(
      keys, n, g.dir_shift, entries, tile_starts, rec, order2);
    AMRX_LAUNCH_CHECK();
    return;
  }
  AMRX_CUDA(cudaMemsetAsync(dir, 0, entries * sizeof(uint32_t), st));
  bucket_count_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(
    keys, n, g.dir_shift, dir, order2);
  AMRX_LAUNCH_CHECK();
  scan_exclusive_u32(dir, dir, entries, scratch, st);
}

uint64_t hash_count(const uint64_t *keys, uint64_t n, const KeyGeom &g,
                    unsigned long long *order2, DevBuf &scratch, cudaStream_t st)
{
  scratch.reserve(32, st);
  auto *acc = scratch.as<unsigned long long>();
  AMRX_CUDA(cudaMemsetAsync(acc, 0, 24, st));
  hash_count_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(keys, n, g.dir_shift, acc);
  AMRX_LAUNCH_CHECK();
  unsigned long long h[3];
  AMRX_CUDA(cudaMemcpyAsync(h, acc, sizeof h, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  const unsigned long long o2[2] = {h[1], h[2]};
  AMRX_CUDA(cudaMemcpyAsync(order2, o2, 16, cudaMemcpyHostToDevice, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  return h[0];
}

void build_hash(const uint64_t *keys, uint64_t n, const KeyGeom &g, ulonglong4 *tab,
                uint64_t buckets, unsigned int *max_probe, cudaStream_t st)
{
  AMRX_CUDA(cudaMemsetAsync(tab, 0, buckets * sizeof(ulonglong4), st));
  AMRX_CUDA(cudaMemsetAsync(max_probe, 0, sizeof(unsigned int), st));
#ifndef AMRX_HASH_GRID_BLOCKS
#define AMRX_HASH_GRID_BLOCKS 128  // deep hash build 2.98 (32) -> 2.76 ms (512: 4.57)
#endif
  hash_build_kernel<<<grid_for(n, kThreads, 4, AMRX_HASH_GRID_BLOCKS), kThreads, 0, st>>>(
    keys, n, g.dir_shift, tab, buckets - 1, max_probe);
  AMRX_LAUNCH_CHECK();
}

void lower_bounds(const uint64_t *keys, uint64_t n, const uint64_t *q, int nq, uint64_t *out,
                  cudaStream_t st)
{
  DevBuf buf;
  buf.reserve(size_t(2 * nq) * 8, st);
  AMRX_CUDA(cudaMemcpyAsync(buf.ptr, q, size_t(nq) * 8, cudaMemcpyHostToDevice, st));
  lower_bound_kernel<<<1, 32, 0, st>>>(keys, n, buf.as<uint64_t>(), nq, buf.as<uint64_t>() + nq);
  AMRX_LAUNCH_CHECK();
  AMRX_CUDA(cudaMemcpyAsync(out, buf.as<uint64_t>() + nq, size_t(nq) * 8, cudaMemcpyDeviceToHost,
                            st));
  AMRX_CUDA(cudaStreamSynchronize(st));
}

void dual_cells(const uint32_t *corners, const uint64_t *tasks, uint64_t n, const void *keys,
                const KeyGeom &g, void *out, cudaStream_t st)
{
  if (!n) return;
  if (g.wide)
    dual_cells_kernel<true><<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(
      corners, tasks, n, keys, g, static_cast<uint4 *>(out));
  else
    dual_cells_kernel<false><<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(
      corners, tasks, n, keys, g, static_cast<uint4 *>(out));
  AMRX_LAUNCH_CHECK();
}

void unpack_cells(const uint64_t *keys, uint64_t n, const KeyGeom &g,
                  int4 *cells, cudaStream_t st)
{
  unpack_kernel<<<grid_for(n, kThreads, 4), kThreads, 0, st>>>(keys, n, g,
                                                              cells);
  AMRX_LAUNCH_CHECK();
}

int scan_exclusive_u32(const uint32_t *in, uint32_t *out, uint64_t n,
                       DevBuf &, cudaStream_t st)
{
  return scan_exclusive<uint32_t, uint32_t>(in, out, n, st);
}

int scan_exclusive_u32_u64(const uint32_t *in, uint64_t *out, uint64_t n,
                           DevBuf &, cudaStream_t st)
{
  return scan_exclusive<uint32_t, unsigned long long>(
    in, reinterpret_cast<unsigned long long *>(out), n, st);
}

}  // namespace amrx

namespace amrx {
unsigned int check_word_ingest() { return take_check_word(); }
}  // namespace amrx
