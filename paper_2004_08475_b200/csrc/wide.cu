// The wide-key path (wide.cuh): ingest into two-word keys, the exact-key
// hash table, the point queries, validate_dataset and the download, for
// datasets whose (i,j,k,level) key needs more than 64 bits.  Same contracts
// as the 64-bit path (build_index locator.cpp:26-92, find_exact/snap
// locator.cpp:94-134, try_build_dual dual.cpp:41-72, validate_dataset
// locator.cpp:136-161); the extraction is in extract.cu (run_extract_wide).
#include "internal.h"
#include "wide.cuh"

#include <algorithm>

namespace amrx {

namespace {

constexpr int kThreads = 256;

int grid_of(uint64_t n)
{
  const uint64_t blocks = (n + kThreads - 1) / kThreads;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(blocks, uint64_t(device_sm_count()) * 32)));
}

/// lo/hi words of every cell's key, idx = input position
__global__ void __launch_bounds__(kThreads)
wide_pack_kernel(const int4 *__restrict__ cells, uint64_t n, const KeyGeom g,
                 uint64_t *__restrict__ lo, uint64_t *__restrict__ hi, uint32_t *__restrict__ idx)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int4 c = cells[i];
    const u128 k = pack128(g, c.x, c.y, c.z, c.w);
    lo[i] = uint64_t(k);
    hi[i] = uint64_t(k >> 64);
    idx[i] = uint32_t(i);
  }
}

__global__ void __launch_bounds__(kThreads)
wide_gather_kernel(const uint32_t *__restrict__ perm, const uint64_t *__restrict__ in,
                   uint64_t n, uint64_t *__restrict__ out)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = AMRX_BOUND(perm[i] < n, kChkPerm) ? __ldg(in + perm[i]) : 0;
}

/// keys and scalars in sorted order from the final permutation; acc[0] +=
/// descents (must stay 0), acc[1] += equal neighbours, acc[2] += distinct keys
__global__ void __launch_bounds__(kThreads)
wide_finish_kernel(const int4 *__restrict__ cells, const double *__restrict__ scal,
                   const uint32_t *__restrict__ perm, uint64_t n, const KeyGeom g,
                   ulonglong2 *__restrict__ keys, double *__restrict__ scal_out,
                   unsigned long long *acc)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  unsigned long long desc = 0, eq = 0, distinct = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t p = perm[i];
    if (!AMRX_BOUND(p < n, kChkPerm)) continue;
    const int4 c = cells[p];
    const u128 k = pack128(g, c.x, c.y, c.z, c.w);
    keys[i] = make_ulonglong2(uint64_t(k), uint64_t(k >> 64));
    scal_out[i] = __ldg(scal + p);
    if (i > 0) {
      const int4 b = cells[perm[i - 1]];
      const u128 kb = pack128(g, b.x, b.y, b.z, b.w);
      desc += kb > k;
      eq += kb == k;
      distinct += kb != k;
    } else {
      distinct += 1;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    desc += __shfl_xor_sync(kFull, desc, off);
    eq += __shfl_xor_sync(kFull, eq, off);
    distinct += __shfl_xor_sync(kFull, distinct, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (desc) atomicAdd(acc, desc);
    if (eq) atomicAdd(acc + 1, eq);
    if (distinct) atomicAdd(acc + 2, distinct);
  }
}

/// the first position of every distinct key into the table (claimed by a
/// CAS on the id word; the key words are written by the claimer)
__global__ void __launch_bounds__(kThreads)
wide_hash_kernel(const ulonglong2 *__restrict__ keys, uint64_t n, ulonglong4 *tab,
                 uint64_t mask, unsigned int *max_probe)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  unsigned int longest = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u128 k = wide_key(keys, i);
    if (i > 0 && wide_key(keys, i - 1) == k) continue;  // a duplicate: the first one answers
    uint64_t h = wide_home(k, mask);
    unsigned int probe = 0;
    while (atomicCAS(reinterpret_cast<unsigned long long *>(&tab[h].z), 0ull,
                     (unsigned long long)(i + 1)) != 0ull) {
      h = (h + 1) & mask;
      probe++;
    }
    tab[h].x = uint64_t(k);
    tab[h].y = uint64_t(k >> 64);
    longest = probe > longest ? probe : longest;
  }
  longest = __reduce_max_sync(kFull, longest);
  if ((threadIdx.x & 31) == 0 && longest) atomicMax(max_probe, longest);
}

__global__ void __launch_bounds__(kThreads)
wide_unpack_kernel(const ulonglong2 *__restrict__ keys, uint64_t n, const KeyGeom g,
                   int4 *__restrict__ cells)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const Cell c = unpack128(g, wide_key(keys, i));
    cells[i] = make_int4(int(c.i), int(c.j), int(c.k), c.level);
  }
}

__global__ void __launch_bounds__(kThreads)
wide_find_kernel(const WideCtx w, const KeyGeom g, const int4 *__restrict__ cells, uint64_t n,
                 int64_t *__restrict__ out)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride) {
    const int4 c = cells[r];
    int64_t id = -1;
    // the full key: the anchor must be the stored one
    if (c.w >= 0 && c.w <= kMaxLevel && anchor_mask(c.x, c.w) == c.x &&
        anchor_mask(c.y, c.w) == c.y && anchor_mask(c.z, c.w) == c.z)
      id = wide_on_level(w, g, c.x, c.y, c.z, c.w);
    out[r] = id;
  }
}

__global__ void __launch_bounds__(kThreads)
wide_snap_kernel(const WideCtx w, const KeyGeom g, const int64_t *__restrict__ points,
                 const int32_t *__restrict__ hints, int32_t hint_all, uint64_t n,
                 int64_t *__restrict__ out)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride) {
    int l = 0;
    out[r] = wide_snap(w, g, points[3 * r], points[3 * r + 1], points[3 * r + 2],
                       hints ? hints[r] : hint_all, l);
  }
}

__global__ void __launch_bounds__(kThreads)
wide_try_kernel(const WideCtx w, const KeyGeom g, const uint64_t *__restrict__ tasks, uint64_t n,
                uint8_t *__restrict__ reject, uint32_t *__restrict__ corners)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint64_t cell = tasks[r] >> 3;
    uint32_t code = 1;
    uint32_t ids[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint8_t lev[8];
    if (cell < w.n)
      code = wide_try(w, g, unpack128(g, wide_key(w.keys, cell)), cell, int(tasks[r] & 7), ids,
                      lev);
    reject[r] = uint8_t(code);
    if (corners)
      for (int d = 0; d < 8; d++) corners[8 * r + d] = code == 0 ? ids[d] : 0;
  }
}

/// validate_dataset: overlaps of cell i -- every present level coarser than
/// its own, ascending, the cell's anchor masked to it, exact lookup
template <bool EMIT>
__device__ __forceinline__ uint32_t wide_overlaps(const WideCtx &w, const KeyGeom &g,
                                                  uint64_t i, uint32_t *out)
{
  const Cell c = unpack128(g, wide_key(w.keys, i));
  uint32_t cand = g.level_mask & ~((2u << c.level) - 1);
  uint32_t cnt = 0;
  while (cand) {
    const int L = __ffs(cand) - 1;
    cand &= cand - 1;
    const int64_t hit = wide_on_level(w, g, c.i, c.j, c.k, L);
    if (hit >= 0) {
      if (EMIT) {
        out[2 * cnt] = uint32_t(i);
        out[2 * cnt + 1] = uint32_t(hit);
      }
      cnt++;
    }
  }
  return cnt;
}

__global__ void __launch_bounds__(kThreads)
wide_validate_count_kernel(const WideCtx w, const KeyGeom g, uint32_t *__restrict__ ovl,
                           uint32_t *__restrict__ dup)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < w.n; i += stride) {
    ovl[i] = wide_overlaps<false>(w, g, i, nullptr);
    dup[i] = i + 1 < w.n && wide_key(w.keys, i) == wide_key(w.keys, i + 1);
  }
}

__global__ void __launch_bounds__(kThreads)
wide_validate_emit_kernel(const WideCtx w, const KeyGeom g, const uint32_t *__restrict__ ovl,
                          const uint64_t *__restrict__ ovl_off, const uint32_t *__restrict__ dup,
                          const uint64_t *__restrict__ dup_off, uint32_t *__restrict__ ovl_pairs,
                          uint64_t ovl_cap, uint32_t *__restrict__ dup_pairs, uint64_t dup_cap)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < w.n; i += stride) {
    if (ovl_pairs && ovl[i] && ovl_off[i] + ovl[i] <= ovl_cap)
      wide_overlaps<true>(w, g, i, ovl_pairs + 2 * ovl_off[i]);
    if (dup_pairs && dup[i] && dup_off[i] < dup_cap) {
      dup_pairs[2 * dup_off[i]] = uint32_t(i);
      dup_pairs[2 * dup_off[i] + 1] = uint32_t(i + 1);
    }
  }
}

}  // namespace

WideBuild wide_build(const int4 *cells, const double *scal, uint64_t n, const KeyGeom &g,
                     ulonglong2 *keys, double *scal_out, DevBuf &table, cudaStream_t st)
{
  WideBuild out{};
  // (1) lo/hi words + positions; (2) stable radix sort by lo; (3) the hi
  // words in that order, stable radix sort by hi -- lexicographic (hi, lo)
  // order with ties in input order (locator.cpp:52-60); (4) keys and
  // scalars gathered through the final permutation
  DevBuf lo, hi, lo2, idx, idx2, scratch, acc;
  lo.reserve(n * 8, st);
  hi.reserve(n * 8, st);
  lo2.reserve(n * 8, st);
  idx.reserve(n * 4, st);
  idx2.reserve(n * 4, st);
  scratch.reserve(radix_sort_scratch_bytes(n), st);
  wide_pack_kernel<<<grid_of(n), kThreads, 0, st>>>(cells, n, g, lo.as<uint64_t>(),
                                                    hi.as<uint64_t>(), idx.as<uint32_t>());
  AMRX_LAUNCH_CHECK();
  uint64_t *k1 = lo.as<uint64_t>(), *k1a = lo2.as<uint64_t>();
  uint32_t *v1 = idx.as<uint32_t>(), *v1a = idx2.as<uint32_t>();
  int passes = 0;
  if (radix_sort_pairs(k1, v1, k1a, v1a, n, 64, scratch.ptr, st, &passes)) {
    std::swap(k1, k1a);
    std::swap(v1, v1a);
  }
  out.passes += passes;
  // the hi words in lo order (k1a is free scratch now)
  wide_gather_kernel<<<grid_of(n), kThreads, 0, st>>>(v1, hi.as<uint64_t>(), n, k1a);
  AMRX_LAUNCH_CHECK();
  uint64_t *k2 = k1a, *k2a = k1;
  if (radix_sort_pairs(k2, v1, k2a, v1a, n, std::max(1, g.total - 64), scratch.ptr, st,
                       &passes))
    std::swap(v1, v1a);
  out.passes += passes;
  acc.reserve(32, st);
  AMRX_CUDA(cudaMemsetAsync(acc.ptr, 0, 32, st));
  wide_finish_kernel<<<grid_of(n), kThreads, 0, st>>>(cells, scal, v1, n, g, keys, scal_out,
                                                      acc.as<unsigned long long>());
  AMRX_LAUNCH_CHECK();
  unsigned long long h[3];
  AMRX_CUDA(cudaMemcpyAsync(h, acc.ptr, sizeof h, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  if (h[0] != 0) throw std::runtime_error("wide index keys are not in (i,j,k,level) order");
  out.equal_pairs = h[1];
  // exact-key table, at least two entries per distinct key
  uint64_t entries = 64;
  while (entries < 2 * h[2]) entries <<= 1;
  table.reserve(entries * sizeof(ulonglong4), st);
  AMRX_CUDA(cudaMemsetAsync(table.ptr, 0, entries * sizeof(ulonglong4), st));
  acc.reserve(32, st);
  AMRX_CUDA(cudaMemsetAsync(acc.ptr, 0, 4, st));
  wide_hash_kernel<<<grid_of(n), kThreads, 0, st>>>(keys, n, table.as<ulonglong4>(),
                                                    entries - 1, acc.as<unsigned int>());
  AMRX_LAUNCH_CHECK();
  unsigned int probe = 0;
  AMRX_CUDA(cudaMemcpyAsync(&probe, acc.ptr, 4, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  out.entries = entries;
  out.max_probe = probe;
  return out;
}

void wide_unpack(const ulonglong2 *keys, uint64_t n, const KeyGeom &g, int4 *cells,
                 cudaStream_t st)
{
  wide_unpack_kernel<<<grid_of(n), kThreads, 0, st>>>(keys, n, g, cells);
  AMRX_LAUNCH_CHECK();
}

void wide_find_exact(const WideCtx &w, const KeyGeom &g, const int4 *cells, uint64_t n,
                     int64_t *out, cudaStream_t st)
{
  if (!n) return;
  wide_find_kernel<<<grid_of(n), kThreads, 0, st>>>(w, g, cells, n, out);
  AMRX_LAUNCH_CHECK();
}

void wide_snap(const WideCtx &w, const KeyGeom &g, const int64_t *points, const int32_t *hints,
               int32_t hint_all, uint64_t n, int64_t *out, cudaStream_t st)
{
  if (!n) return;
  wide_snap_kernel<<<grid_of(n), kThreads, 0, st>>>(w, g, points, hints, hint_all, n, out);
  AMRX_LAUNCH_CHECK();
}

void wide_try_build(const WideCtx &w, const KeyGeom &g, const uint64_t *tasks, uint64_t n,
                    uint8_t *reject, uint32_t *corners, cudaStream_t st)
{
  if (!n) return;
  wide_try_kernel<<<grid_of(n), kThreads, 0, st>>>(w, g, tasks, n, reject, corners);
  AMRX_LAUNCH_CHECK();
}

void wide_validate(const WideCtx &w, const KeyGeom &g, uint32_t *ovl_pairs, uint64_t ovl_cap,
                   uint64_t *n_ovl, uint32_t *dup_pairs, uint64_t dup_cap, uint64_t *n_dup,
                   cudaStream_t st)
{
  const uint64_t n = w.n;
  *n_ovl = *n_dup = 0;
  if (n == 0) return;
  DevBuf ovl, dup, ovl_off, dup_off, scratch;
  ovl.reserve(n * 4, st);
  dup.reserve(n * 4, st);
  ovl_off.reserve((n + 1) * 8, st);
  dup_off.reserve((n + 1) * 8, st);
  wide_validate_count_kernel<<<grid_of(n), kThreads, 0, st>>>(w, g, ovl.as<uint32_t>(),
                                                              dup.as<uint32_t>());
  AMRX_LAUNCH_CHECK();
  scan_exclusive_u32_u64(ovl.as<uint32_t>(), ovl_off.as<uint64_t>(), n, scratch, st);
  scan_exclusive_u32_u64(dup.as<uint32_t>(), dup_off.as<uint64_t>(), n, scratch, st);
  uint64_t off[2];
  uint32_t last[2];
  AMRX_CUDA(cudaMemcpyAsync(&off[0], ovl_off.as<uint64_t>() + n - 1, 8, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaMemcpyAsync(&off[1], dup_off.as<uint64_t>() + n - 1, 8, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaMemcpyAsync(&last[0], ovl.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaMemcpyAsync(&last[1], dup.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  *n_ovl = off[0] + last[0];
  *n_dup = off[1] + last[1];
  if ((ovl_pairs && *n_ovl) || (dup_pairs && *n_dup)) {
    wide_validate_emit_kernel<<<grid_of(n), kThreads, 0, st>>>(
      w, g, ovl.as<uint32_t>(), ovl_off.as<uint64_t>(), dup.as<uint32_t>(),
      dup_off.as<uint64_t>(), ovl_pairs, ovl_cap, dup_pairs, dup_cap);
    AMRX_LAUNCH_CHECK();
  }
  AMRX_CUDA(cudaStreamSynchronize(st));
}

}  // namespace amrx

namespace amrx {
unsigned int check_word_wide() { return take_check_word(); }
}  // namespace amrx
