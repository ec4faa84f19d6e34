// GPU weld: the fat triangle soup -> an indexed face set, identical to
// amriso::weld (proj/src/weld.cpp:31-64, weld.hpp:28-43).
//
// The reference tags each of the 3T corners with 3*triangle + corner, sorts
// the tagged corners by (x, y, z, tag) with double comparisons, opens a new
// vertex whenever a position differs from its predecessor, and writes each
// corner's vertex id into its triangle slot.  Here the lexicographic sort is
// three stable LSD radix sorts (z, then y, then x) of order-preserving
// 64-bit images of the coordinates, carrying the tag; the initial order is
// tag order, so ties end in tag order exactly like the reference's
// comparator.  -0.0 maps to the image of +0.0 because the reference's
// comparison and vec3d == treat them as equal (and no NaN reaches the weld,
// weld.cpp:43-44).  Run starts are flagged, an exclusive scan numbers the
// vertices, and one scatter by tag fills the triangles.
#include "internal.h"

#include <cstdlib>
#include <string>

namespace amrx {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint64_t order_image(double d)
{
  const uint64_t b = uint64_t(__double_as_longlong(d == 0.0 ? 0.0 : d));
  return (b >> 63) ? ~b : (b | (uint64_t(1) << 63));
}

/// keys[i] = image of coordinate `axis` of corner perm[i] (perm null: i, and
/// vals[i] = i); corner c = 3 * triangle + k sits at xyz9[3 * c]
__global__ void __launch_bounds__(kThreads)
corner_keys_kernel(const double *__restrict__ xyz9, uint64_t n, int axis,
                   const uint32_t *__restrict__ perm, uint64_t *__restrict__ keys,
                   uint32_t *__restrict__ vals)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t c = perm ? __ldg(perm + i) : i;
    keys[i] = order_image(__ldg(xyz9 + 3 * c + axis));
    if (!perm) vals[i] = uint32_t(i);
  }
}

/// flags[i] = 1 where sorted corner i opens a new vertex (weld.cpp:58)
__global__ void __launch_bounds__(kThreads)
weld_flags_kernel(const double *__restrict__ xyz9, const uint32_t *__restrict__ perm,
                  uint64_t n, uint32_t *__restrict__ flags)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint32_t f = 1;
    if (i > 0) {
      const uint64_t c = __ldg(perm + i), p = __ldg(perm + i - 1);
      f = !(__ldg(xyz9 + 3 * c) == __ldg(xyz9 + 3 * p) &&
            __ldg(xyz9 + 3 * c + 1) == __ldg(xyz9 + 3 * p + 1) &&
            __ldg(xyz9 + 3 * c + 2) == __ldg(xyz9 + 3 * p + 2));
    }
    flags[i] = f;
  }
}

/// vertices (first corner of each run) and triangle slots (weld.cpp:57-62)
__global__ void __launch_bounds__(kThreads)
weld_emit_kernel(const double *__restrict__ xyz9, const uint32_t *__restrict__ perm,
                 const uint32_t *__restrict__ flags, const uint32_t *__restrict__ excl,
                 uint64_t n, double *__restrict__ verts, uint64_t vcap,
                 uint32_t *__restrict__ tris)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t c = __ldg(perm + i);
    const uint32_t f = __ldg(flags + i);
    const uint32_t v = __ldg(excl + i) + f - 1;
    if (f && verts && v < vcap) {
      verts[3 * uint64_t(v)] = __ldg(xyz9 + 3 * uint64_t(c));
      verts[3 * uint64_t(v) + 1] = __ldg(xyz9 + 3 * uint64_t(c) + 1);
      verts[3 * uint64_t(v) + 2] = __ldg(xyz9 + 3 * uint64_t(c) + 2);
    }
    if (tris) tris[c] = v;
  }
}

// ---- hash weld: deduplicate the corners first, sort only the vertices ----
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

__device__ __forceinline__ uint64_t pos_hash(double x, double y, double z)
{
  // -0.0 hashes like +0.0: the reference's == treats them as one position
  uint64_t h = uint64_t(__double_as_longlong(x == 0.0 ? 0.0 : x)) * 0x9E3779B97F4A7C15ull;
  h ^= uint64_t(__double_as_longlong(y == 0.0 ? 0.0 : y)) * 0xC2B2AE3D27D4EB4Full;
  h ^= uint64_t(__double_as_longlong(z == 0.0 ? 0.0 : z)) * 0x165667B19E3779F9ull;
  h ^= h >> 31;
  h *= 0xD6E8FEB86659FD93ull;
  h ^= h >> 32;
  return h;
}

/*! one slot per distinct position (== on all three coordinates, like
    vec3d's operator==), open addressing with linear probing; corner c
    records its slot, and the slot keeps the lowest corner of its group
    (rep): the reference's sort by (x, y, z, tag) makes that corner's bits
    the vertex position */
__global__ void __launch_bounds__(kThreads)
weld_insert_kernel(const double *__restrict__ xyz9, uint64_t n, uint32_t *slot, uint32_t *rep,
                   uint64_t cap, uint32_t *__restrict__ corner_slot)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n; c += stride) {
    const double x = __ldg(xyz9 + 3 * c), y = __ldg(xyz9 + 3 * c + 1), z = __ldg(xyz9 + 3 * c + 2);
    uint64_t h = __umul64hi(pos_hash(x, y, z), cap);  // uniform in [0, cap)
    uint32_t s;
    while (true) {
      s = *(volatile uint32_t *)(slot + h);
      if (s == kEmpty) {
        s = atomicCAS(slot + h, kEmpty, uint32_t(c));
        if (s == kEmpty) {  // opened the group
          s = ~0u;
          break;
        }
      }
      if (__ldg(xyz9 + 3 * uint64_t(s)) == x && __ldg(xyz9 + 3 * uint64_t(s) + 1) == y &&
          __ldg(xyz9 + 3 * uint64_t(s) + 2) == z)
        break;
      h = h + 1 == cap ? 0 : h + 1;
    }
    // the group's lowest corner: only a corner below the one that opened
    // the group can be it
    if (uint32_t(c) < s) atomicMin(rep + h, uint32_t(c));
    corner_slot[c] = uint32_t(h);
  }
}

__global__ void __launch_bounds__(kThreads)
slot_flags_kernel(const uint32_t *__restrict__ rep, uint64_t cap, uint32_t *__restrict__ flags)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < cap; h += stride)
    flags[h] = __ldg(rep + h) != kEmpty;
}

/// occupied slot h -> its group number u: gslot[u] = h, gpos[u] = the
/// position (bits) of the group's lowest corner rep[h]
__global__ void __launch_bounds__(kThreads)
slot_compact_kernel(const double *__restrict__ xyz9, const uint32_t *__restrict__ rep,
                    const uint32_t *__restrict__ excl, uint64_t cap, uint32_t *__restrict__ gslot,
                    double *__restrict__ gpos)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < cap; h += stride) {
    const uint32_t r = __ldg(rep + h);
    if (r != kEmpty) {
      const uint64_t u = __ldg(excl + h);
      gslot[u] = uint32_t(h);
      gpos[3 * u] = __ldg(xyz9 + 3 * uint64_t(r));
      gpos[3 * u + 1] = __ldg(xyz9 + 3 * uint64_t(r) + 1);
      gpos[3 * u + 2] = __ldg(xyz9 + 3 * uint64_t(r) + 2);
    }
  }
}

/// keys[i] = image of coordinate `axis` of group perm[i] (perm null: i)
__global__ void __launch_bounds__(kThreads)
group_keys_kernel(const double *__restrict__ gpos, uint64_t n, int axis,
                  const uint32_t *__restrict__ perm, uint64_t *__restrict__ keys,
                  uint32_t *__restrict__ vals)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t u = perm ? __ldg(perm + i) : i;
    keys[i] = order_image(__ldg(gpos + 3 * u + axis));
    if (!perm) vals[i] = uint32_t(i);
  }
}

/// vertex v = the v-th group in position order: its coordinates, and the
/// vertex id written into the group's table slot (slot[gslot[u]] = v)
__global__ void __launch_bounds__(kThreads)
group_emit_kernel(const double *__restrict__ gpos, const uint32_t *__restrict__ perm, uint64_t nv,
                  double *__restrict__ verts, uint64_t vcap, const uint32_t *__restrict__ gslot,
                  uint32_t *__restrict__ slot)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv; v += stride) {
    const uint64_t u = __ldg(perm + v);
    slot[__ldg(gslot + u)] = uint32_t(v);
    if (verts && v < vcap) {
      verts[3 * v] = __ldg(gpos + 3 * u);
      verts[3 * v + 1] = __ldg(gpos + 3 * u + 1);
      verts[3 * v + 2] = __ldg(gpos + 3 * u + 2);
    }
  }
}

__global__ void __launch_bounds__(kThreads)
corner_vid_kernel(const uint32_t *__restrict__ corner_slot, const uint32_t *__restrict__ slot,
                  uint64_t n, uint32_t *__restrict__ tris)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n; c += stride)
    tris[c] = __ldg(slot + __ldg(corner_slot + c));
}

int grid_of(uint64_t n)
{
  const uint64_t blocks = (n + kThreads * 4 - 1) / (kThreads * 4);
  return int(std::max<uint64_t>(1, std::min<uint64_t>(blocks, uint64_t(device_sm_count()) * 32)));
}

}  // namespace

uint64_t run_weld_sort(const double *xyz9, uint64_t n_tris, double *verts, uint64_t vcap,
                       uint32_t *tris, cudaStream_t st)
{
  const uint64_t n = 3 * n_tris;
  if (n == 0) return 0;
  DevBuf kb[2], vb[2], sort_scratch, flags, excl, scan_scratch;
  for (int b = 0; b < 2; b++) {
    kb[b].reserve(n * 8, st);
    vb[b].reserve(n * 4, st);
  }
  sort_scratch.reserve(radix_sort_scratch_bytes(n), st);
  int cur = 0;  // buffer pair holding the current (keys, perm)
  for (int pass = 0; pass < 3; pass++) {
    const int axis = 2 - pass;  // z, y, x: LSD over the fields
    corner_keys_kernel<<<grid_of(n), kThreads, 0, st>>>(
      xyz9, n, axis, pass ? vb[cur].as<uint32_t>() : nullptr, kb[cur].as<uint64_t>(),
      vb[cur].as<uint32_t>());
    AMRX_LAUNCH_CHECK();
    int passes = 0;
    if (radix_sort_pairs(kb[cur].as<uint64_t>(), vb[cur].as<uint32_t>(),
                         kb[cur ^ 1].as<uint64_t>(), vb[cur ^ 1].as<uint32_t>(), n, 64,
                         sort_scratch.ptr, st, &passes))
      cur ^= 1;
  }
  const uint32_t *perm = vb[cur].as<uint32_t>();
  flags.reserve(n * 4, st);
  excl.reserve(n * 4, st);
  weld_flags_kernel<<<grid_of(n), kThreads, 0, st>>>(xyz9, perm, n, flags.as<uint32_t>());
  AMRX_LAUNCH_CHECK();
  scan_exclusive_u32(flags.as<uint32_t>(), excl.as<uint32_t>(), n, scan_scratch, st);
  uint32_t tail[2];
  AMRX_CUDA(cudaMemcpyAsync(&tail[0], excl.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaMemcpyAsync(&tail[1], flags.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  weld_emit_kernel<<<grid_of(n), kThreads, 0, st>>>(xyz9, perm, flags.as<uint32_t>(),
                                                    excl.as<uint32_t>(), n, verts, vcap, tris);
  AMRX_LAUNCH_CHECK();
  AMRX_CUDA(cudaStreamSynchronize(st));
  return uint64_t(tail[0]) + tail[1];
}

/*! Hash weld: identical result, sorts V vertices instead of 3T corners
    (C4: 68.6M vs 383M).  Open-addressed table of 1.5x the corner count
    (u32 slots), group numbering by a scan over the table, three stable LSD
    sorts of the groups' representative positions, then one gather per
    corner. */
uint64_t run_weld_hash(const double *xyz9, uint64_t n_tris, double *verts, uint64_t vcap,
                       uint32_t *tris, cudaStream_t st)
{
  const uint64_t n = 3 * n_tris;
  if (n == 0) return 0;
  // load factor <= 2/3 even if no corner is shared; slots are u32 (n < 2^32,
  // so a clamped table still has room for every corner)
  const uint64_t cap = std::min<uint64_t>(n + n / 2 + 1, 0xFFFFFFFFull);
  DevBuf slot, rep, cslot, flags, excl, scan_scratch;
  slot.reserve(cap * 4, st);
  rep.reserve(cap * 4, st);
  cslot.reserve(n * 4, st);
  AMRX_CUDA(cudaMemsetAsync(slot.ptr, 0xff, cap * 4, st));
  AMRX_CUDA(cudaMemsetAsync(rep.ptr, 0xff, cap * 4, st));
  weld_insert_kernel<<<grid_of(n), kThreads, 0, st>>>(xyz9, n, slot.as<uint32_t>(),
                                                       rep.as<uint32_t>(), cap,
                                                       cslot.as<uint32_t>());
  AMRX_LAUNCH_CHECK();
  flags.reserve(cap * 4, st);
  excl.reserve(cap * 4, st);
  slot_flags_kernel<<<grid_of(cap), kThreads, 0, st>>>(rep.as<uint32_t>(), cap,
                                                       flags.as<uint32_t>());
  AMRX_LAUNCH_CHECK();
  scan_exclusive_u32(flags.as<uint32_t>(), excl.as<uint32_t>(), cap, scan_scratch, st);
  uint32_t tail[2];
  AMRX_CUDA(cudaMemcpyAsync(&tail[0], excl.as<uint32_t>() + cap - 1, 4, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaMemcpyAsync(&tail[1], flags.as<uint32_t>() + cap - 1, 4, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  const uint64_t nv = uint64_t(tail[0]) + tail[1];
  flags.release();
  DevBuf gpos, gslot;
  gpos.reserve(nv * 24, st);
  gslot.reserve(nv * 4, st);
  slot_compact_kernel<<<grid_of(cap), kThreads, 0, st>>>(xyz9, rep.as<uint32_t>(),
                                                         excl.as<uint32_t>(), cap,
                                                         gslot.as<uint32_t>(), gpos.as<double>());
  AMRX_LAUNCH_CHECK();
  excl.release();
  rep.release();
  DevBuf kb[2], vb[2], sort_scratch;
  for (int b = 0; b < 2; b++) {
    kb[b].reserve(nv * 8, st);
    vb[b].reserve(nv * 4, st);
  }
  sort_scratch.reserve(radix_sort_scratch_bytes(nv), st);
  int cur = 0;
  for (int pass = 0; pass < 3; pass++) {
    const int axis = 2 - pass;  // z, y, x: LSD over the fields
    group_keys_kernel<<<grid_of(nv), kThreads, 0, st>>>(
      gpos.as<double>(), nv, axis, pass ? vb[cur].as<uint32_t>() : nullptr,
      kb[cur].as<uint64_t>(), vb[cur].as<uint32_t>());
    AMRX_LAUNCH_CHECK();
    int passes = 0;
    if (radix_sort_pairs(kb[cur].as<uint64_t>(), vb[cur].as<uint32_t>(),
                         kb[cur ^ 1].as<uint64_t>(), vb[cur ^ 1].as<uint32_t>(), nv, 64,
                         sort_scratch.ptr, st, &passes))
      cur ^= 1;
  }
  group_emit_kernel<<<grid_of(nv), kThreads, 0, st>>>(gpos.as<double>(), vb[cur].as<uint32_t>(),
                                                      nv, verts, vcap, gslot.as<uint32_t>(),
                                                      slot.as<uint32_t>());
  AMRX_LAUNCH_CHECK();
  if (tris) {
    corner_vid_kernel<<<grid_of(n), kThreads, 0, st>>>(cslot.as<uint32_t>(), slot.as<uint32_t>(),
                                                       n, tris);
    AMRX_LAUNCH_CHECK();
  }
  AMRX_CUDA(cudaStreamSynchronize(st));
  return nv;
}

uint64_t run_weld(const double *xyz9, uint64_t n_tris, double *verts, uint64_t vcap,
                  uint32_t *tris, cudaStream_t st)
{
  static const bool use_sort = [] {
    const char *e = std::getenv("AMRX_WELD");
    return e && std::string(e) == "sort";
  }();
  return use_sort ? run_weld_sort(xyz9, n_tris, verts, vcap, tris, st)
                  : run_weld_hash(xyz9, n_tris, verts, vcap, tris, st);
}

}  // namespace amrx

namespace amrx {
unsigned int check_word_weld() { return take_check_word(); }
}  // namespace amrx
