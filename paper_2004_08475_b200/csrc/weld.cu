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

int grid_of(uint64_t n)
{
  const uint64_t blocks = (n + kThreads * 4 - 1) / (kThreads * 4);
  return int(std::max<uint64_t>(1, std::min<uint64_t>(blocks, uint64_t(device_sm_count()) * 32)));
}

}  // namespace

uint64_t run_weld(const double *xyz9, uint64_t n_tris, double *verts, uint64_t vcap,
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

}  // namespace amrx
