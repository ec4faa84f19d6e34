// validate_dataset (proj/src/locator.cpp:136-161) on the GPU.
//
// Duplicates: adjacent equal cells of the sorted index, as (n, n+1) pairs in
// n order.  Overlaps: for every cell n and every present level coarser than
// it, in the index's level order (finest first, i.e. ascending), the exact
// lookup of the cell's anchor masked to that level; a hit is the pair
// (n, hit).  One count pass, an exclusive scan of the per-cell counts, one
// emit pass -- the reference's output order.  The masked anchor is the
// cell's packed key with the low bits of each coordinate field cleared
// (KeyGeom::cmask, when the key origin is aligned to the coarsest level),
// else it is re-packed from the decoded coordinates (query_key).
#include "internal.h"

namespace amrx {

namespace {

constexpr int kThreads = 256;

/// overlaps of cell i; EMIT writes (i, hit) pairs from out[0]
template <bool EMIT>
__device__ __forceinline__ uint32_t cell_overlaps(const SearchCtx &s, const KeyGeom &g,
                                                  uint64_t i, uint32_t *out)
{
  const uint64_t k = ldg_u64(s.keys + i);
  const int level = int(k & s.lmask) + s.shift;
  uint32_t cand = g.level_mask & ~((2u << level) - 1);
  uint32_t cnt = 0;
  Cell c{};
  if (!g.aligned) c = unpack(g, k);
  while (cand) {
    const int L = __ffs(cand) - 1;
    cand &= cand - 1;
    uint64_t q[1];
    bool v[1];
    if (g.aligned) {
      q[0] = (k & g.cmask[L]) | uint64_t(L - g.shift);
      v[0] = true;
    } else {
      v[0] = query_key(g, c.i, c.j, c.k, L, q[0]);
    }
    int64_t o[1] = {-1};
    int l1[1];
    batch_find<1, false>(s, q, v, o, l1);
    if (v[0] && o[0] >= 0) {
      if (EMIT) {
        out[2 * cnt] = uint32_t(int64_t(i) + s.id_base);
        out[2 * cnt + 1] = uint32_t(o[0] + s.id_base);
      }
      cnt++;
    }
  }
  return cnt;
}

__global__ void __launch_bounds__(kThreads)
validate_count_kernel(const SearchCtx s, const KeyGeom g, uint64_t n,
                      uint32_t *__restrict__ ovl, uint32_t *__restrict__ dup)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    ovl[i] = cell_overlaps<false>(s, g, i, nullptr);
    dup[i] = i + 1 < n && ldg_u64(s.keys + i) == ldg_u64(s.keys + i + 1);
  }
}

__global__ void __launch_bounds__(kThreads)
validate_emit_kernel(const SearchCtx s, const KeyGeom g, uint64_t n,
                     const uint32_t *__restrict__ ovl, const uint64_t *__restrict__ ovl_off,
                     const uint32_t *__restrict__ dup, const uint64_t *__restrict__ dup_off,
                     uint32_t *__restrict__ ovl_pairs, uint64_t ovl_cap,
                     uint32_t *__restrict__ dup_pairs, uint64_t dup_cap)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (ovl_pairs && ovl[i] && ovl_off[i] + ovl[i] <= ovl_cap)
      cell_overlaps<true>(s, g, i, ovl_pairs + 2 * ovl_off[i]);
    if (dup_pairs && dup[i] && dup_off[i] < dup_cap) {
      dup_pairs[2 * dup_off[i]] = uint32_t(int64_t(i) + s.id_base);
      dup_pairs[2 * dup_off[i] + 1] = uint32_t(int64_t(i) + 1 + s.id_base);
    }
  }
}

int grid_of(uint64_t n)
{
  const uint64_t blocks = (n + kThreads - 1) / kThreads;
  return int(std::max<uint64_t>(1, std::min<uint64_t>(blocks, uint64_t(device_sm_count()) * 32)));
}

}  // namespace

void run_validate(const SearchCtx &s, const KeyGeom &g, uint32_t *ovl_pairs, uint64_t ovl_cap,
                  uint64_t *n_ovl, uint32_t *dup_pairs, uint64_t dup_cap, uint64_t *n_dup,
                  cudaStream_t st)
{
  const uint64_t n = s.n;
  *n_ovl = *n_dup = 0;
  if (n == 0) return;
  DevBuf ovl, dup, ovl_off, dup_off, scratch;
  ovl.reserve(n * 4, st);
  dup.reserve(n * 4, st);
  ovl_off.reserve((n + 1) * 8, st);
  dup_off.reserve((n + 1) * 8, st);
  validate_count_kernel<<<grid_of(n), kThreads, 0, st>>>(s, g, n, ovl.as<uint32_t>(),
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
    validate_emit_kernel<<<grid_of(n), kThreads, 0, st>>>(
      s, g, n, ovl.as<uint32_t>(), ovl_off.as<uint64_t>(), dup.as<uint32_t>(),
      dup_off.as<uint64_t>(), ovl_pairs, ovl_cap, dup_pairs, dup_cap);
    AMRX_LAUNCH_CHECK();
  }
  AMRX_CUDA(cudaStreamSynchronize(st));
}

}  // namespace amrx

namespace amrx {
unsigned int check_word_validate() { return take_check_word(); }
}  // namespace amrx
