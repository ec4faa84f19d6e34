// The device index handle behind the C ABI's opaque amrx_index (api.cu,
// comm.cu): the sorted packed keys + scalars, the lookup structure, the
// cached last extraction.  Mirrors the reference's CellIndex
// (proj/include/amriso/locator.hpp:38-45) as device-resident SoA.
#pragma once

#include <mutex>

#include "amrx.h"
#include "internal.h"
#include "wide.cuh"

using namespace amrx;

struct amrx_index {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint64_t n = 0;
  KeyGeom g{};
  int64_t bounds_hi[3] = {0, 0, 0};
  DevBuf keys, scal, dir, rec, order, scratch;
  // partitions of a distributed index (amrx_index_from_keys): records of
  // buckets [rec_lo, rec_lo + rec_n) only, global id of local position 0
  uint64_t rec_lo = 0, rec_n = 0;
  int64_t id_base = 0;
  uint64_t key_lo = 0, key_hi = 0;
  bool partition = false;  // amrx_index_from_keys: a key range of a distributed index
  // a partition's interior: the local positions whose every lookup stays in
  // [key_lo, key_hi) (extraction ranges must lie inside it)
  uint64_t safe_lo = 0, safe_hi = ~0ull;
  uint64_t hmask = 0;      // hashed records: table buckets - 1
  bool searchable = true;  // false: sorted arrays only (amrx_index_sort_part)
  uint32_t jobs_per_kcell = 0;  // marching-cubes jobs per 1024 cells, last extraction
  amrx_index_info info{};
  // last extraction kept on the device for the count-then-copy pattern
  struct Cached {
    bool valid = false;
    int kind = 0;  // 1 dual, 2 iso
    uint64_t begin = 0, end = 0;
    double iso = 0;
    int f32 = 0;
    uint64_t count = 0;
    amrx_stats stats{};
  } cache;
  DevBuf out_a, out_b;  // arena: corners/xyz, tasks
  // the welded mesh of the cached soup (amrx_extract_iso_mesh)
  DevBuf mesh_v, mesh_t;
  bool mesh_valid = false;
  uint64_t mesh_nv = 0;
  double mesh_weld_s = 0;
  std::recursive_mutex mu;  // extract_iso_mesh holds it across extraction + weld

  /// the wide-key lookup context (g.wide)
  WideCtx wctx() const
  {
    WideCtx w;
    w.keys = keys.as<ulonglong2>();
    w.tab = rec.as<ulonglong4>();
    w.mask = hmask;
    w.n = n;
    w.id_base = 0;
    return w;
  }

  SearchCtx ctx() const
  {
    SearchCtx s;
    s.keys = keys.as<uint64_t>();
    // dense or hashed occupancy records (unique keys: positions are
    // popcounts), else the bucket directory (ensure_search_dir switches an
    // index with duplicate keys to it)
    s.rec = g.occ == kOccDense ? rec.as<uint2>() - rec_lo : nullptr;
    s.rec_lo = rec_lo;
    s.rec_cnt = g.occ == kOccDense ? info.lookup_entries : 0;
    s.htab = g.occ == kOccHash ? rec.as<ulonglong4>() : nullptr;
    s.hmask = hmask;
    s.dir = g.occ == kOccNone ? dir.as<uint32_t>() : nullptr;
    s.id_base = id_base;
    s.n = n;
    s.dir_shift = g.dir_shift;
    s.shift = g.shift;
    s.lmask = (uint64_t(1) << g.lbits) - 1;
    s.dbg = nullptr;
    return s;
  }
};


namespace amrx {

/*! extract_dual_mesh / extract_isosurface over a cell range (amrx_extract_*
    without the status wrapper: they throw ApiError).  cached = true runs
    the extraction into the index's device arena (or reuses it) and copies
    from there into any kind of output pointer (the multi-GPU gather) */
void extract_dual_impl(amrx_index *index, const amrx_range *range, uint32_t *corners8,
                       uint64_t *task_ids, uint64_t cap, uint64_t *count, amrx_stats *stats,
                       bool cached);
void extract_iso_impl(amrx_index *index, const amrx_range *range,
                      const amrx_iso_params *params, void *xyz9, uint64_t cap,
                      uint64_t *count, amrx_stats *stats, bool cached);

}  // namespace amrx
