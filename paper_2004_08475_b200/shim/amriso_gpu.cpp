// GPU drop-in for the reference's hot path, with its exact C++ signatures:
//
//   CellIndex build_index(vector<CellCoord>, vector<double>)
//                                      proj/include/amriso/locator.hpp:52-53
//   ExtractionResult extract_isosurface(const CellIndex&, const IsoParams&)
//                                      proj/include/amriso/pipeline.hpp:65-66
//   vector<DualCell> extract_dual_mesh(const CellIndex&, int)
//                                      proj/include/amriso/pipeline.hpp:70-71
//   IndexedMesh weld(span<const FatTriangle>)
//                                      proj/include/amriso/weld.hpp:33-43
//   ValidationReport validate_dataset(const CellIndex&)
//                                      proj/include/amriso/locator.hpp:80
//   CellIndex read_amr(const std::filesystem::path&)
//                                      proj/include/amriso/io.hpp:43
//   write_obj / write_ply / write_dual_mesh  proj/include/amriso/io.hpp:51-64
//
// Compiled against the reference's own headers and linked in place of
// proj/src/pipeline.cpp, proj/src/weld.cpp, of build_index and
// validate_dataset in proj/src/locator.cpp and of read_amr and the three
// file writers in proj/src/io.cpp; everything else --
// snap/find_exact, the dual rules used by tests, contour_hex, the string
// formatters, generators, the CLI -- stays the reference's.  All computation goes through the C ABI
// (include/amrx.h) to libamrx.so on the GPU; there is no CPU fallback.
//
// Error mapping (amrx_status -> the reference's exception types):
//   AMRX_ERR_LOAD -> LoadError, AMRX_ERR_INVALID_ARG -> invalid_argument,
//   AMRX_ERR_LENGTH -> length_error, AMRX_ERR_INTERNAL -> logic_error,
//   AMRX_ERR_IO -> runtime_error (the message as is), anything else (CUDA,
//   no device) -> runtime_error.
#include "amriso/io.hpp"
#include "amriso/pipeline.hpp"
#include "amriso/weld.hpp"

#include "amrx.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

namespace amriso {

namespace {

static_assert(sizeof(CellCoord) == 16, "CellCoord must be 4 x int32");
static_assert(sizeof(FatTriangle) == 72, "FatTriangle must be 9 x f64");

[[noreturn]] void rethrow(amrx_status s)
{
  const std::string msg = amrx_last_error();
  switch (s) {
  case AMRX_ERR_LOAD: throw LoadError(msg);
  case AMRX_ERR_INVALID_ARG: throw std::invalid_argument(msg);
  case AMRX_ERR_LENGTH: throw std::length_error(msg);
  case AMRX_ERR_INTERNAL: throw std::logic_error(msg);
  case AMRX_ERR_IO: throw std::runtime_error(msg);  // write_file_atomic's wording
  default: throw std::runtime_error("amrx: " + msg);
  }
}

void check(amrx_status s)
{
  if (s != AMRX_OK) rethrow(s);
}

struct IndexHandle {
  amrx_index *p = nullptr;
  ~IndexHandle()
  {
    if (p) amrx_index_destroy(p);
  }
};

/// a device index over an existing (already sorted) CellIndex
void upload(const CellIndex &index, IndexHandle &h)
{
  amrx_index_opts opts{-1, nullptr, AMRX_FLAG_PRESORTED};
  check(amrx_index_create(reinterpret_cast<const int32_t *>(index.data.cells.data()),
                          index.data.scalars.data(), index.data.cells.size(),
                          index.data.scalars.size(), &opts, &h.p));
}

/*! Device indexes kept alive between calls, so the reference's CLI flow
    build_index -> validate_dataset -> extract_isosurface -> extract_dual_mesh
    (proj/src/cli.cpp:76-118) ingests once.  A CellIndex is immutable after
    build_index, so an entry is keyed on its arrays' addresses
    and size plus a fingerprint of 4096 evenly spaced records and scalars;
    the two most recent datasets are kept. */
struct IndexCache {
  struct Entry {
    const void *cells = nullptr, *scalars = nullptr;
    size_t n = 0;
    uint64_t fp = 0;
    std::shared_ptr<IndexHandle> h;
  };
  std::mutex mu;
  Entry e[2];

  static uint64_t fingerprint(const CellIndex &ix)
  {
    const size_t n = ix.data.cells.size();
    uint64_t f = 0x9e3779b97f4a7c15ull ^ n;
    const auto mix = [&](uint64_t v) {
      f ^= v + 0x9e3779b97f4a7c15ull + (f << 6) + (f >> 2);
    };
    const size_t step = n > 4096 ? n / 4096 : 1;
    for (size_t i = 0; i < n; i += step) {
      const CellCoord &c = ix.data.cells[i];
      uint64_t s;
      std::memcpy(&s, &ix.data.scalars[i], 8);
      mix(uint64_t(uint32_t(c.i)) | uint64_t(uint32_t(c.j)) << 32);
      mix(uint64_t(uint32_t(c.k)) | uint64_t(uint32_t(c.level)) << 32);
      mix(s);
    }
    if (n) {
      uint64_t s;
      std::memcpy(&s, &ix.data.scalars[n - 1], 8);
      mix(s ^ uint64_t(uint32_t(ix.data.cells[n - 1].k)));
    }
    return f;
  }

  /// the device index of `ix`, from the cache or uploaded (presorted)
  std::shared_ptr<IndexHandle> get(const CellIndex &ix)
  {
    const uint64_t fp = fingerprint(ix);
    {
      std::lock_guard<std::mutex> lock(mu);
      for (Entry &x : e)
        if (x.h && x.cells == ix.data.cells.data() && x.scalars == ix.data.scalars.data() &&
            x.n == ix.data.cells.size() && x.fp == fp)
          return x.h;
    }
    auto h = std::make_shared<IndexHandle>();
    upload(ix, *h);
    put(ix, fp, h);
    return h;
  }

  void put(const CellIndex &ix, uint64_t fp, std::shared_ptr<IndexHandle> h)
  {
    std::lock_guard<std::mutex> lock(mu);
    e[1] = std::move(e[0]);
    e[0] = Entry{ix.data.cells.data(), ix.data.scalars.data(), ix.data.cells.size(), fp,
                 std::move(h)};
  }
};

IndexCache &index_cache()
{
  static IndexCache c;
  return c;
}

/*! every GPU of the box (or AMRISO_GPUS of them, like the reference's
    AMRISO_THREADS): with more than one, extract_isosurface and
    extract_dual_mesh run through one amrx_comm (NCCL broadcast of the
    sorted index, each GPU its share of the cells, parts concatenated in
    candidate order) */
struct MultiGpu {
  std::mutex mu;
  amrx_comm *comm = nullptr;
  int gpus = -1;
  // the last dataset's replicated index (same key as IndexCache)
  const void *cells = nullptr, *scalars = nullptr;
  size_t n = 0;
  uint64_t fp = 0;
  amrx_comm_index *index = nullptr;

  ~MultiGpu()
  {
    if (index) amrx_comm_index_destroy(index);
    if (comm) amrx_comm_destroy(comm);
  }

  int count()
  {
    if (gpus < 0) {
      int n = 1;
      if (amrx_device_count(&n) != AMRX_OK) n = 1;
      if (const char *e = std::getenv("AMRISO_GPUS")) {
        const int want = std::atoi(e);
        if (want > 0 && want < n) n = want;
      }
      gpus = n;
    }
    return gpus;
  }

  /// the replicated index of `ix` over all GPUs (mu held)
  amrx_comm_index *get(const CellIndex &ix)
  {
    if (!comm) check(amrx_comm_init(count(), nullptr, &comm));
    const uint64_t f = IndexCache::fingerprint(ix);
    if (index && cells == ix.data.cells.data() && scalars == ix.data.scalars.data() &&
        n == ix.data.cells.size() && fp == f)
      return index;
    if (index) amrx_comm_index_destroy(index);
    index = nullptr;
    check(amrx_comm_index_create(comm, reinterpret_cast<const int32_t *>(ix.data.cells.data()),
                                 ix.data.scalars.data(), ix.data.cells.size(),
                                 ix.data.scalars.size(), AMRX_FLAG_PRESORTED, &index));
    cells = ix.data.cells.data();
    scalars = ix.data.scalars.data();
    n = ix.data.cells.size();
    fp = f;
    return index;
  }
};

MultiGpu &multi_gpu()
{
  static MultiGpu m;
  return m;
}

using Clock = std::chrono::steady_clock;

double seconds_since(Clock::time_point t)
{
  return std::chrono::duration<double>(Clock::now() - t).count();
}

}  // namespace

namespace {

/// the host CellIndex of a device index (tests read index.data directly)
CellIndex host_index(IndexHandle &h)
{
  amrx_index_info info;
  check(amrx_index_get_info(h.p, &info));
  CellIndex index;
  index.data.cells.resize(info.cell_count);
  index.data.scalars.resize(info.cell_count);
  check(amrx_index_download(h.p, reinterpret_cast<int32_t *>(index.data.cells.data()),
                            index.data.scalars.data()));
  index.data.max_level = info.max_level;
  index.data.bounds = {{info.bounds_lo[0], info.bounds_lo[1], info.bounds_lo[2]},
                       {info.bounds_hi[0], info.bounds_hi[1], info.bounds_hi[2]}};
  index.levels.assign(info.levels, info.levels + info.level_count);
  return index;
}

}  // namespace

CellIndex build_index(std::vector<CellCoord> cells, std::vector<double> scalars)
{
  auto h = std::make_shared<IndexHandle>();
  check(amrx_index_create(reinterpret_cast<const int32_t *>(cells.data()),
                          scalars.data(), cells.size(), scalars.size(), nullptr,
                          &h->p));
  CellIndex index = host_index(*h);
  // the returned CellIndex keeps these arrays (moved out, same addresses)
  index_cache().put(index, IndexCache::fingerprint(index), std::move(h));
  return index;
}

CellIndex read_amr(const std::filesystem::path &path)
{
  auto h = std::make_shared<IndexHandle>();
  check(amrx_read_amr(path.c_str(), nullptr, &h->p));
  CellIndex index = host_index(*h);
  index_cache().put(index, IndexCache::fingerprint(index), std::move(h));
  return index;
}

static_assert(sizeof(vec3d) == 24, "vec3d must be 3 x f64");

void write_obj(const IndexedMesh &mesh, const std::filesystem::path &path)
{
  check(amrx_write_obj(path.c_str(), mesh.vertices.empty() ? nullptr : &mesh.vertices[0].x,
                       mesh.vertices.size(),
                       mesh.triangles.empty() ? nullptr : mesh.triangles.data()->data(),
                       mesh.triangles.size(), 0));
}

void write_ply(const IndexedMesh &mesh, const std::filesystem::path &path)
{
  check(amrx_write_ply(path.c_str(), mesh.vertices.empty() ? nullptr : &mesh.vertices[0].x,
                       mesh.vertices.size(),
                       mesh.triangles.empty() ? nullptr : mesh.triangles.data()->data(),
                       mesh.triangles.size(), 0));
}

void write_dual_mesh(const std::vector<DualCell> &duals, const CellIndex &index,
                     const std::filesystem::path &path)
{
  std::vector<uint32_t> corners(duals.size() * 8);
  for (size_t d = 0; d < duals.size(); d++)
    for (int k = 0; k < 8; k++) corners[8 * d + k] = duals[d].corners[k].index;
  check(amrx_write_dual_mesh(path.c_str(), corners.data(), duals.size(),
                             reinterpret_cast<const int32_t *>(index.data.cells.data()),
                             index.data.scalars.data(), index.size(), 0));
}

std::vector<DualCell> extract_dual_mesh(const CellIndex &index, int)
{
  if (index.size() == 0)
    throw std::invalid_argument("extract_dual_mesh: empty dataset");
  static_assert(sizeof(DualCell) == 64, "DualCell must be 8 x u32 + 3 x i64 + i32 + u32");
  uint64_t count = 0;
  amrx_stats st;
  MultiGpu &mg = multi_gpu();
  if (mg.count() <= 1) {
    // the DualCell records are built on the device and land in the vector
    // with one copy (pipeline.cpp:160-194)
    const auto hp = index_cache().get(index);
    IndexHandle &h = *hp;
    check(amrx_extract_dual_cells(h.p, nullptr, nullptr, 0, &count, &st));
    std::vector<DualCell> duals(count);
    if (count) check(amrx_extract_dual_cells(h.p, nullptr, duals.data(), count, &count, &st));
    return duals;
  }
  std::vector<uint32_t> corners;
  std::vector<uint64_t> tasks;
  {
    std::lock_guard<std::mutex> lock(mg.mu);
    amrx_comm_index *m = mg.get(index);
    check(amrx_comm_extract_dual(m, nullptr, nullptr, 0, &count, &st));
    corners.resize(count * 8);
    tasks.resize(count);
    if (count)
      check(amrx_comm_extract_dual(m, corners.data(), tasks.data(), count, &count, &st));
  }
  std::vector<DualCell> duals(count);
  // DualCell{corners, base, level, owner} from the corner ids and the task
  // id owner*8+delta (dual_base_of, dual.hpp:61-67), on every host core
  const auto fill = [&](uint64_t lo, uint64_t hi) {
    for (uint64_t n = lo; n < hi; n++) {
      DualCell &d = duals[n];
      const uint32_t owner = uint32_t(tasks[n] >> 3);
      const int delta = int(tasks[n] & 7);
      const CellCoord &c = index.data.cells[owner];
      for (int k = 0; k < 8; k++) d.corners[k] = CellId{corners[8 * n + k]};
      d.base = dual_base_of(c, delta);
      d.level = c.level;
      d.owner = CellId{owner};
    }
  };
  const unsigned nt = count > (1u << 20) ? std::max(1u, std::thread::hardware_concurrency()) : 1u;
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nt; t++) th.emplace_back(fill, count * t / nt, count * (t + 1) / nt);
  fill(0, count / nt);
  for (auto &x : th) x.join();
  return duals;
}

ExtractionResult extract_isosurface(const CellIndex &index, const IsoParams &params)
{
  if (index.size() == 0)
    throw std::invalid_argument("extract_isosurface: empty dataset");

  ExtractionResult result;
  ExtractionStats &stats = result.stats;
  amrx_iso_params p{params.iso, 0, 1};
  uint64_t count = 0;
  amrx_stats st;
  MultiGpu &mg = multi_gpu();
  if (mg.count() > 1) {
    // every GPU extracts its share; the soup meets on the host and is
    // welded on the first GPU
    std::vector<FatTriangle> fat;
    {
      std::lock_guard<std::mutex> lock(mg.mu);
      amrx_comm_index *m = mg.get(index);
      check(amrx_comm_extract_iso(m, &p, nullptr, 0, &count, &st));
      fat.resize(count);
      if (count) check(amrx_comm_extract_iso(m, &p, fat.data(), count, &count, &st));
    }
    const auto t_weld = Clock::now();
    result.mesh = weld(fat);
    stats.seconds_weld = seconds_since(t_weld);
  } else {
    // passes 1+2 and the weld on the device (pipeline.cpp:67-158): only the
    // indexed mesh crosses to the host; the soup stays in the index's arena
    const auto hp = index_cache().get(index);
    IndexHandle &h = *hp;
    uint64_t nv = 0;
    double t_weld = 0;
    check(amrx_extract_iso_mesh(h.p, nullptr, &p, nullptr, 0, nullptr, 0, &nv, &count, &t_weld,
                                &st));
    result.mesh.vertices.resize(nv);
    result.mesh.triangles.resize(count);
    if (nv || count)
      check(amrx_extract_iso_mesh(
        h.p, nullptr, &p, nv ? &result.mesh.vertices[0].x : nullptr, nv,
        count ? result.mesh.triangles.data()->data() : nullptr, count, &nv, &count, &t_weld,
        &st));
    stats.seconds_weld = t_weld;
  }

  stats.cell_count = st.cell_count;
  stats.duals_accepted = st.duals_accepted;
  stats.duals_missing_corner = st.duals_missing_corner;
  stats.duals_finer_corner = st.duals_finer_corner;
  stats.duals_lower_key_corner = st.duals_lower_key_corner;
  stats.pass1_triangle_count = st.pass1_triangle_count;
  stats.fat_triangle_count = st.fat_triangle_count;
  stats.seconds_pass1 = st.seconds_pass1;
  stats.seconds_pass2 = st.seconds_pass2;
  stats.welded_vertex_count = result.mesh.vertices.size();
  stats.welded_triangle_count = result.mesh.triangles.size();

  if (params.emit_dual_mesh) result.duals = extract_dual_mesh(index, params.thread_count);
  return result;
}

ValidationReport validate_dataset(const CellIndex &index)
{
  ValidationReport report;
  if (index.size() == 0) return report;
  const auto hp = index_cache().get(index);
  IndexHandle &h = *hp;
  uint64_t nd = 0, no = 0;
  check(amrx_validate(h.p, nullptr, 0, &nd, nullptr, 0, &no));
  std::vector<uint32_t> dup(2 * nd), ovl(2 * no);
  check(amrx_validate(h.p, nd ? dup.data() : nullptr, nd, &nd, no ? ovl.data() : nullptr, no,
                      &no));
  for (uint64_t n = 0; n < nd; n++)
    report.duplicates.push_back({CellId{dup[2 * n]}, CellId{dup[2 * n + 1]}});
  for (uint64_t n = 0; n < no; n++)
    report.overlaps.push_back({CellId{ovl[2 * n]}, CellId{ovl[2 * n + 1]}});
  return report;
}

IndexedMesh weld(std::span<const FatTriangle> triangles)
{
  IndexedMesh mesh;
  if (triangles.empty()) return mesh;
  const uint64_t n = triangles.size();
  if (n > std::numeric_limits<uint32_t>::max() / 3)
    throw std::length_error("weld: too many triangles for 32-bit indices");
  std::vector<vec3d> verts(3 * n);
  mesh.triangles.resize(n);
  uint64_t nv = 0;
  check(amrx_weld(reinterpret_cast<const double *>(triangles.data()), n,
                  reinterpret_cast<double *>(verts.data()), 3 * n,
                  reinterpret_cast<uint32_t *>(mesh.triangles.data()), &nv, nullptr));
  verts.resize(nv);
  mesh.vertices = std::move(verts);
  return mesh;
}

}  // namespace amriso
