// TEST ORACLE INFRASTRUCTURE -- never linked into the product.
//
// C entry points over the *unmodified* reference library (the amriso
// sources under /root/reference/proj/src, compiled in place by
// oracle/Makefile into oracle/_ref/libamriso_ref.so).  Python tests and
// bench.py's cpu_baseline leg drive the reference through these via
// ctypes.  Everything here is glue: all arithmetic is the reference's.
//
// Reference interfaces wrapped (file:line under /root/reference/):
//   build_index            proj/src/locator.cpp:26-92
//   find_exact / snap      proj/src/locator.cpp:94-134
//   validate_dataset       proj/src/locator.cpp:136-161
//   try_build_dual         proj/src/dual.cpp:41-72
//   extract_dual_mesh      proj/src/pipeline.cpp:160-194
//   extract_isosurface     proj/src/pipeline.cpp:67-158
//   contour_hex            proj/src/contour.cpp:52-87
//   gen_uniform/octree/blocks, exhaustive_duals  proj/src/synth.cpp
//   random_slot_dataset    proj/tests/fixtures.hpp:38-69
//   make_random_fixtures   proj/tests/acceptance.cpp:64-136 (restated below,
//                          same rng consumption order)

#include "fixtures.hpp"

#include "amriso/io.hpp"
#include "amriso/mc_tables.hpp"
#include "amriso/pipeline.hpp"

#include <chrono>
#include <cstring>
#include <memory>
#include <random>
#include <string>

using namespace amriso;

namespace {

  thread_local std::string g_error;

  struct RefIndex {
    CellIndex index;
  };

  struct RefIso {
    ExtractionResult result;
  };

  struct RefDuals {
    std::vector<DualCell> duals;
  };

  struct RefKeys {
    std::vector<DualKey> keys;
  };

  RefIndex *wrap(CellIndex &&index)
  {
    return new RefIndex{std::move(index)};
  }

  template <typename Fn>
  auto guarded(Fn &&fn) -> decltype(fn())
  {
    try {
      return fn();
    } catch (const LoadError &e) {
      g_error = std::string("LoadError: ") + e.what();
    } catch (const std::invalid_argument &e) {
      g_error = std::string("invalid_argument: ") + e.what();
    } catch (const std::length_error &e) {
      g_error = std::string("length_error: ") + e.what();
    } catch (const std::logic_error &e) {
      g_error = std::string("logic_error: ") + e.what();
    } catch (const std::exception &e) {
      g_error = std::string("exception: ") + e.what();
    }
    return decltype(fn())();
  }

  FieldSpec field_of(int kind, const double *p)
  {
    switch (kind) {
    case 0: return FieldSpec::sphere({p[0], p[1], p[2]}, p[3]);
    case 1: return FieldSpec::linear({p[0], p[1], p[2]}, p[3]);
    default: return FieldSpec::radial_sine({p[0], p[1], p[2]}, p[3]);
    }
  }

  /*! acceptance.cpp:64-136 -- the 100 randomized fixtures, same rng
      consumption order, so fixture n here is fixture n there */
  struct AcceptFixture {
    CellIndex index;
    double iso;
  };

  std::vector<AcceptFixture> make_random_fixtures()
  {
    std::vector<AcceptFixture> fixtures;
    std::mt19937 rng(20260825);
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    for (int n = 0; n < 100; n++) {
      switch (n % 3) {
      case 0: {
        // function-argument evaluation order is unspecified in C++, and
        // it decides the rng stream here: keep the reference's exact
        // call shape so g++ orders the draws the same way
        const FieldSpec field =
          FieldSpec::sphere({0.5 + 3.0 * u01(rng), 0.5 + 3.0 * u01(rng),
                             0.5 + 3.0 * u01(rng)},
                            0.5 + 1.5 * u01(rng));
        const double thr = 0.3 + 2.0 * u01(rng);
        fixtures.push_back({gen_octree(2, field, thr), 0.0});
        break;
      }
      case 1: {
        const int split = 4 * (1 + int(rng() % 3));
        const int axis = int(rng() % 3);
        const int fine_level = int(rng() % 2);
        const int wf = 1 << fine_level;
        BlockSpec coarse{{0, 0, 0}, {4, 4, 4}, 2};
        BlockSpec fine{{0, 0, 0}, {16 / wf, 16 / wf, 16 / wf},
                       int32_t(fine_level)};
        switch (axis) {
        case 0:
          coarse.size.x = split / 4;
          fine.anchor.x = split;
          fine.size.x = (16 - split) / wf;
          break;
        case 1:
          coarse.size.y = split / 4;
          fine.anchor.y = split;
          fine.size.y = (16 - split) / wf;
          break;
        default:
          coarse.size.z = split / 4;
          fine.anchor.z = split;
          fine.size.z = (16 - split) / wf;
          break;
        }
        std::vector<Box3l> holes;
        const int hole_count = int(rng() % 3);
        for (int h = 0; h < hole_count; h++) {
          const vec3l lo{int64_t(rng() % 13), int64_t(rng() % 13),
                         int64_t(rng() % 13)};
          const int64_t s = 2 + int64_t(rng() % 3);
          holes.push_back({lo, {lo.x + s, lo.y + s, lo.z + s}});
        }
        const vec3d g{u01(rng) - 0.5, u01(rng) - 0.5, u01(rng) - 0.5};
        const FieldSpec field =
          FieldSpec::linear(g, -8.0 * (g.x + g.y + g.z));
        fixtures.push_back({gen_blocks({coarse, fine}, field, holes), 0.0});
        break;
      }
      default:
        fixtures.push_back({testing::random_slot_dataset(rng, 4, 2), 0.1});
        break;
      }
    }
    return fixtures;
  }

  double now_s()
  {
    return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
  }

} // namespace

extern "C" {

const char *ref_last_error() { return g_error.c_str(); }

// ---------------------------------------------------------------- index
void *ref_build_index(const int32_t *cells4, const double *scalars,
                      uint64_t n, uint64_t n_scalars)
{
  return guarded([&]() -> void * {
    std::vector<CellCoord> cells(n);
    for (uint64_t c = 0; c < n; c++)
      cells[c] = {cells4[4 * c], cells4[4 * c + 1], cells4[4 * c + 2],
                  cells4[4 * c + 3]};
    std::vector<double> s(scalars, scalars + n_scalars);
    return wrap(build_index(std::move(cells), std::move(s)));
  });
}

void ref_index_free(void *h) { delete static_cast<RefIndex *>(h); }

uint64_t ref_index_size(void *h)
{
  return static_cast<RefIndex *>(h)->index.size();
}

void ref_index_get(void *h, int32_t *cells4, double *scalars)
{
  const CellIndex &idx = static_cast<RefIndex *>(h)->index;
  for (size_t c = 0; c < idx.size(); c++) {
    const CellCoord &cc = idx.data.cells[c];
    cells4[4 * c + 0] = cc.i;
    cells4[4 * c + 1] = cc.j;
    cells4[4 * c + 2] = cc.k;
    cells4[4 * c + 3] = cc.level;
    scalars[c] = idx.data.scalars[c];
  }
}

/// levels finest first into out[<=31]; returns the count
int ref_index_levels(void *h, int32_t *out)
{
  const CellIndex &idx = static_cast<RefIndex *>(h)->index;
  for (size_t n = 0; n < idx.levels.size(); n++)
    out[n] = idx.levels[n];
  return int(idx.levels.size());
}

/// bounds lo.xyz, hi.xyz then max_level
void ref_index_bounds(void *h, int64_t *out7)
{
  const CellIndex &idx = static_cast<RefIndex *>(h)->index;
  const Box3l &b = idx.data.bounds;
  out7[0] = b.lo.x; out7[1] = b.lo.y; out7[2] = b.lo.z;
  out7[3] = b.hi.x; out7[4] = b.hi.y; out7[5] = b.hi.z;
  out7[6] = idx.data.max_level;
}

// ----------------------------------------------------------- generators
void *ref_gen_uniform(int32_t n, int field_kind, const double *field4)
{
  return guarded([&]() -> void * {
    return wrap(gen_uniform(n, field_of(field_kind, field4)));
  });
}

void *ref_gen_octree(int32_t depth, int field_kind, const double *field4,
                     double threshold)
{
  return guarded([&]() -> void * {
    return wrap(gen_octree(depth, field_of(field_kind, field4), threshold));
  });
}

/// blocks: n_blocks x {ax,ay,az,sx,sy,sz,level}; holes: n_holes x lo3,hi3
void *ref_gen_blocks(const int32_t *blocks7, int n_blocks, int field_kind,
                     const double *field4, const int64_t *holes6,
                     int n_holes)
{
  return guarded([&]() -> void * {
    std::vector<BlockSpec> blocks(n_blocks);
    for (int b = 0; b < n_blocks; b++) {
      const int32_t *p = blocks7 + 7 * b;
      blocks[b] = {{p[0], p[1], p[2]}, {p[3], p[4], p[5]}, p[6]};
    }
    std::vector<Box3l> holes(n_holes);
    for (int h = 0; h < n_holes; h++) {
      const int64_t *p = holes6 + 6 * h;
      holes[h] = {{p[0], p[1], p[2]}, {p[3], p[4], p[5]}};
    }
    return wrap(gen_blocks(blocks, field_of(field_kind, field4), holes));
  });
}

void *ref_gen_slots(uint32_t seed, int slots, int max_level,
                    double hole_prob)
{
  return guarded([&]() -> void * {
    std::mt19937 rng(seed);
    return wrap(testing::random_slot_dataset(rng, slots, max_level,
                                             hole_prob));
  });
}

/*! fixture n (0..99) of acceptance.cpp's randomized pool, plus
    100 = sphere16 and 101 = octree_sphere (acceptance.cpp:140-159);
    *iso receives the fixture's iso value */
void *ref_acceptance_fixture(int n, double *iso)
{
  return guarded([&]() -> void * {
    if (n == 100) {
      *iso = 0.0;
      return wrap(gen_uniform(16, FieldSpec::sphere({8, 8, 8}, 5.0)));
    }
    if (n == 101) {
      *iso = 0.0;
      return wrap(gen_octree(4, FieldSpec::sphere({5, 6, 7}, 3.5), 3.0));
    }
    auto fixtures = make_random_fixtures();
    *iso = fixtures.at(size_t(n)).iso;
    return wrap(std::move(fixtures.at(size_t(n)).index));
  });
}

// -------------------------------------------------------------- queries
/// returns the CellId or -1
int64_t ref_snap(void *h, const int64_t *p3, int32_t hint)
{
  const auto hit =
    snap(static_cast<RefIndex *>(h)->index, {p3[0], p3[1], p3[2]}, hint);
  return hit ? int64_t(hit->index) : -1;
}

int64_t ref_find_exact(void *h, const int32_t *c4)
{
  const auto hit = find_exact(static_cast<RefIndex *>(h)->index,
                              {c4[0], c4[1], c4[2], c4[3]});
  return hit ? int64_t(hit->index) : -1;
}

/// returns the DualReject code; corners8 filled when accepted
int ref_try_build_dual(void *h, const int64_t *base3, int32_t level,
                       uint32_t self, uint32_t *corners8)
{
  DualReject why = DualReject::accepted;
  const auto dual = try_build_dual(static_cast<RefIndex *>(h)->index,
                                   {base3[0], base3[1], base3[2]}, level,
                                   CellId{self}, &why);
  if (dual)
    for (int d = 0; d < 8; d++)
      corners8[d] = dual->corners[d].index;
  return int(why);
}

/// validate_dataset: returns duplicates+overlaps count, fills the split
int64_t ref_validate(void *h, uint64_t *dups, uint64_t *overlaps)
{
  const ValidationReport r =
    validate_dataset(static_cast<RefIndex *>(h)->index);
  *dups = r.duplicates.size();
  *overlaps = r.overlaps.size();
  return int64_t(r.duplicates.size() + r.overlaps.size());
}

/// validate_dataset pairs: dup2 / ovl2 (2 x u32 each, may be null) get the
/// first `cap` pairs of each list
void ref_validate_pairs(void *h, uint32_t *dup2, uint32_t *ovl2, uint64_t cap)
{
  const ValidationReport r =
    validate_dataset(static_cast<RefIndex *>(h)->index);
  for (size_t n = 0; dup2 && n < r.duplicates.size() && n < cap; n++) {
    dup2[2 * n] = r.duplicates[n].first.index;
    dup2[2 * n + 1] = r.duplicates[n].second.index;
  }
  for (size_t n = 0; ovl2 && n < r.overlaps.size() && n < cap; n++) {
    ovl2[2 * n] = r.overlaps[n].first.index;
    ovl2[2 * n + 1] = r.overlaps[n].second.index;
  }
}

// ----------------------------------------------------------- dual mesh
void *ref_extract_dual(void *h, int threads, double *seconds)
{
  return guarded([&]() -> void * {
    const double t0 = now_s();
    auto *r = new RefDuals{
      extract_dual_mesh(static_cast<RefIndex *>(h)->index, threads)};
    if (seconds) *seconds = now_s() - t0;
    return r;
  });
}

uint64_t ref_duals_count(void *r)
{
  return static_cast<RefDuals *>(r)->duals.size();
}

/// corners8 (u32), base3 (i64), level (i32), owner (u32) per dual
void ref_duals_get(void *r, uint32_t *corners8, int64_t *base3,
                   int32_t *level, uint32_t *owner)
{
  const auto &duals = static_cast<RefDuals *>(r)->duals;
  for (size_t n = 0; n < duals.size(); n++) {
    const DualCell &d = duals[n];
    for (int c = 0; c < 8; c++)
      corners8[8 * n + c] = d.corners[c].index;
    if (base3) {
      base3[3 * n + 0] = d.base.x;
      base3[3 * n + 1] = d.base.y;
      base3[3 * n + 2] = d.base.z;
    }
    if (level) level[n] = d.level;
    if (owner) owner[n] = d.owner.index;
  }
}

void ref_duals_free(void *r) { delete static_cast<RefDuals *>(r); }

/// exhaustive_duals (synth.cpp:238-282); returns a RefKeys handle
void *ref_exhaustive_duals(void *h)
{
  return guarded([&]() -> void * {
    const auto keys = exhaustive_duals(static_cast<RefIndex *>(h)->index);
    return new RefKeys{std::vector<DualKey>(keys.begin(), keys.end())};
  });
}

uint64_t ref_keys_count(void *r)
{
  return static_cast<RefKeys *>(r)->keys.size();
}

void ref_keys_get(void *r, uint32_t *keys8)
{
  const auto &keys = static_cast<RefKeys *>(r)->keys;
  for (size_t n = 0; n < keys.size(); n++)
    for (int c = 0; c < 8; c++)
      keys8[8 * n + c] = keys[n][c];
}

void ref_keys_free(void *r) { delete static_cast<RefKeys *>(r); }

// ---------------------------------------------------------- iso-surface
void *ref_extract_iso(void *h, double iso, int threads, int emit_dual)
{
  return guarded([&]() -> void * {
    IsoParams p;
    p.iso = iso;
    p.thread_count = threads;
    p.emit_dual_mesh = emit_dual != 0;
    return new RefIso{
      extract_isosurface(static_cast<RefIndex *>(h)->index, p)};
  });
}

/*! stats: cell_count, accepted, missing, finer, lower_key, pass1 tris,
    fat tris, welded vertices, welded triangles (9 u64) and seconds
    sort, pass1, pass2, weld (4 f64) */
void ref_iso_stats(void *r, uint64_t *u9, double *t4)
{
  const ExtractionStats &s = static_cast<RefIso *>(r)->result.stats;
  u9[0] = s.cell_count;
  u9[1] = s.duals_accepted;
  u9[2] = s.duals_missing_corner;
  u9[3] = s.duals_finer_corner;
  u9[4] = s.duals_lower_key_corner;
  u9[5] = s.pass1_triangle_count;
  u9[6] = s.fat_triangle_count;
  u9[7] = s.welded_vertex_count;
  u9[8] = s.welded_triangle_count;
  if (t4) {
    t4[0] = s.seconds_sort;
    t4[1] = s.seconds_pass1;
    t4[2] = s.seconds_pass2;
    t4[3] = s.seconds_weld;
  }
}

/*! the fat triangle soup in emission order, 9 doubles per triangle.
    weld keeps triangle order and exact positions (weld.cpp:56-62), so
    expanding the welded mesh reproduces pass 2's soup bit for bit */
void ref_iso_fat(void *r, double *xyz9)
{
  const IndexedMesh &m = static_cast<RefIso *>(r)->result.mesh;
  for (size_t t = 0; t < m.triangles.size(); t++)
    for (int c = 0; c < 3; c++) {
      const vec3d &v = m.vertices[m.triangles[t][c]];
      xyz9[9 * t + 3 * c + 0] = v.x;
      xyz9[9 * t + 3 * c + 1] = v.y;
      xyz9[9 * t + 3 * c + 2] = v.z;
    }
}

/// welded mesh: vertices (3 f64 each) and triangles (3 u32 each)
void ref_iso_mesh(void *r, double *verts3, uint32_t *tris3)
{
  const IndexedMesh &m = static_cast<RefIso *>(r)->result.mesh;
  for (size_t v = 0; v < m.vertices.size(); v++) {
    verts3[3 * v + 0] = m.vertices[v].x;
    verts3[3 * v + 1] = m.vertices[v].y;
    verts3[3 * v + 2] = m.vertices[v].z;
  }
  for (size_t t = 0; t < m.triangles.size(); t++)
    for (int c = 0; c < 3; c++)
      tris3[3 * t + c] = m.triangles[t][c];
}

/// OBJ text of the welded mesh (io.cpp:225-238); caller frees with free()
char *ref_iso_obj(void *r)
{
  const std::string s = obj_string(static_cast<RefIso *>(r)->result.mesh);
  char *out = static_cast<char *>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

uint64_t ref_iso_dual_count(void *r)
{
  return static_cast<RefIso *>(r)->result.duals.size();
}

void ref_iso_free(void *r) { delete static_cast<RefIso *>(r); }

/*! weld (weld.cpp:31-64) of an arbitrary soup; returns a RefIso handle
    whose mesh is the welded result */
void *ref_weld(const double *xyz9, uint64_t n_tris)
{
  return guarded([&]() -> void * {
    std::vector<FatTriangle> fat(n_tris);
    for (uint64_t t = 0; t < n_tris; t++) {
      const double *p = xyz9 + 9 * t;
      fat[t] = {{p[0], p[1], p[2]}, {p[3], p[4], p[5]}, {p[6], p[7], p[8]}};
    }
    auto *r = new RefIso{};
    r->result.mesh = weld(fat);
    return r;
  });
}

uint64_t ref_mesh_sizes(void *r, uint64_t *n_tris)
{
  const IndexedMesh &m = static_cast<RefIso *>(r)->result.mesh;
  *n_tris = m.triangles.size();
  return m.vertices.size();
}

// -------------------------------------------------------------- contour
/*! contour_hex on an explicit hex: cells8 ids, pos24, value8; returns the
    triangle count (-1 on logic_error) and writes up to 5*9 doubles */
int ref_contour_hex(const uint32_t *cells8, const double *pos24,
                    const double *value8, double iso, double *out45)
{
  HexInput hex;
  for (int d = 0; d < 8; d++) {
    hex.cell[d] = CellId{cells8[d]};
    hex.pos[d] = {pos24[3 * d], pos24[3 * d + 1], pos24[3 * d + 2]};
    hex.value[d] = value8[d];
  }
  try {
    const TriangleBatch b = contour_hex(hex, iso);
    for (int t = 0; t < b.count; t++) {
      const FatTriangle &f = b.tri[t];
      const vec3d v[3] = {f.v0, f.v1, f.v2};
      for (int c = 0; c < 3; c++) {
        out45[9 * t + 3 * c + 0] = v[c].x;
        out45[9 * t + 3 * c + 1] = v[c].y;
        out45[9 * t + 3 * c + 2] = v[c].z;
      }
    }
    return b.count;
  } catch (const std::logic_error &e) {
    g_error = e.what();
    return -1;
  }
}

/*! random_degenerate_hex (fixtures.hpp:98-138) stream with seed; writes
    count hexes (cells8, pos24, value8) and one iso per hex drawn as
    acceptance.cpp:289-291 does */
void ref_degenerate_hexes(uint32_t seed, int count, uint32_t *cells8,
                          double *pos24, double *value8, double *iso)
{
  std::mt19937 rng(seed);
  for (int n = 0; n < count; n++) {
    const HexInput hex = testing::random_degenerate_hex(rng);
    iso[n] = testing::unit_scalar(rng);
    for (int d = 0; d < 8; d++) {
      cells8[8 * n + d] = hex.cell[d].index;
      pos24[24 * n + 3 * d + 0] = hex.pos[d].x;
      pos24[24 * n + 3 * d + 1] = hex.pos[d].y;
      pos24[24 * n + 3 * d + 2] = hex.pos[d].z;
      value8[8 * n + d] = hex.value[d];
    }
  }
}

/// MC tables (mc_tables.cpp) for pinning the restatement's copy
void ref_mc_tables(int8_t *tri256x16, uint16_t *edge256, uint8_t *corner8,
                   uint8_t *edge_corner24)
{
  std::memcpy(tri256x16, mc::tri_table, sizeof(mc::tri_table));
  std::memcpy(edge256, mc::edge_table, sizeof(mc::edge_table));
  std::memcpy(corner8, mc::table_corner, sizeof(mc::table_corner));
  std::memcpy(edge_corner24, mc::edge_corner, sizeof(mc::edge_corner));
}

// ---------------------------------------------------------------- writers
// the reference's write_obj / write_ply / write_dual_mesh (io.cpp:235-305)
// on caller arrays; 0 = ok, else ref_last_error()
int ref_write_mesh(const char *path, int ply, const double *verts3, uint64_t nv,
                   const uint32_t *tris3, uint64_t nt)
{
  return guarded([&]() -> void * {
           IndexedMesh m;
           m.vertices.resize(nv);
           for (uint64_t v = 0; v < nv; v++)
             m.vertices[v] = {verts3[3 * v], verts3[3 * v + 1], verts3[3 * v + 2]};
           m.triangles.resize(nt);
           for (uint64_t t = 0; t < nt; t++)
             m.triangles[t] = {tris3[3 * t], tris3[3 * t + 1], tris3[3 * t + 2]};
           if (ply)
             write_ply(m, path);
           else
             write_obj(m, path);
           return reinterpret_cast<void *>(1);
         })
           ? 0
           : 1;
}

int ref_write_dual_mesh(const char *path, const uint32_t *corners8, uint64_t nd,
                        const int32_t *cells4, const double *scalars, uint64_t nc)
{
  return guarded([&]() -> void * {
           CellIndex index;
           index.data.cells.resize(nc);
           for (uint64_t c = 0; c < nc; c++)
             index.data.cells[c] = {cells4[4 * c], cells4[4 * c + 1], cells4[4 * c + 2],
                                    cells4[4 * c + 3]};
           index.data.scalars.assign(scalars, scalars + nc);
           std::vector<DualCell> duals(nd);
           for (uint64_t d = 0; d < nd; d++)
             for (int k = 0; k < 8; k++) duals[d].corners[k] = CellId{corners8[8 * d + k]};
           write_dual_mesh(duals, index, path);
           return reinterpret_cast<void *>(1);
         })
           ? 0
           : 1;
}

} // extern "C"
