// The reference CLI's flow (proj/src/cli.cpp:76-118: read -> validate ->
// extract -> dual mesh) through the reference's own C++ API, timed.  Built
// twice by oracle/Makefile: against the unmodified reference sources
// (amriso_ref_bench) and against the GPU drop-in shim + libamrx.so
// (amriso_dropin_bench), so the two implementations run the identical caller.
//
//   amriso_*_bench <cells.amr> <iso> [reps]   -> one JSON line on stdout
#include "amriso/io.hpp"
#include "amriso/locator.hpp"
#include "amriso/pipeline.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

using namespace amriso;

namespace {
double since(std::chrono::steady_clock::time_point t)
{
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}
}  // namespace

int main(int argc, char **argv)
{
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s <cells.amr> <iso> [reps]\n", argv[0]);
    return 2;
  }
  const std::string path = argv[1];
  const double iso = std::atof(argv[2]);
  const int reps = argc > 3 ? std::atoi(argv[3]) : 2;
  auto t = std::chrono::steady_clock::now();
  CellIndex index = read_amr(path);
  const double t_read = since(t);
  t = std::chrono::steady_clock::now();
  const ValidationReport rep = validate_dataset(index);
  const double t_validate = since(t);
  IsoParams p;
  p.iso = iso;
  double t_iso_first = 0, t_iso = 1e30, t_dual_first = 0, t_dual = 1e30;
  uint64_t tris = 0, verts = 0, duals = 0, accepted = 0;
  for (int r = 0; r <= reps; r++) {
    t = std::chrono::steady_clock::now();
    ExtractionResult res = extract_isosurface(index, p);
    const double ti = since(t);
    t = std::chrono::steady_clock::now();
    const std::vector<DualCell> d = extract_dual_mesh(index, 0);
    const double td = since(t);
    if (r == 0) {
      t_iso_first = ti;
      t_dual_first = td;
    } else {
      t_iso = ti < t_iso ? ti : t_iso;
      t_dual = td < t_dual ? td : t_dual;
    }
    tris = res.mesh.triangles.size();
    verts = res.mesh.vertices.size();
    accepted = res.stats.duals_accepted;
    duals = d.size();
  }
  std::printf("{\"cells\": %zu, \"valid\": %s, \"triangles\": %llu, \"vertices\": %llu, "
              "\"duals\": %llu, \"duals_accepted\": %llu, \"seconds\": {\"read_amr\": %.6f, "
              "\"validate_dataset\": %.6f, \"extract_isosurface_first\": %.6f, "
              "\"extract_isosurface\": %.6f, \"extract_dual_mesh_first\": %.6f, "
              "\"extract_dual_mesh\": %.6f}}\n",
              index.size(), rep.duplicates.empty() && rep.overlaps.empty() ? "true" : "false",
              (unsigned long long)tris, (unsigned long long)verts, (unsigned long long)duals,
              (unsigned long long)accepted, t_read, t_validate, t_iso_first,
              reps ? t_iso : t_iso_first, t_dual_first, reps ? t_dual : t_dual_first);
  return 0;
}
