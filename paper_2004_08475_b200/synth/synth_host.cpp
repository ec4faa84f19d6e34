// Host generators for the small configurations, matching the reference's
// generators record for record (same libstdc++ <random>, same expression
// order, -ffp-contract=off), so the bench and the GPU tests can build their
// inputs without the reference tree:
//
//   amrxs_octree_sphere  gen_octree + FieldSpec::sphere   proj/src/synth.cpp:105-181
//   amrxs_uniform        gen_uniform                      proj/src/synth.cpp:122-137
//   amrxs_slots          random_slot_dataset              proj/tests/fixtures.hpp:38-69
//
// Output is the generator's record order (the cell list BEFORE build_index
// sorts it) -- exactly what a caller hands the library.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>
#include <vector>

#define AMRXS_API extern "C" __attribute__((visibility("default")))

namespace {

struct Sphere {
  double cx, cy, cz, r;
  double eval(double x, double y, double z) const
  {
    const double dx = x - cx, dy = y - cy, dz = z - cz;
    return std::sqrt(dx * dx + dy * dy + dz * dz) - r;
  }
};

struct Out {
  std::vector<int32_t> cells;
  std::vector<double> scalars;
  void push(int32_t i, int32_t j, int32_t k, int32_t l, double s)
  {
    cells.insert(cells.end(), {i, j, k, l});
    scalars.push_back(s);
  }
};

double centre(int32_t a, int32_t level)
{
  const double half = 0.5 * double(int64_t(1) << level);
  return double(a) + half;
}

double field_range(const Sphere &f, int32_t i, int32_t j, int32_t k, int32_t l)
{
  const int64_t w = int64_t(1) << l;
  double lo = std::numeric_limits<double>::infinity();
  double hi = -std::numeric_limits<double>::infinity();
  for (int d = 0; d < 8; d++) {
    const double x = double((d & 1) ? i + w : i);
    const double y = double((d & 2) ? j + w : j);
    const double z = double((d & 4) ? k + w : k);
    const double v = f.eval(x, y, z);
    lo = std::min(lo, v);
    hi = std::max(hi, v);
  }
  return hi - lo;
}

void visit(const Sphere &f, double thr, int32_t i, int32_t j, int32_t k,
           int32_t l, Out &o)
{
  if (l > 0 && field_range(f, i, j, k, l) > thr) {
    const int32_t half = int32_t((int64_t(1) << l) / 2);
    for (int d = 0; d < 8; d++)
      visit(f, thr, i + ((d & 1) ? half : 0), j + ((d & 2) ? half : 0),
            k + ((d & 4) ? half : 0), l - 1, o);
  } else {
    o.push(i, j, k, l, f.eval(centre(i, l), centre(j, l), centre(k, l)));
  }
}

struct Result {
  uint64_t n;
  int32_t *cells;
  double *scalars;
};

Result *finish(Out &o)
{
  auto *r = static_cast<Result *>(std::malloc(sizeof(Result)));
  r->n = o.scalars.size();
  r->cells = static_cast<int32_t *>(std::malloc(o.cells.size() * 4 + 16));
  r->scalars = static_cast<double *>(std::malloc(o.scalars.size() * 8 + 16));
  std::memcpy(r->cells, o.cells.data(), o.cells.size() * 4);
  std::memcpy(r->scalars, o.scalars.data(), o.scalars.size() * 8);
  return r;
}

}  // namespace

AMRXS_API void *amrxs_octree_sphere(int32_t depth, double cx, double cy,
                                    double cz, double r, double threshold)
{
  Out o;
  visit(Sphere{cx, cy, cz, r}, threshold, 0, 0, 0, depth, o);
  return finish(o);
}

AMRXS_API void *amrxs_uniform_sphere(int32_t n, double cx, double cy,
                                     double cz, double r)
{
  Out o;
  const Sphere f{cx, cy, cz, r};
  for (int32_t k = 0; k < n; k++)
    for (int32_t j = 0; j < n; j++)
      for (int32_t i = 0; i < n; i++)
        o.push(i, j, k, 0, f.eval(centre(i, 0), centre(j, 0), centre(k, 0)));
  return finish(o);
}

AMRXS_API void *amrxs_slots(uint32_t seed, int slots, int max_level,
                            double hole_prob)
{
  Out o;
  std::mt19937 rng(seed);
  const int64_t W = int64_t(1) << max_level;
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  std::uniform_int_distribution<int> pick_level(0, max_level);
  std::uniform_real_distribution<double> unit(-1.0, 1.0);
  for (int sz = 0; sz < slots; sz++)
    for (int sy = 0; sy < slots; sy++)
      for (int sx = 0; sx < slots; sx++) {
        if (u01(rng) < hole_prob) continue;
        const int32_t level = pick_level(rng);
        const int64_t w = int64_t(1) << level;
        for (int64_t dz = 0; dz < W; dz += w)
          for (int64_t dy = 0; dy < W; dy += w)
            for (int64_t dx = 0; dx < W; dx += w)
              o.push(int32_t(sx * W + dx), int32_t(sy * W + dy),
                     int32_t(sz * W + dz), level, unit(rng));
      }
  if (o.scalars.empty()) o.push(0, 0, 0, max_level, 0.5);
  return finish(o);
}

AMRXS_API uint64_t amrxs_size(void *h) { return static_cast<Result *>(h)->n; }

AMRXS_API void amrxs_get(void *h, int32_t *cells4, double *scalars)
{
  auto *r = static_cast<Result *>(h);
  if (cells4) std::memcpy(cells4, r->cells, r->n * 16);
  if (scalars) std::memcpy(scalars, r->scalars, r->n * 8);
}

AMRXS_API void amrxs_free(void *h)
{
  auto *r = static_cast<Result *>(h);
  if (!r) return;
  std::free(r->cells);
  std::free(r->scalars);
  std::free(r);
}
