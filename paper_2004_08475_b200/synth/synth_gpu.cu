// GPU generator for the large configurations: a
// block-structured 4-level AMR (levels 0..3) over a grid of level-3 bricks
// (8 finest units a side).  Each brick is refined uniformly to the level its
// refinement indicator asks for -- fine near the cores of a set of Gaussian
// vortex tubes -- so neighbouring bricks can jump by up to three levels, and
// bricks that touch the "aircraft body" boxes are holes.  The scalar is a
// vorticity-like field: |omega| of the superposed tubes (Lamb-Oseen cores,
// omega = Gamma/(pi a^2) exp(-r^2/a^2) along each tube axis) plus hashed
// lattice value noise, in FP64 at cell centres.  Optionally the records are
// written in a fixed-seed bijective-hash order (Feistel network with cycle
// walking over [0, N)): the "cell soup" with no hierarchy left in it.
//
// Test-data generation only: not part of the extraction path (libamrx.so).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#define AMRXS_API extern "C" __attribute__((visibility("default")))

namespace {

constexpr int kMaxTubes = 32;

struct Tube {
  double px, py, pz;   // point on the axis
  double dx, dy, dz;   // unit direction
  double a;            // core radius
  double amp;          // Gamma / (pi a^2)
};

struct Params {
  int32_t bricks[3];
  int32_t ntubes;
  Tube tubes[kMaxTubes];
  double t0, t1, t2;       // indicator thresholds for levels 0, 1, 2
  double reach;            // indicator length scale in core radii
  double noise_amp, noise_scale;
  int32_t nholes;
  int64_t holes[4][6];
  uint64_t seed;
};

__host__ __device__ inline uint64_t mix64(uint64_t x)
{
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

__device__ double lattice(int64_t i, int64_t j, int64_t k, uint64_t seed)
{
  const uint64_t h = mix64(seed ^ mix64(uint64_t(i) * 0x9E3779B97F4A7C15ull ^
                                        mix64(uint64_t(j) * 0xC2B2AE3D27D4EB4Full ^
                                              uint64_t(k) * 0x165667B19E3779F9ull)));
  return double(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

__device__ double smooth(double t) { return t * t * (3.0 - 2.0 * t); }

/// trilinear value noise with smoothstep weights, lattice spacing `scale`
__device__ double value_noise(double x, double y, double z, double scale,
                              uint64_t seed)
{
  const double fx = x / scale, fy = y / scale, fz = z / scale;
  const double ix = floor(fx), iy = floor(fy), iz = floor(fz);
  const double tx = smooth(fx - ix), ty = smooth(fy - iy), tz = smooth(fz - iz);
  const int64_t i = int64_t(ix), j = int64_t(iy), k = int64_t(iz);
  double acc = 0;
  for (int d = 0; d < 8; d++) {
    const double w = ((d & 1) ? tx : 1 - tx) * ((d & 2) ? ty : 1 - ty) *
                     ((d & 4) ? tz : 1 - tz);
    acc += w * lattice(i + (d & 1), j + ((d >> 1) & 1), k + ((d >> 2) & 1), seed);
  }
  return acc;
}

__device__ double tube_r2(const Tube &t, double x, double y, double z)
{
  const double vx = x - t.px, vy = y - t.py, vz = z - t.pz;
  const double s = vx * t.dx + vy * t.dy + vz * t.dz;
  const double ox = vx - s * t.dx, oy = vy - s * t.dy, oz = vz - s * t.dz;
  return ox * ox + oy * oy + oz * oz;
}

__device__ double vorticity(const Params &p, double x, double y, double z)
{
  double wx = 0, wy = 0, wz = 0;
  for (int t = 0; t < p.ntubes; t++) {
    const Tube &T = p.tubes[t];
    const double r2 = tube_r2(T, x, y, z);
    const double m = T.amp * exp(-r2 / (T.a * T.a));
    wx += m * T.dx;
    wy += m * T.dy;
    wz += m * T.dz;
  }
  double v = sqrt(wx * wx + wy * wy + wz * wz);
  if (p.noise_amp != 0) {
    v += p.noise_amp * (value_noise(x, y, z, p.noise_scale, p.seed) +
                        0.5 * value_noise(x, y, z, 0.5 * p.noise_scale, p.seed + 1));
  }
  return v;
}

__device__ int brick_level(const Params &p, int64_t bx, int64_t by, int64_t bz)
{
  const int64_t lo[3] = {bx * 8, by * 8, bz * 8};
  for (int h = 0; h < p.nholes; h++) {
    const int64_t *H = p.holes[h];
    if (lo[0] < H[3] && H[0] < lo[0] + 8 && lo[1] < H[4] && H[1] < lo[1] + 8 &&
        lo[2] < H[5] && H[2] < lo[2] + 8)
      return -1;
  }
  const double cx = double(lo[0]) + 4, cy = double(lo[1]) + 4, cz = double(lo[2]) + 4;
  double ind = 0;
  for (int t = 0; t < p.ntubes; t++) {
    const Tube &T = p.tubes[t];
    const double s = p.reach * T.a;
    const double e = exp(-tube_r2(T, cx, cy, cz) / (s * s));
    ind = e > ind ? e : ind;
  }
  if (ind > p.t0) return 0;
  if (ind > p.t1) return 1;
  if (ind > p.t2) return 2;
  return 3;
}

__global__ void count_kernel(const Params p, uint32_t *counts, int8_t *levels,
                             uint64_t nbricks)
{
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t b = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < nbricks;
       b += stride) {
    const int64_t bx = int64_t(b % p.bricks[0]);
    const int64_t by = int64_t((b / p.bricks[0]) % p.bricks[1]);
    const int64_t bz = int64_t(b / (uint64_t(p.bricks[0]) * p.bricks[1]));
    const int L = brick_level(p, bx, by, bz);
    levels[b] = int8_t(L);
    const uint32_t side = L < 0 ? 0u : (8u >> L);
    counts[b] = side * side * side;
  }
}

struct Feistel {
  int half_lo, half_hi;  // bit widths of the two halves
  uint64_t n;
  uint64_t seed;
  __device__ uint64_t round_f(uint64_t v, int r) const
  {
    return mix64(v ^ (seed + 0x9E3779B97F4A7C15ull * uint64_t(r + 1)));
  }
  __device__ uint64_t once(uint64_t x) const
  {
    uint64_t L = x >> half_lo, R = x & ((1ull << half_lo) - 1);
    // unbalanced Feistel on (hi, lo) halves, 4 rounds, stays in [0, 2^k)
    for (int r = 0; r < 4; r++) {
      if (r & 1) {
        R = (R ^ round_f(L, r)) & ((1ull << half_lo) - 1);
      } else {
        L = (L ^ round_f(R, r)) & ((1ull << half_hi) - 1);
      }
    }
    return (L << half_lo) | R;
  }
  __device__ uint64_t operator()(uint64_t x) const
  {
    do {
      x = once(x);
    } while (x >= n);
    return x;
  }
};

__global__ void emit_kernel(const Params p, const uint32_t *counts,
                            const uint64_t *offsets, const int8_t *levels,
                            uint64_t nbricks, int shuffle, Feistel perm,
                            int4 *cells, double *scal)
{
  const int lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t b = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
       b < nbricks; b += warps) {
    const int L = levels[b];
    if (L < 0) continue;
    const int64_t bx = int64_t(b % p.bricks[0]);
    const int64_t by = int64_t((b / p.bricks[0]) % p.bricks[1]);
    const int64_t bz = int64_t(b / (uint64_t(p.bricks[0]) * p.bricks[1]));
    const int side = 8 >> L, w = 1 << L;
    const uint32_t cnt = counts[b];
    const uint64_t off = offsets[b];
    for (uint32_t m = lane; m < cnt; m += 32) {
      const int ci = int(m % side), cj = int((m / side) % side), ck = int(m / (side * side));
      const int64_t i = bx * 8 + ci * w, j = by * 8 + cj * w, k = bz * 8 + ck * w;
      const double h = 0.5 * double(w);
      const double v = vorticity(p, double(i) + h, double(j) + h, double(k) + h);
      uint64_t at = off + m;
      if (shuffle) at = perm(at);
      cells[at] = make_int4(int(i), int(j), int(k), L);
      scal[at] = v;
    }
  }
}

uint64_t host_mix(uint64_t x) { return mix64(x); }

double urand(uint64_t &s)
{
  s = host_mix(s + 0x9E3779B97F4A7C15ull);
  return double(s >> 11) / 9007199254740992.0;
}

}  // namespace

/*! Build the brick AMR on the current device.  knobs (8 doubles):
    ntubes, core radius min, core radius max, reach, t0, t1, t2, noise_amp.
    Returns the cell count; cells/scalars are cudaMalloc'd device arrays
    that the caller frees with amrxs_device_free. */
AMRXS_API int amrxs_bricks(const int32_t *bricks3, uint64_t seed, int shuffle,
                           const double *knobs8, int nholes,
                           const int64_t *holes6, void **cells_out,
                           void **scal_out, uint64_t *n_out,
                           uint64_t *level_counts4)
{
  Params p{};
  for (int a = 0; a < 3; a++) p.bricks[a] = bricks3[a];
  p.ntubes = int(knobs8[0]);
  if (p.ntubes > kMaxTubes) p.ntubes = kMaxTubes;
  const double amin = knobs8[1], amax = knobs8[2];
  p.reach = knobs8[3];
  p.t0 = knobs8[4];
  p.t1 = knobs8[5];
  p.t2 = knobs8[6];
  p.noise_amp = knobs8[7];
  p.noise_scale = 6.0;
  p.seed = seed;
  const double ext[3] = {8.0 * bricks3[0], 8.0 * bricks3[1], 8.0 * bricks3[2]};
  uint64_t s = seed;
  for (int t = 0; t < p.ntubes; t++) {
    Tube &T = p.tubes[t];
    T.px = ext[0] * (0.1 + 0.8 * urand(s));
    T.py = ext[1] * (0.1 + 0.8 * urand(s));
    T.pz = ext[2] * (0.1 + 0.8 * urand(s));
    // mostly stream-wise (x) tubes, like wing-tip / wake vortices
    double dx = 1.0, dy = 0.6 * (urand(s) - 0.5), dz = 0.6 * (urand(s) - 0.5);
    if (t % 3 == 2) {
      dx = 0.3 * (urand(s) - 0.5);
      dy = 1.0;
      dz = 0.5 * (urand(s) - 0.5);
    }
    const double len = std::sqrt(dx * dx + dy * dy + dz * dz);
    T.dx = dx / len;
    T.dy = dy / len;
    T.dz = dz / len;
    T.a = amin + (amax - amin) * urand(s);
    T.amp = (0.7 + 0.6 * urand(s)) * 100.0;  // peak |omega| ~ 100
  }
  p.nholes = nholes > 4 ? 4 : nholes;
  for (int h = 0; h < p.nholes; h++)
    for (int c = 0; c < 6; c++) p.holes[h][c] = holes6[6 * h + c];

  const uint64_t nb = uint64_t(p.bricks[0]) * p.bricks[1] * p.bricks[2];
  uint32_t *counts = nullptr;
  uint64_t *offsets = nullptr;
  int8_t *levels = nullptr;
  if (cudaMalloc(&counts, nb * 4) || cudaMalloc(&offsets, (nb + 1) * 8) ||
      cudaMalloc(&levels, nb))
    return -1;
  count_kernel<<<4096, 256>>>(p, counts, levels, nb);
  // u32 counts -> u64 offsets
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offsets, nb + 1);
  void *tmp = nullptr;
  if (cudaMalloc(&tmp, tmp_bytes)) return -1;
  // nb+1 entries: counts has nb; scan nb then add the total separately
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, offsets, nb);
  uint64_t last_off = 0;
  uint32_t last_cnt = 0;
  cudaMemcpy(&last_off, offsets + nb - 1, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&last_cnt, counts + nb - 1, 4, cudaMemcpyDeviceToHost);
  const uint64_t n = last_off + last_cnt;

  int4 *cells = nullptr;
  double *scal = nullptr;
  if (cudaMalloc(&cells, n * 16 + 16) || cudaMalloc(&scal, n * 8 + 16)) return -1;
  Feistel perm{};
  int k = 1;
  while ((1ull << k) < n) k++;
  perm.half_lo = k / 2;
  perm.half_hi = k - k / 2;
  perm.n = n;
  perm.seed = seed ^ 0x5eedull;
  emit_kernel<<<8192, 256>>>(p, counts, offsets, levels, nb, shuffle, perm,
                             cells, scal);
  if (level_counts4) {
    // brick level histogram -> cell counts per level
    int8_t *hl = new int8_t[nb];
    cudaMemcpy(hl, levels, nb, cudaMemcpyDeviceToHost);
    for (int l = 0; l < 4; l++) level_counts4[l] = 0;
    for (uint64_t b = 0; b < nb; b++)
      if (hl[b] >= 0) {
        const uint64_t side = 8u >> hl[b];
        level_counts4[hl[b]] += side * side * side;
      }
    delete[] hl;
  }
  const cudaError_t e = cudaDeviceSynchronize();
  cudaFree(counts);
  cudaFree(offsets);
  cudaFree(levels);
  cudaFree(tmp);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "amrxs_bricks: %s\n", cudaGetErrorString(e));
    return -2;
  }
  *cells_out = cells;
  *scal_out = scal;
  *n_out = n;
  return 0;
}

AMRXS_API void amrxs_device_free(void *p) { cudaFree(p); }

AMRXS_API int amrxs_memcpy(void *dst, const void *src, uint64_t bytes)
{
  return int(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
}
