// Output writers: write_obj / write_ply / write_dual_mesh
// (proj/src/io.cpp:212-305, io.hpp:48-66) for meshes of 10^8 triangles.
//
// The reference builds one std::string serially and hands it to
// write_file_atomic.  Here the items are split into contiguous ranges that
// host threads format concurrently (std::to_chars shortest round trip for
// doubles, the same function format_double uses, so every number prints
// identically), and the pieces are written with pwrite at their prefix-sum
// offsets by parallel threads into the sibling ".tmp" file, which is then
// renamed over the target -- the reference's atomic-replace contract
// (io.cpp:307-333, same error messages).  Host code: formatting is the
// bottleneck and has no GPU-friendly shortest-decimal form worth the
// complexity; the GPU's job ends when the mesh is downloaded.
#include "amrx.h"

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <unistd.h>

namespace amrx {
void set_last_error(const std::string &msg, bool clear);
}

namespace {

struct WriteError : std::runtime_error {
  int code;
  WriteError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

template <typename Fn>
amrx_status guarded_write(Fn &&fn)
{
  try {
    fn();
    amrx::set_last_error("", true);
    return AMRX_OK;
  } catch (const WriteError &e) {
    amrx::set_last_error(e.what(), false);
    return amrx_status(e.code);
  } catch (const std::bad_alloc &) {
    amrx::set_last_error("host allocation failed", false);
    return AMRX_ERR_IO;
  } catch (const std::exception &e) {
    amrx::set_last_error(e.what(), false);
    return AMRX_ERR_INTERNAL;
  }
}

int resolve_threads(int t)
{
  if (t > 0) return t;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? int(std::min(h, 64u)) : 1;
}

inline void put_double(std::string &out, double v)
{
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, r.ptr);
}

inline void put_uint(std::string &out, uint64_t v)
{
  char buf[24];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, r.ptr);
}

template <typename T>
inline void put_raw(std::string &out, T v)
{
  char b[sizeof(T)];
  std::memcpy(b, &v, sizeof(T));
  out.append(b, sizeof(T));
}

/// items [0, n) formatted by fn(out, i) into per-thread contiguous pieces
template <typename Fn>
std::vector<std::string> format_parts(uint64_t n, int threads, size_t bytes_per_item, Fn fn)
{
  const int parts = n < 65536 ? 1 : threads;
  std::vector<std::string> out(parts);
  auto run = [&](int p) {
    const uint64_t lo = n * uint64_t(p) / uint64_t(parts), hi = n * uint64_t(p + 1) / uint64_t(parts);
    out[p].reserve((hi - lo) * bytes_per_item);
    for (uint64_t i = lo; i < hi; i++) fn(out[p], i);
  };
  if (parts == 1) {
    run(0);
    return out;
  }
  std::vector<std::thread> pool;
  for (int p = 0; p < parts; p++) pool.emplace_back(run, p);
  for (auto &t : pool) t.join();
  return out;
}

/// write_file_atomic (io.cpp:307-333) over pieces written in parallel
void write_atomic(const std::string &path, const std::vector<const std::string *> &pieces,
                  int threads)
{
  const std::string tmp = path + ".tmp";
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0666);
  if (fd < 0) throw WriteError(AMRX_ERR_IO, "cannot open " + tmp + " for writing");
  std::vector<uint64_t> off(pieces.size() + 1, 0);
  for (size_t p = 0; p < pieces.size(); p++) off[p + 1] = off[p] + pieces[p]->size();
  std::atomic<bool> bad{false};
  std::atomic<size_t> next{0};
  auto worker = [&] {
    for (size_t p; (p = next.fetch_add(1)) < pieces.size();) {
      const char *d = pieces[p]->data();
      uint64_t left = pieces[p]->size(), at = off[p];
      while (left && !bad) {
        const ssize_t w = ::pwrite(fd, d, left, off_t(at));
        if (w <= 0) {
          bad = true;
          break;
        }
        d += w;
        at += uint64_t(w);
        left -= uint64_t(w);
      }
    }
  };
  const int nw = int(std::min<size_t>(size_t(std::max(1, threads)), pieces.size()));
  if (nw <= 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nw; t++) pool.emplace_back(worker);
    for (auto &t : pool) t.join();
  }
  if (::close(fd) != 0) bad = true;
  if (bad) {
    ::unlink(tmp.c_str());
    throw WriteError(AMRX_ERR_IO, "write to " + tmp + " failed");
  }
  if (::rename(tmp.c_str(), path.c_str()) != 0) {
    const std::string why = std::strerror(errno);
    ::unlink(tmp.c_str());
    throw WriteError(AMRX_ERR_IO, "cannot move " + tmp + " to " + path + ": " + why);
  }
}

void need(bool ok, const char *what)
{
  if (!ok) throw WriteError(AMRX_ERR_INVALID_ARG, what);
}

void check_tris(const uint32_t *tris3, uint64_t n_tris, uint64_t n_verts, int threads)
{
  std::atomic<bool> bad{false};
  format_parts(n_tris, threads, 0, [&](std::string &, uint64_t t) {
    if (tris3[3 * t] >= n_verts || tris3[3 * t + 1] >= n_verts || tris3[3 * t + 2] >= n_verts)
      bad = true;
  });
  need(!bad, "triangle index out of range");
}

}  // namespace

extern "C" {

amrx_status amrx_write_obj(const char *path, const double *verts3, uint64_t n_verts,
                           const uint32_t *tris3, uint64_t n_tris, int threads)
{
  return guarded_write([&] {
    need(path && (verts3 || !n_verts) && (tris3 || !n_tris), "null argument");
    const int T = resolve_threads(threads);
    check_tris(tris3, n_tris, n_verts, T);
    // obj_string (io.cpp:219-233)
    const std::string head = "# amriso mesh: " + std::to_string(n_verts) + " vertices, " +
                             std::to_string(n_tris) + " triangles\n";
    auto vparts = format_parts(n_verts, T, 64, [&](std::string &o, uint64_t v) {
      o += "v ";
      put_double(o, verts3[3 * v]);
      o += ' ';
      put_double(o, verts3[3 * v + 1]);
      o += ' ';
      put_double(o, verts3[3 * v + 2]);
      o += '\n';
    });
    auto fparts = format_parts(n_tris, T, 32, [&](std::string &o, uint64_t t) {
      o += "f ";
      put_uint(o, uint64_t(tris3[3 * t]) + 1);
      o += ' ';
      put_uint(o, uint64_t(tris3[3 * t + 1]) + 1);
      o += ' ';
      put_uint(o, uint64_t(tris3[3 * t + 2]) + 1);
      o += '\n';
    });
    std::vector<const std::string *> pieces{&head};
    for (auto &p : vparts) pieces.push_back(&p);
    for (auto &p : fparts) pieces.push_back(&p);
    write_atomic(path, pieces, T);
  });
}

amrx_status amrx_write_ply(const char *path, const double *verts3, uint64_t n_verts,
                           const uint32_t *tris3, uint64_t n_tris, int threads)
{
  return guarded_write([&] {
    need(path && (verts3 || !n_verts) && (tris3 || !n_tris), "null argument");
    const int T = resolve_threads(threads);
    check_tris(tris3, n_tris, n_verts, T);
    // ply_string (io.cpp:241-266): float32 positions, uchar 3 + 3 x uint32
    std::string head = "ply\nformat binary_little_endian 1.0\ncomment amriso mesh\n";
    head += "element vertex " + std::to_string(n_verts) + "\n";
    head += "property float x\nproperty float y\nproperty float z\n";
    head += "element face " + std::to_string(n_tris) + "\n";
    head += "property list uchar uint vertex_indices\nend_header\n";
    auto vparts = format_parts(n_verts, T, 12, [&](std::string &o, uint64_t v) {
      put_raw<float>(o, float(verts3[3 * v]));
      put_raw<float>(o, float(verts3[3 * v + 1]));
      put_raw<float>(o, float(verts3[3 * v + 2]));
    });
    auto fparts = format_parts(n_tris, T, 13, [&](std::string &o, uint64_t t) {
      put_raw<uint8_t>(o, 3);
      put_raw<uint32_t>(o, tris3[3 * t]);
      put_raw<uint32_t>(o, tris3[3 * t + 1]);
      put_raw<uint32_t>(o, tris3[3 * t + 2]);
    });
    std::vector<const std::string *> pieces{&head};
    for (auto &p : vparts) pieces.push_back(&p);
    for (auto &p : fparts) pieces.push_back(&p);
    write_atomic(path, pieces, T);
  });
}

amrx_status amrx_write_dual_mesh(const char *path, const uint32_t *corners8, uint64_t n_duals,
                                 const int32_t *cells4, const double *scalars, uint64_t n_cells,
                                 int threads)
{
  return guarded_write([&] {
    need(path && (corners8 || !n_duals) && (n_duals == 0 || (cells4 && scalars)),
         "null argument");
    const int T = resolve_threads(threads);
    {
      std::atomic<bool> bad{false};
      format_parts(n_duals, T, 0, [&](std::string &, uint64_t d) {
        for (int k = 0; k < 8; k++)
          if (corners8[8 * d + k] >= n_cells) bad = true;
      });
      need(!bad, "corner CellId out of range");
    }
    // dual_mesh_string (io.cpp:274-298): 8 cell centres (cell_center,
    // core.hpp:114-118), then the 8 scalars
    const std::string head = "# amriso dual cells: " + std::to_string(n_duals) +
                             "\n# per line: 8 corner centers (slot order, x fastest), "
                             "then 8 scalars\n";
    auto parts = format_parts(n_duals, T, 400, [&](std::string &o, uint64_t d) {
      for (int k = 0; k < 8; k++) {
        const int32_t *c = cells4 + 4 * uint64_t(corners8[8 * d + k]);
        const double half = 0.5 * double(int64_t(1) << c[3]);
        for (int a = 0; a < 3; a++) {
          put_double(o, double(c[a]) + half);
          o += ' ';
        }
      }
      for (int k = 0; k < 8; k++) {
        put_double(o, scalars[corners8[8 * d + k]]);
        o += k == 7 ? '\n' : ' ';
      }
    });
    std::vector<const std::string *> pieces{&head};
    for (auto &p : parts) pieces.push_back(&p);
    write_atomic(path, pieces, T);
  });
}

}  // extern "C"
