// Single-process multi-GPU extraction over NCCL, the C ABI
// behind amrx_comm_* (include/amrx.h): a C++ host -- the drop-in shim's
// extract_isosurface -- drives every GPU of the box from one process.
//
// The reference's only parallelism is a thread pool over chunks of the
// candidate tasks (proj/include/amriso/parallel.hpp:49-85); its output order
// is candidate order, owner-cell major (proj/src/pipeline.cpp:40-57), so a
// contiguous range of sorted cells per GPU concatenates, in device order, to
// exactly the single-GPU output.  The plan:
//   1. build_index on the first device (pack + radix sort + lookup build);
//   2. ncclBroadcast of the sorted keys + scalars (16 B/cell) to every other
//      device over NVLink/NVSwitch, one ncclGroup over all communicators;
//   3. every other device adopts them (its own lookup structure, no sort);
//   4. extraction: one host thread per device extracts cells
//      [n d / N, n (d+1) / N) into its device arena; the per-device counts
//      give the output offsets (an exclusive scan on the host -- the
//      single-process form of the count all-gather); each device copies its
//      part into the caller's buffer at its offset.
// NCCL is loaded with dlopen on first use (libnccl.so.2, the copy torch
// bundles when it is already in the process), so the library has no link
// dependency on it.
#include "index.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <exception>
#include <limits>
#include <mutex>
#include <thread>
#include <vector>

namespace {

struct Nccl {
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl &nccl()
{
  static std::once_flag once;
  static Nccl n;
  static std::string why;
  std::call_once(once, [] {
    void *h = nullptr;
    for (const char *name : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    if (!h) {
      why = std::string("NCCL not found (dlopen libnccl.so.2: ") + dlerror() + ")";
      return;
    }
    n.init_all = reinterpret_cast<decltype(n.init_all)>(dlsym(h, "ncclCommInitAll"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "ncclCommDestroy"));
    n.broadcast = reinterpret_cast<decltype(n.broadcast)>(dlsym(h, "ncclBroadcast"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(h, "ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!n.init_all || !n.destroy || !n.broadcast || !n.group_start || !n.group_end ||
        !n.error_string) {
      why = "libnccl.so.2 lacks a needed symbol";
      n = Nccl{};
    }
  });
  if (!n.init_all) fail(AMRX_ERR_NCCL, why);
  return n;
}

void nccl_check(ncclResult_t r, const char *what)
{
  if (r != ncclSuccess)
    fail(AMRX_ERR_NCCL, std::string(what) + ": " + nccl().error_string(r));
}

/// run fn(d) for every device d on its own host thread; the first error
/// (by device order) is rethrown here with its status code
template <typename Fn>
void per_device(int ndev, Fn &&fn)
{
  std::vector<std::exception_ptr> err(ndev);
  std::vector<std::thread> th;
  th.reserve(ndev);
  for (int d = 0; d < ndev; d++)
    th.emplace_back([&, d] {
      try {
        fn(d);
      } catch (...) {
        err[d] = std::current_exception();
      }
    });
  for (auto &t : th) t.join();
  for (auto &e : err)
    if (e) std::rethrow_exception(e);
}

template <typename Fn>
amrx_status guarded_comm(Fn &&fn)
{
  try {
    fn();
    set_last_error("", true);
    return AMRX_OK;
  } catch (const ApiError &e) {
    set_last_error(e.what(), false);
    return amrx_status(e.code);
  } catch (const std::bad_alloc &) {
    set_last_error("host allocation failed", false);
    return AMRX_ERR_CUDA;
  } catch (const std::exception &e) {
    set_last_error(e.what(), false);
    return AMRX_ERR_INTERNAL;
  }
}

}  // namespace

struct amrx_comm {
  std::vector<int> dev;
  std::vector<ncclComm_t> comm;
  std::vector<cudaStream_t> st;
};

struct amrx_comm_index {
  amrx_comm *comm = nullptr;
  std::vector<amrx_index *> ix;
  uint64_t n = 0;
};

namespace {

void destroy_index(amrx_comm_index *m)
{
  for (amrx_index *p : m->ix)
    if (p) amrx_index_destroy(p);
  m->ix.clear();
}

/// device d's contiguous share of the cells
amrx_range share(const amrx_comm_index *m, int d)
{
  const uint64_t nd = m->ix.size();
  return amrx_range{m->n * uint64_t(d) / nd, m->n * uint64_t(d + 1) / nd};
}

void add_stats(amrx_stats &t, const amrx_stats &s)
{
  t.cell_count += s.cell_count;
  t.duals_accepted += s.duals_accepted;
  t.duals_missing_corner += s.duals_missing_corner;
  t.duals_finer_corner += s.duals_finer_corner;
  t.duals_lower_key_corner += s.duals_lower_key_corner;
  t.pass1_triangle_count += s.pass1_triangle_count;
  t.fat_triangle_count += s.fat_triangle_count;
  t.dual_count += s.dual_count;
  // device times: the devices run side by side, the slowest sets the pace
  t.seconds_pass1 = std::max(t.seconds_pass1, s.seconds_pass1);
  t.seconds_pass2 = std::max(t.seconds_pass2, s.seconds_pass2);
  t.kernel_launches += s.kernel_launches;
}

}  // namespace

extern "C" {

amrx_status amrx_comm_init(int ndev, const int *devices, amrx_comm **out)
{
  return guarded_comm([&] {
    if (!out) fail(AMRX_ERR_INVALID_ARG, "out is null");
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      fail(AMRX_ERR_NO_DEVICE, "no CUDA device available");
    }
    if (ndev <= 0) ndev = count;
    auto c = std::make_unique<amrx_comm>();
    for (int d = 0; d < ndev; d++) {
      const int dv = devices ? devices[d] : d;
      if (dv < 0 || dv >= count)
        fail(AMRX_ERR_INVALID_ARG, "device " + std::to_string(dv) + " does not exist (" +
                                     std::to_string(count) + " visible)");
      if (std::find(c->dev.begin(), c->dev.end(), dv) != c->dev.end())
        fail(AMRX_ERR_INVALID_ARG, "device " + std::to_string(dv) + " listed twice");
      c->dev.push_back(dv);
    }
    c->comm.resize(ndev);
    nccl_check(nccl().init_all(c->comm.data(), ndev, c->dev.data()), "ncclCommInitAll");
    c->st.resize(ndev);
    for (int d = 0; d < ndev; d++) {
      AMRX_CUDA(cudaSetDevice(c->dev[d]));
      AMRX_CUDA(cudaStreamCreateWithFlags(&c->st[d], cudaStreamNonBlocking));
    }
    *out = c.release();
  });
}

amrx_status amrx_device_count(int *n)
{
  return guarded_comm([&] {
    if (!n) fail(AMRX_ERR_INVALID_ARG, "null argument");
    *n = 0;
    if (cudaGetDeviceCount(n) != cudaSuccess) {
      cudaGetLastError();
      *n = 0;
    }
  });
}

amrx_status amrx_comm_destroy(amrx_comm *comm)
{
  return guarded_comm([&] {
    if (!comm) return;
    for (size_t d = 0; d < comm->dev.size(); d++) {
      cudaSetDevice(comm->dev[d]);
      if (comm->st[d]) cudaStreamDestroy(comm->st[d]);
      if (comm->comm[d]) nccl().destroy(comm->comm[d]);
    }
    delete comm;
  });
}

amrx_status amrx_comm_size(const amrx_comm *comm, int *ndev)
{
  return guarded_comm([&] {
    if (!comm || !ndev) fail(AMRX_ERR_INVALID_ARG, "null argument");
    *ndev = int(comm->dev.size());
  });
}

amrx_status amrx_comm_index_create(amrx_comm *comm, const int32_t *cells4, const double *scalars,
                                   uint64_t n_cells, uint64_t n_scalars, uint32_t flags,
                                   amrx_comm_index **out)
{
  return guarded_comm([&] {
    if (!comm || !out) fail(AMRX_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    const int nd = int(comm->dev.size());
    auto m = std::make_unique<amrx_comm_index>();
    struct Guard {
      amrx_comm_index *m;
      ~Guard()
      {
        if (m) destroy_index(m);
      }
    } guard{m.get()};
    m->comm = comm;
    m->ix.assign(nd, nullptr);
    // 1. the sort on the first device
    amrx_index_opts o0{comm->dev[0], nullptr, flags};
    const amrx_status s0 = amrx_index_create(cells4, scalars, n_cells, n_scalars, &o0, &m->ix[0]);
    if (s0 != AMRX_OK) fail(s0, amrx_last_error());
    amrx_index_info info{};
    amrx_index_get_info(m->ix[0], &info);
    m->n = info.cell_count;
    if (nd > 1) {
      int64_t g16[16];
      void *k0 = nullptr, *s0 = nullptr;
      amrx_index_geometry(m->ix[0], g16);
      amrx_index_device_arrays(m->ix[0], &k0, &s0);
      // 2. broadcast the sorted keys + scalars from device 0
      std::vector<void *> keys(nd, nullptr), scal(nd, nullptr);
      struct Free {
        std::vector<void *> *k, *s;
        const std::vector<int> *dev;
        ~Free()
        {
          for (size_t d = 1; d < k->size(); d++) {
            cudaSetDevice((*dev)[d]);
            if ((*k)[d]) cudaFree((*k)[d]);
            if ((*s)[d]) cudaFree((*s)[d]);
          }
        }
      } fr{&keys, &scal, &comm->dev};
      keys[0] = k0;
      scal[0] = s0;
      for (int d = 1; d < nd; d++) {
        AMRX_CUDA(cudaSetDevice(comm->dev[d]));
        AMRX_CUDA(cudaMalloc(&keys[d], m->n * 8));
        AMRX_CUDA(cudaMalloc(&scal[d], m->n * 8));
      }
      const Nccl &N = nccl();
      nccl_check(N.group_start(), "ncclGroupStart");
      for (int d = 0; d < nd; d++) {
        N.broadcast(keys[0], keys[d], m->n, ncclUint64, 0, comm->comm[d], comm->st[d]);
        N.broadcast(scal[0], scal[d], m->n, ncclFloat64, 0, comm->comm[d], comm->st[d]);
      }
      nccl_check(N.group_end(), "ncclGroupEnd (broadcast of the sorted index)");
      for (int d = 0; d < nd; d++) {
        AMRX_CUDA(cudaSetDevice(comm->dev[d]));
        AMRX_CUDA(cudaStreamSynchronize(comm->st[d]));
      }
      // 3. every other device indexes the broadcast arrays (no sort)
      per_device(nd - 1, [&](int i) {
        const int d = i + 1;
        amrx_index_opts od{comm->dev[d], nullptr, flags};
        if (amrx_index_adopt(keys[d], static_cast<const double *>(scal[d]), m->n, g16, &od,
                             &m->ix[d]) != AMRX_OK)
          fail(AMRX_ERR_INTERNAL, std::string("device ") + std::to_string(comm->dev[d]) +
                                    ": " + amrx_last_error());
      });
    }
    guard.m = nullptr;
    *out = m.release();
  });
}

amrx_status amrx_comm_index_destroy(amrx_comm_index *index)
{
  return guarded_comm([&] {
    if (!index) return;
    destroy_index(index);
    delete index;
  });
}

amrx_status amrx_comm_extract_iso(amrx_comm_index *m, const amrx_iso_params *params, void *xyz9,
                                  uint64_t cap, uint64_t *count, amrx_stats *stats)
{
  return guarded_comm([&] {
    if (!m || !params || !count) fail(AMRX_ERR_INVALID_ARG, "null argument");
    const int nd = int(m->ix.size());
    const size_t tb = params->xyz_is_f32 ? 36 : 72;
    std::vector<uint64_t> cnt(nd, 0);
    std::vector<amrx_stats> st(nd);
    amrx_iso_params p = *params;
    p.check_length = 0;  // checked on the total below
    // 4. every device extracts its share into its device arena
    per_device(nd, [&](int d) {
      const amrx_range r = share(m, d);
      extract_iso_impl(m->ix[d], &r, &p, nullptr, 0, &cnt[d], &st[d], true);
    });
    uint64_t total = 0;
    amrx_stats sum{};
    for (int d = 0; d < nd; d++) {
      total += cnt[d];
      add_stats(sum, st[d]);
    }
    *count = total;
    if (stats) *stats = sum;
    if (params->check_length && total > uint64_t(std::numeric_limits<uint32_t>::max()) / 3)
      fail(AMRX_ERR_LENGTH, "extract_isosurface: mesh too large for 32-bit indices");
    if (!xyz9) return;
    if (total > cap)
      fail(AMRX_ERR_CAPACITY, "output capacity " + std::to_string(cap) + " < " +
                                std::to_string(total) + " triangles");
    // each device's part at its offset in candidate order
    per_device(nd, [&](int d) {
      uint64_t off = 0;
      for (int e = 0; e < d; e++) off += cnt[e];
      const amrx_range r = share(m, d);
      uint64_t c = 0;
      amrx_stats s{};
      if (cnt[d])
        extract_iso_impl(m->ix[d], &r, &p, static_cast<char *>(xyz9) + off * tb, cnt[d], &c, &s,
                         true);
    });
  });
}

amrx_status amrx_comm_extract_dual(amrx_comm_index *m, uint32_t *corners8, uint64_t *task_ids,
                                   uint64_t cap, uint64_t *count, amrx_stats *stats)
{
  return guarded_comm([&] {
    if (!m || !count) fail(AMRX_ERR_INVALID_ARG, "null argument");
    const int nd = int(m->ix.size());
    std::vector<uint64_t> cnt(nd, 0);
    std::vector<amrx_stats> st(nd);
    per_device(nd, [&](int d) {
      const amrx_range r = share(m, d);
      extract_dual_impl(m->ix[d], &r, nullptr, nullptr, 0, &cnt[d], &st[d], true);
    });
    uint64_t total = 0;
    amrx_stats sum{};
    for (int d = 0; d < nd; d++) {
      total += cnt[d];
      add_stats(sum, st[d]);
    }
    *count = total;
    if (stats) *stats = sum;
    if (!corners8 && !task_ids) return;
    if (total > cap)
      fail(AMRX_ERR_CAPACITY, "output capacity " + std::to_string(cap) + " < " +
                                std::to_string(total) + " duals");
    per_device(nd, [&](int d) {
      uint64_t off = 0;
      for (int e = 0; e < d; e++) off += cnt[e];
      const amrx_range r = share(m, d);
      uint64_t c = 0;
      amrx_stats s{};
      if (cnt[d])
        extract_dual_impl(m->ix[d], &r, corners8 ? corners8 + off * 8 : nullptr,
                          task_ids ? task_ids + off : nullptr, cnt[d], &c, &s, true);
    });
  });
}

}  // extern "C"
