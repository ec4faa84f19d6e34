// C ABI (include/amrx.h): the device index handle, host/device pointer
// handling, error mapping and the orchestration of the ingest/extract
// kernels.  Every entry point catches everything and returns a status; the
// message is kept per thread for amrx_last_error().
#include "amrx.h"
#include "internal.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <thread>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace amrx {

namespace {
thread_local std::string g_last_error;


/// checked builds: any violated device bound of the call is an error
void check_bounds()
{
#if AMRX_CHECKED
  cudaDeviceSynchronize();
  const unsigned int w = check_word_extract() | check_word_sort() | check_word_wide() |
                         check_word_ingest() | check_word_validate() | check_word_weld();
  if (w) fail(AMRX_ERR_INTERNAL, "checked build: device bounds violated (codes 0x" +
                                   [&] {
                                     char b[16];
                                     std::snprintf(b, sizeof b, "%x", w);
                                     return std::string(b);
                                   }() + ", CheckCode in common.cuh)");
#endif
}

template <typename Fn>
amrx_status guarded(Fn &&fn)
{
  try {
    fn();
    check_bounds();
    g_last_error.clear();
    return AMRX_OK;
  } catch (const ApiError &e) {
    g_last_error = e.what();
    return amrx_status(e.code);
  } catch (const std::bad_alloc &) {
    g_last_error = "host allocation failed";
    return AMRX_ERR_CUDA;
  } catch (const std::exception &e) {
    g_last_error = e.what();
    return AMRX_ERR_INTERNAL;
  }
}

bool is_device_ptr(const void *p)
{
  if (!p) return false;
  cudaPointerAttributes attr;
  const cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear sticky-free error state
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

/// the pointer itself if it is device memory (inputs: staged otherwise)
const void *device_view(const void *p)
{
  return is_device_ptr(p) ? p : nullptr;
}

/*! a device-writable alias of an output pointer: device memory, or pinned
    (page-locked, mapped) host memory the kernels can stream into directly
    over the host link; nullptr for pageable host memory */
void *device_writable(void *p)
{
  if (!p) return nullptr;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged)
    return p;
  if (attr.type == cudaMemoryTypeHost && attr.devicePointer) return attr.devicePointer;
  return nullptr;
}

int bit_width(uint64_t v)
{
  int b = 0;
  while (v) {
    b++;
    v >>= 1;
  }
  return b;
}

/// a device view of a caller pointer: the pointer itself or a staged copy
template <typename T>
struct DevIn {
  const T *ptr = nullptr;
  DevBuf stage;
  DevIn(const T *p, size_t count, cudaStream_t st)
  {
    if (!p || count == 0) return;
    if (is_device_ptr(p)) {
      ptr = p;
      return;
    }
    stage.reserve(count * sizeof(T), st);
    AMRX_CUDA(cudaMemcpyAsync(stage.ptr, p, count * sizeof(T),
                              cudaMemcpyHostToDevice, st));
    ptr = stage.as<T>();
  }
};

template <typename T>
struct DevOut {
  T *user = nullptr;
  T *ptr = nullptr;
  size_t count = 0;
  bool staged = false;
  DevBuf stage;
  DevOut(T *p, size_t n, cudaStream_t st) : user(p), count(n)
  {
    if (!p || n == 0) return;
    if (is_device_ptr(p)) {
      ptr = p;
      return;
    }
    staged = true;
    stage.reserve(n * sizeof(T), st);
    ptr = stage.as<T>();
  }
  void finish(cudaStream_t st)
  {
    if (staged)
      AMRX_CUDA(cudaMemcpyAsync(user, ptr, count * sizeof(T),
                                cudaMemcpyDeviceToHost, st));
  }
};

}  // namespace

[[noreturn]] void throw_cuda(cudaError_t e, const char *what, const char *file,
                             int line)
{
  const char *base = std::strrchr(file, '/');
  std::string msg = std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                    cudaGetErrorString(e) + ") in " + what + " at " +
                    (base ? base + 1 : file) + ":" + std::to_string(line);
  const int code = (e == cudaErrorNoDevice || e == cudaErrorNoKernelImageForDevice ||
                    e == cudaErrorInsufficientDriver)
                     ? AMRX_ERR_NO_DEVICE
                     : AMRX_ERR_CUDA;
  throw ApiError(code, msg);
}

DevBuf::~DevBuf() { release(); }

namespace {
void release_idle_memory(int device);
}

void DevBuf::reserve(size_t n, cudaStream_t st)
{
  if (n <= bytes && ptr) return;
  release();
  if (n == 0) n = 16;
  stream = st;
  if (cudaMallocAsync(&ptr, n, st) != cudaSuccess) {
    // out of memory: give back idle workspace slots and the pool's cached
    // blocks, then try once more
    cudaGetLastError();
    int dev = 0;
    cudaGetDevice(&dev);
    release_idle_memory(dev);
    AMRX_CUDA(cudaMallocAsync(&ptr, n, st));
  }
  bytes = n;
}

void DevBuf::release()
{
  if (ptr) cudaFreeAsync(ptr, stream);
  ptr = nullptr;
  bytes = 0;
}

void enable_pool_caching(int device)
{
  static std::mutex mu;
  static bool done[64] = {false};
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  AMRX_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = ~0ull;
  AMRX_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  done[device] = true;
}

namespace {
std::atomic<uint64_t> g_launches{0};

struct WsDevice {
  std::mutex mu;
  void *ptr[kWsCount] = {};
  size_t bytes[kWsCount] = {};
  bool busy[kWsCount] = {};
};

WsDevice &ws_device(int dev)
{
  static WsDevice devices[64];
  return devices[dev & 63];
}

/// free the idle workspace slots (caller holds no lock on w) and trim the
/// stream-ordered pool: the memory-pressure fallback of every allocation
void release_idle_slots(WsDevice &w)
{
  cudaDeviceSynchronize();
  for (int i = 0; i < kWsCount; i++)
    if (!w.busy[i] && w.ptr[i]) {
      cudaFree(w.ptr[i]);
      w.ptr[i] = nullptr;
      w.bytes[i] = 0;
    }
}

void release_idle_memory(int device)
{
  WsDevice &w = ws_device(device);
  {
    std::lock_guard<std::mutex> lock(w.mu);
    release_idle_slots(w);
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
}

/// cudaMalloc with the memory-pressure fallback (w.mu held by the caller)
void slot_malloc(WsDevice &w, int device, void **p, size_t n, int slot)
{
  if (cudaMalloc(p, n) == cudaSuccess) return;
  cudaGetLastError();
  release_idle_slots(w);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
  if (cudaMalloc(p, n) != cudaSuccess) {
    cudaGetLastError();
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    throw ApiError(AMRX_ERR_CUDA, "out of device memory for a " + std::to_string(n >> 20) +
                                    " MiB workspace buffer (slot " + std::to_string(slot) + ", " +
                                    std::to_string(fr >> 20) +
                                    " of " + std::to_string(tot >> 20) + " MiB free)");
  }
}
}  // namespace

void *WsLease::get(int slot, size_t n, cudaStream_t st)
{
  if (ptr && bytes >= n) return ptr;
  if (ptr && slot_ >= 0) {
    // grow a slot this lease holds (rare)
    WsDevice &w = ws_device(device_);
    std::lock_guard<std::mutex> lock(w.mu);
    AMRX_CUDA(cudaDeviceSynchronize());
    cudaFree(w.ptr[slot_]);
    w.ptr[slot_] = nullptr;
    w.bytes[slot_] = 0;
    slot_malloc(w, device_, &w.ptr[slot_], n, slot_);
    w.bytes[slot_] = n;
    ptr = w.ptr[slot_];
    bytes = n;
    return ptr;
  }
  if (ptr) {
    own_.reserve(n, st);
    ptr = own_.ptr;
    bytes = own_.bytes;
    return ptr;
  }
  int dev = 0;
  AMRX_CUDA(cudaGetDevice(&dev));
  WsDevice &w = ws_device(dev);
  {
    std::lock_guard<std::mutex> lock(w.mu);
    if (!w.busy[slot]) {
      if (w.bytes[slot] < n) {
        // grow (rare): the slot outlives every stream, so plain cudaMalloc
        if (w.ptr[slot]) {
          AMRX_CUDA(cudaDeviceSynchronize());
          cudaFree(w.ptr[slot]);
          w.ptr[slot] = nullptr;
          w.bytes[slot] = 0;
        }
        const size_t want = std::max<size_t>(n, 256);
        slot_malloc(w, dev, &w.ptr[slot], want, slot);
        w.bytes[slot] = want;
      }
      w.busy[slot] = true;
      device_ = dev;
      slot_ = slot;
      ptr = w.ptr[slot];
      bytes = w.bytes[slot];
      return ptr;
    }
  }
  own_.reserve(n, st);
  ptr = own_.ptr;
  bytes = own_.bytes;
  return ptr;
}

WsLease::~WsLease()
{
  if (slot_ >= 0) {
    WsDevice &w = ws_device(device_);
    std::lock_guard<std::mutex> lock(w.mu);
    w.busy[slot_] = false;
  }
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void ensure_smem_attr(const void *kernel, size_t bytes)
{
  int dev = 0;
  AMRX_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::vector<std::pair<const void *, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto &d : done)
    if (d.first == kernel && d.second == dev) return;
  AMRX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(bytes)));
  done.emplace_back(kernel, dev);
}

int device_sm_count()
{
  int dev = 0;
  cudaGetDevice(&dev);
  static int cached[64] = {0};
  if (dev < 64 && cached[dev]) return cached[dev];
  int sms = 0;
  AMRX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (dev < 64) cached[dev] = sms;
  return sms;
}

}  // namespace amrx

using namespace amrx;

#include "index.h"

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev)
  {
    cudaGetDevice(&prev);
    if (dev != prev) AMRX_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard()
  {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

/// directory size for the binary-search lookup: about two buckets per cell
int directory_bits(const KeyGeom &g, uint64_t n)
{
  return std::min(g.total, std::min(30, std::max(10, bit_width(n) + 1)));
}

/*! the key geometry of a dataset (field widths from its extent) and its
    lookup structure: AMRX_FLAG_LOOKUP_* in `flags` forces one; by default
    dense occupancy records while they cost at most ~192 B per cell (or
    1 GB), else hashed records */
KeyGeom make_geometry(const int64_t mn[3], const int64_t mx[3],
                      uint32_t level_mask, uint64_t n, uint32_t flags)
{
  KeyGeom g{};
  int lo_level = 0, hi_level = 0;
  for (int l = 0; l <= kMaxLevel; l++)
    if ((level_mask >> l) & 1u) {
      lo_level = l;
      break;
    }
  for (int l = kMaxLevel; l >= 0; l--)
    if ((level_mask >> l) & 1u) {
      hi_level = l;
      break;
    }
  g.shift = lo_level;
  for (int a = 0; a < 3; a++) {
    g.mn[a] = mn[a];
    g.mx[a] = mx[a];
    g.bits[a] = bit_width(uint64_t(mx[a] - mn[a]) >> g.shift);
  }
  g.lbits = bit_width(uint64_t(hi_level - lo_level));
  g.total = g.bits[0] + g.bits[1] + g.bits[2] + g.lbits;
  g.sh[2] = g.lbits;
  g.sh[1] = g.sh[2] + g.bits[2];
  g.sh[0] = g.sh[1] + g.bits[1];
  g.level_mask = level_mask;
  g.nlevels = 0;
  for (int l = 0; l <= kMaxLevel; l++)
    if ((level_mask >> l) & 1u) g.levels[g.nlevels++] = int8_t(l);
  for (int a = 0; a < 3; a++) g.umax[a] = uint64_t(g.mx[a] - g.mn[a]) >> g.shift;
  if (g.total > 64) {
    // two-word keys (wide.cuh): an exact-key table, per-level probes
    g.wide = 1;
    g.occ = kOccNone;
    return g;
  }
  const uint32_t force = flags & (AMRX_FLAG_LOOKUP_RECORDS | AMRX_FLAG_LOOKUP_HASH |
                                  AMRX_FLAG_LOOKUP_DIRECTORY);
  if (force & (force - 1))
    fail(AMRX_ERR_INVALID_ARG, "more than one AMRX_FLAG_LOOKUP_* flag");
  const int occ_bits = std::max(0, g.total - kOccShift);
  const uint64_t dense_bytes = occ_bits <= 32 ? uint64_t(8) << occ_bits : ~0ull;
  if (force == AMRX_FLAG_LOOKUP_DIRECTORY) {
    g.occ = kOccNone;
  } else if (force == AMRX_FLAG_LOOKUP_HASH) {
    g.occ = kOccHash;
  } else if (force == AMRX_FLAG_LOOKUP_RECORDS) {
    if (dense_bytes > (uint64_t(64) << 30))
      fail(AMRX_ERR_UNSUPPORTED, "dense occupancy records for a " + std::to_string(g.total) +
                                   "-bit key space would exceed 64 GB (use the hash lookup)");
    g.occ = kOccDense;
  } else {
    g.occ = dense_bytes <= std::max<uint64_t>(192 * n, uint64_t(1) << 30) ? kOccDense
                                                                          : kOccHash;
  }
  g.dir_bits = g.occ == kOccNone ? directory_bits(g, n) : occ_bits;
  // records: buckets of 32 key values whatever the width (a key space of
  // fewer than 5 bits is one bucket), so lookups shift by a constant
  g.dir_shift = g.occ == kOccNone ? g.total - g.dir_bits : kOccShift;

  g.aligned = 1;
  for (int a = 0; a < 3; a++)
    if (mn[a] & ((int64_t(1) << hi_level) - 1)) g.aligned = 0;
  const uint64_t lmask = (uint64_t(1) << g.lbits) - 1;
  for (int L = 0; L < 32; L++) {
    uint64_t clear = lmask;
    if (L >= g.shift)
      for (int a = 0; a < 3; a++) {
        const int low = std::min(L - g.shift, g.bits[a]);
        clear |= ((uint64_t(1) << low) - 1) << g.sh[a];
      }
    g.cmask[L] = ~clear;
  }
  return g;
}

void finish_info(amrx_index *ix, uint64_t equal_pairs, double ms)
{
  amrx_index_info &in = ix->info;
  in.cell_count = ix->n;
  in.level_count = ix->g.nlevels;
  in.max_level = ix->g.nlevels ? ix->g.levels[ix->g.nlevels - 1] : 0;
  for (int l = 0; l < ix->g.nlevels; l++) in.levels[l] = ix->g.levels[l];
  for (int a = 0; a < 3; a++) {
    in.bounds_lo[a] = ix->g.mn[a];
    in.bounds_hi[a] = ix->bounds_hi[a];
  }
  in.key_bits = ix->g.total;
  in.lookup = ix->g.wide ? AMRX_LOOKUP_WIDE
              : ix->g.occ == kOccDense  ? AMRX_LOOKUP_RECORDS
              : ix->g.occ == kOccHash ? AMRX_LOOKUP_HASH
                                      : AMRX_LOOKUP_DIRECTORY;
  in.directory_bits =
    (ix->g.occ == kOccHash || ix->g.wide) ? bit_width(ix->hmask) : ix->g.dir_bits;
  in.duplicate_keys = equal_pairs;
  in.device_bytes = ix->keys.bytes + ix->scal.bytes + ix->dir.bytes +
                    ix->rec.bytes;
  in.seconds_ingest = ms / 1000.0;
}

void setup_stream(amrx_index *ix, const amrx_index_opts *opts)
{
  int dev = opts && opts->device >= 0 ? opts->device : -1;
  if (dev < 0) AMRX_CUDA(cudaGetDevice(&dev));
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(AMRX_ERR_NO_DEVICE, "no CUDA device available");
  }
  ix->device = dev;
  AMRX_CUDA(cudaSetDevice(dev));
  enable_pool_caching(dev);
  if (opts && opts->stream) {
    ix->stream = static_cast<cudaStream_t>(opts->stream);
  } else {
    AMRX_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
    ix->own_stream = true;
  }
}

/// bring the device-side lookup structure + padding up for sorted keys;
/// ix->order receives {descents, equal pairs, longest hash probe}
void finalize_index(amrx_index *ix, const uint32_t *tile_starts = nullptr)
{
  cudaStream_t st = ix->stream;
  pad_keys(ix->keys.as<uint64_t>(), ix->n, st);
  const uint64_t entries = (uint64_t(1) << ix->g.dir_bits) + 1;
  ix->order.reserve(32, st);
  AMRX_CUDA(cudaMemsetAsync(ix->order.ptr, 0, 32, st));
  auto *order = ix->order.as<unsigned long long>();
  if (!ix->searchable) return;
  if (ix->g.occ == kOccDense) {
    ix->rec.reserve((ix->rec_n ? ix->rec_n + 1 : entries) * sizeof(uint2), st);
    build_directory(ix->keys.as<uint64_t>(), ix->n, ix->g, nullptr, ix->rec.as<uint2>(), order,
                    ix->scratch, st, ix->rec_lo, ix->rec_n, ix->rec_n ? nullptr : tile_starts);
    ix->info.lookup_entries = ix->rec_n ? ix->rec_n + 1 : entries;
  } else if (ix->g.occ == kOccHash) {
    const uint64_t buckets = hash_count(ix->keys.as<uint64_t>(), ix->n, ix->g, order,
                                        ix->scratch, st);
    // >= 12 entries per occupied record bucket: most lookups end in their
    // home table bucket, a miss after one load (deep, 143M cells: 3 entries
    // 69.3 ms extraction, 6: 62.5, 12: 59.7, 24: 58.2 with a slower build);
    // fewer (>= 3) when the table would pass 48 GB
#ifndef AMRX_HASH_ENTRIES
#define AMRX_HASH_ENTRIES 12
#endif
    uint64_t tb = 32;
    while (2 * tb < AMRX_HASH_ENTRIES * buckets) tb <<= 1;
    while (tb * sizeof(ulonglong4) > (uint64_t(48) << 30) && 2 * (tb / 2) >= 3 * buckets)
      tb >>= 1;
    if (tb > (uint64_t(1) << 32))
      fail(AMRX_ERR_UNSUPPORTED, "hashed records: more than 2^32 table buckets");
    ix->rec.reserve(tb * sizeof(ulonglong4), st);
    ix->hmask = tb - 1;
    build_hash(ix->keys.as<uint64_t>(), ix->n, ix->g, ix->rec.as<ulonglong4>(), tb,
               reinterpret_cast<unsigned int *>(order + 2), st);
    ix->info.lookup_entries = 2 * tb;
  } else {
    ix->dir.reserve(entries * sizeof(uint32_t), st);
    build_directory(ix->keys.as<uint64_t>(), ix->n, ix->g, ix->dir.as<uint32_t>(), nullptr,
                    order, ix->scratch, st);
    ix->info.lookup_entries = entries;
  }
}

/*! the order check fused into the lookup build (after the stream has
    synchronised): sorted keys may not descend; equal neighbours are
    duplicate cells */
uint64_t sorted_equal_pairs(amrx_index *ix)
{
  unsigned long long h[3];
  AMRX_CUDA(cudaMemcpy(h, ix->order.ptr, sizeof h, cudaMemcpyDeviceToHost));
  if (h[0] != 0) fail(AMRX_ERR_INTERNAL, "index keys are not in (i,j,k,level) order");
  ix->info.max_probe = uint32_t(h[2]);
  return h[1];
}

/*! an index with duplicate keys cannot use occupancy records (positions
    are not popcounts): it switches to the bucket directory */
void ensure_search_dir(amrx_index *ix, uint64_t equal_pairs)
{
  if (ix->g.occ == kOccNone || equal_pairs == 0 || !ix->searchable) return;
  if (ix->partition)
    fail(AMRX_ERR_UNSUPPORTED, "a partition of a distributed index needs unique cells (" +
                                 std::to_string(equal_pairs) + " duplicate keys)");
  ix->rec.release();
  ix->g.occ = kOccNone;
  ix->g.dir_bits = directory_bits(ix->g, ix->n);
  ix->g.dir_shift = ix->g.total - ix->g.dir_bits;
  ix->info.max_probe = 0;
  const uint64_t entries = (uint64_t(1) << ix->g.dir_bits) + 1;
  ix->info.lookup_entries = entries;
  ix->dir.reserve(entries * sizeof(uint32_t), ix->stream);
  build_directory(ix->keys.as<uint64_t>(), ix->n, ix->g, ix->dir.as<uint32_t>(), nullptr,
                  ix->order.as<unsigned long long>(), ix->scratch, ix->stream);
}

void require_searchable(const amrx_index *ix)
{
  if (ix && !ix->searchable)
    fail(AMRX_ERR_INVALID_ARG, "this index holds sorted arrays only (amrx_index_sort_part)");
}

/// point queries (find_exact, snap, try_build_dual, validate) need every
/// cell: a partition holds one key range plus its halo
void require_full(const amrx_index *ix)
{
  require_searchable(ix);
  if (ix && ix->partition)
    fail(AMRX_ERR_INVALID_ARG, "point queries need a full index; this is one partition of a "
                               "distributed index (extract its owned cell range instead)");
}

void check_range(const amrx_index *ix, const amrx_range *range, uint64_t &b,
                 uint64_t &e)
{
  const uint64_t lo = std::min(ix->safe_lo, ix->n), hi = std::min(ix->safe_hi, ix->n);
  b = range ? range->cell_begin : lo;
  e = range ? std::min<uint64_t>(range->cell_end, ix->n) : hi;
  if (b > e) fail(AMRX_ERR_INVALID_ARG, "cell range begins after it ends");
  if (b < e && (b < lo || e > hi))
    fail(AMRX_ERR_INVALID_ARG, "cell range [" + std::to_string(b) + ", " + std::to_string(e) +
                                 ") leaves the partition's interior [" + std::to_string(lo) +
                                 ", " + std::to_string(hi) + "): its halo cells' neighbours "
                                 "live on other ranks");
}

void fill_stats(amrx_stats *st, const ExtractResult &r, uint64_t cells)
{
  if (!st) return;
  std::memset(st, 0, sizeof *st);
  st->cell_count = cells;
  st->duals_accepted = r.counters[0];
  st->duals_missing_corner = r.counters[1];
  st->duals_finer_corner = r.counters[2];
  st->duals_lower_key_corner = r.counters[3];
  st->pass1_triangle_count = r.tris_counted;
  st->fat_triangle_count = r.tris_written;
  st->dual_count = r.duals;
  st->seconds_pass1 = r.ms / 1000.0;
  st->seconds_pass2 = r.ms2 / 1000.0;
  st->kernel_launches = r.launches;
}

/// internal-consistency checks of pipeline.cpp:106-107,130-138
void check_result(const ExtractResult &r, uint64_t cells, bool tri)
{
  if (r.error_flags & 1u)
    fail(AMRX_ERR_INTERNAL, "contour_hex: case table selected a collapsed edge");
  if (r.error_flags & 2u)
    fail(AMRX_ERR_INTERNAL, "extract: candidate left undecided");
  const uint64_t total = r.counters[0] + r.counters[1] + r.counters[2] + r.counters[3];
  if (total != cells * 8)
    fail(AMRX_ERR_INTERNAL, "extract_isosurface: candidate accounting broken");
  if (tri && r.tris_counted != r.tris_written)
    fail(AMRX_ERR_INTERNAL,
         "extract_isosurface: pass 2 emitted a different number of "
         "triangles than pass 1 counted");
}

}  // namespace

namespace amrx {

/// the extraction over whichever key width the index has
ExtractResult run_any(amrx_index *index, const ExtractRequest &rq, cudaStream_t st)
{
  return index->g.wide ? run_extract_wide(rq, index->wctx(), st) : run_extract(rq, st);
}

void extract_dual_impl(amrx_index *index, const amrx_range *range, uint32_t *corners8,
                     uint64_t *task_ids, uint64_t cap, uint64_t *count, amrx_stats *stats,
                     bool cached)
{
  require_searchable(index);
  if (!index || !count) fail(AMRX_ERR_INVALID_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock(index->mu);
  DeviceGuard dg(index->device);
  cudaStream_t st = index->stream;
  uint64_t b, e;
  check_range(index, range, b, e);
  const uint64_t cells = e - b;
  auto &C = index->cache;
  // device memory or pinned host memory: written by the rounds directly
  uint32_t *corners_w = static_cast<uint32_t *>(device_writable(corners8));
  uint64_t *tasks_w = static_cast<uint64_t *>(device_writable(task_ids));
  const bool dev_out = !cached && corners_w && (!task_ids || tasks_w);

  ExtractRequest rq{};
  rq.s = index->ctx();
  rq.g = index->g;
  rq.scal = index->scal.as<double>();
  rq.unique = index->info.duplicate_keys == 0;
  rq.cell_begin = b;
  rq.cell_end = e;
  rq.emit_dual = true;
  if (dev_out) {
    rq.final_host = !is_device_ptr(corners8);
    rq.corners = rq.final_host ? corners8 : corners_w;
    rq.tasks = rq.final_host ? task_ids : tasks_w;
    rq.dual_cap = cap;
    const ExtractResult r = run_any(index, rq, st);
    check_result(r, cells, false);
    fill_stats(stats, r, cells);
    *count = r.duals;
    C.valid = false;
    if (r.duals > cap)
      fail(AMRX_ERR_CAPACITY, "output capacity " + std::to_string(cap) +
                                " < " + std::to_string(r.duals) + " duals");
    return;
  }
  // pageable host (or absent) output: extract into the index's device
  // arena, which grows to fit, and keep it for the count-then-copy pattern
  const bool hit = C.valid && C.kind == 1 && C.begin == b && C.end == e;
  if (!hit) {
    C.valid = false;
    rq.grow_a = &index->out_a;
    rq.grow_b = &index->out_b;
    const ExtractResult r = run_any(index, rq, st);
    check_result(r, cells, false);
    C.valid = true;
    C.kind = 1;
    C.begin = b;
    C.end = e;
    C.count = r.duals;
    fill_stats(&C.stats, r, cells);
  }
  *count = C.count;
  if (stats) *stats = C.stats;
  if (!corners8 && !task_ids) return;  // count query
  if (C.count > cap)
    fail(AMRX_ERR_CAPACITY, "output capacity " + std::to_string(cap) + " < " +
                              std::to_string(C.count) + " duals");
  if (corners8 && C.count)
    AMRX_CUDA(cudaMemcpyAsync(corners8, index->out_a.ptr, C.count * 32,
                              cudaMemcpyDefault, st));
  if (task_ids && C.count)
    AMRX_CUDA(cudaMemcpyAsync(task_ids, index->out_b.ptr, C.count * 8,
                              cudaMemcpyDefault, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
}

void extract_iso_impl(amrx_index *index, const amrx_range *range,
                    const amrx_iso_params *params, void *xyz9, uint64_t cap,
                    uint64_t *count, amrx_stats *stats, bool cached)
{
  require_searchable(index);
  if (!index || !count || !params) fail(AMRX_ERR_INVALID_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> lock(index->mu);
  DeviceGuard dg(index->device);
  cudaStream_t st = index->stream;
  uint64_t b, e;
  check_range(index, range, b, e);
  const uint64_t cells = e - b;
  const size_t tri_bytes = params->xyz_is_f32 ? 36 : 72;
  auto &C = index->cache;
  // device memory or pinned host memory: written by the rounds directly
  void *xyz_w = device_writable(xyz9);
  const bool dev_out = !cached && xyz_w != nullptr;

  ExtractRequest rq{};
  rq.s = index->ctx();
  rq.g = index->g;
  rq.scal = index->scal.as<double>();
  rq.unique = index->info.duplicate_keys == 0;
  rq.cell_begin = b;
  rq.cell_end = e;
  rq.emit_tri = true;
  rq.tri_f32 = params->xyz_is_f32 != 0;
  rq.iso = params->iso;
  const auto length_check = [&](uint64_t tris) {
    if (params->check_length &&
        tris > uint64_t(std::numeric_limits<uint32_t>::max()) / 3)
      fail(AMRX_ERR_LENGTH, "extract_isosurface: mesh too large for 32-bit indices");
  };
  if (dev_out) {
    rq.final_host = !is_device_ptr(xyz9);
    rq.xyz = rq.final_host ? xyz9 : xyz_w;
    rq.tri_cap = cap;
    // pinned host output of a large input: small first rounds, each
    // round's download overlapping the next round's extraction
    rq.stream_rounds = rq.final_host && cells >= (uint64_t(1) << 24);
    const ExtractResult r = run_any(index, rq, st);
    check_result(r, cells, true);
    fill_stats(stats, r, cells);
    *count = r.tris_written;
    C.valid = false;
    length_check(r.tris_written);
    if (r.tris_written > cap)
      fail(AMRX_ERR_CAPACITY, "output capacity " + std::to_string(cap) +
                                " < " + std::to_string(r.tris_written) + " triangles");
    return;
  }
  const bool hit = C.valid && C.kind == 2 && C.begin == b && C.end == e &&
                   C.iso == params->iso && C.f32 == params->xyz_is_f32;
  if (!hit) {
    C.valid = false;
    rq.grow_a = &index->out_a;
    const ExtractResult r = run_any(index, rq, st);
    check_result(r, cells, true);
    C.valid = true;
    C.kind = 2;
    C.begin = b;
    C.end = e;
    C.iso = params->iso;
    C.f32 = params->xyz_is_f32;
    C.count = r.tris_written;
    fill_stats(&C.stats, r, cells);
  }
  *count = C.count;
  if (stats) *stats = C.stats;
  length_check(C.count);
  if (!xyz9) return;  // count query
  if (C.count > cap)
    fail(AMRX_ERR_CAPACITY, "output capacity " + std::to_string(cap) + " < " +
                              std::to_string(C.count) + " triangles");
  if (C.count)
    AMRX_CUDA(cudaMemcpyAsync(xyz9, index->out_a.ptr, C.count * tri_bytes,
                              cudaMemcpyDefault, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
}

}  // namespace amrx

extern "C" {

const char *amrx_last_error(void) { return g_last_error.c_str(); }

const char *amrx_version(void) { return "amrx 0.1 (sm_100a)"; }

uint64_t amrx_kernel_launches(void) { return g_launches.load(); }

void amrx_debug_round_limit(uint64_t items) { amrx::g_round_limit.store(items); }

namespace {

/*! build_index over n_cells records.  g16 = NULL: the geometry comes from
    the records' own bounds; else from the global geometry words of a
    distributed build (every record must lie inside them).  search = false:
    stop after the sort (sorted keys + scalars only, for the exchange). */
void create_impl(const int32_t *cells4, const double *scalars, uint64_t n_cells,
                 uint64_t n_scalars, const amrx_index_opts *opts, const int64_t *g16,
                 bool search, amrx_index **out)
{
  {
    NvtxRange range("amrx build_index");
    if (!out) fail(AMRX_ERR_INVALID_ARG, "out is null");
    *out = nullptr;
    // locator.cpp:29-36, same order and wording
    if (n_cells == 0) fail(AMRX_ERR_LOAD, "dataset is empty");
    if (n_cells != n_scalars)
      fail(AMRX_ERR_LOAD, "cell count " + std::to_string(n_cells) +
                            " does not match scalar count " +
                            std::to_string(n_scalars));
    if (n_cells > uint64_t(std::numeric_limits<uint32_t>::max()))
      fail(AMRX_ERR_LOAD, "dataset too large for 32-bit cell ids");
    if (!cells4 || !scalars) fail(AMRX_ERR_INVALID_ARG, "null input array");

    auto ix = std::make_unique<amrx_index>();
    setup_stream(ix.get(), opts);
    cudaStream_t st = ix->stream;
    const uint64_t n = n_cells;
    ix->n = n;

    cudaEvent_t e0, e1;
    AMRX_CUDA(cudaEventCreate(&e0));
    AMRX_CUDA(cudaEventCreate(&e1));
    AMRX_CUDA(cudaEventRecord(e0, st));

    // inputs: device pointers are used in place; host arrays are staged
    // into workspace slots.  The scalar upload runs on a side stream so it
    // overlaps the pack + radix sort (the scalars are first needed by the
    // gather that follows the sort).
    WsLease l_cells, l_scal, l_idx, l_ialt, l_sort;
    const int4 *cells_d = reinterpret_cast<const int4 *>(device_view(cells4));
    if (!cells_d) {
      cells_d = static_cast<const int4 *>(l_cells.get(kWsCells, n * 16, st));
      AMRX_CUDA(cudaMemcpyAsync(const_cast<int4 *>(cells_d), cells4, n * 16,
                                cudaMemcpyHostToDevice, st));
    }
    // host scalars are uploaded after the cells, in chunks on a side stream:
    // they are first needed once the keys are sorted, and each chunk is
    // scattered into key order as soon as it lands (scalar_chunks below)
    const double *sc_d = static_cast<const double *>(device_view(scalars));
    constexpr int kScalChunks = 8;
    cudaStream_t aux = nullptr;
    cudaEvent_t sc_ev[kScalChunks] = {};
    cudaEvent_t sc_ready = nullptr;  // all chunks landed
    uint64_t sc_cut[kScalChunks + 1] = {};
    if (!sc_d) {
      sc_d = static_cast<const double *>(l_scal.get(kWsScal, n * 8, st));
      AMRX_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
      for (int c = 0; c < kScalChunks; c++)
        AMRX_CUDA(cudaEventCreateWithFlags(&sc_ev[c], cudaEventDisableTiming));
      // the slot is free and the cells copy queued in st order: the side
      // stream starts after it, so the cells get the host link first
      AMRX_CUDA(cudaEventRecord(sc_ev[0], st));
      AMRX_CUDA(cudaStreamWaitEvent(aux, sc_ev[0], 0));
      for (int c = 0; c <= kScalChunks; c++) sc_cut[c] = n * uint64_t(c) / kScalChunks;
      for (int c = 0; c < kScalChunks; c++) {
        if (sc_cut[c + 1] > sc_cut[c])
          AMRX_CUDA(cudaMemcpyAsync(const_cast<double *>(sc_d) + sc_cut[c], scalars + sc_cut[c],
                                    (sc_cut[c + 1] - sc_cut[c]) * 8, cudaMemcpyHostToDevice,
                                    aux));
        AMRX_CUDA(cudaEventRecord(sc_ev[c], aux));
      }
      sc_ready = sc_ev[kScalChunks - 1];
    }
    struct AuxGuard {
      cudaStream_t s;
      cudaEvent_t *e;
      int ne;
      ~AuxGuard()
      {
        if (s) {
          cudaStreamSynchronize(s);
          cudaStreamDestroy(s);
        }
        for (int c = 0; c < ne; c++)
          if (e[c]) cudaEventDestroy(e[c]);
      }
    } aux_guard{aux, sc_ev, kScalChunks};

    nvtxRangePushA("prepass");
    const PrepassResult pre = ingest_prepass(cells_d, n, ix->scratch, st);
    nvtxRangePop();
    if (pre.first_bad != ~0ull) {
      int4 c;
      AMRX_CUDA(cudaMemcpy(&c, cells_d + pre.first_bad, sizeof c,
                           cudaMemcpyDeviceToHost));
      const std::string rec = "record " + std::to_string(pre.first_bad);
      if (c.w < 0 || c.w > kMaxLevel)
        fail(AMRX_ERR_LOAD, rec + ": level " + std::to_string(c.w) +
                              " out of range [0," + std::to_string(kMaxLevel) + "]");
      fail(AMRX_ERR_LOAD, rec + ": anchor (" + std::to_string(c.x) + " " +
                            std::to_string(c.y) + " " + std::to_string(c.z) +
                            ") is not a multiple of the level-" +
                            std::to_string(c.w) + " cell width");
    }
    ix->searchable = search;
    if (g16) {
      for (int a = 0; a < 3; a++)
        if (pre.mn[a] < g16[a] || pre.mx[a] > g16[3 + a])
          fail(AMRX_ERR_INVALID_ARG, "records outside the given geometry");
      if ((pre.level_mask & ~uint32_t(g16[9])) != 0)
        fail(AMRX_ERR_INVALID_ARG, "records on levels outside the given geometry");
      const int64_t mn[3] = {g16[0], g16[1], g16[2]};
      const int64_t mx[3] = {g16[3], g16[4], g16[5]};
      ix->g = make_geometry(mn, mx, uint32_t(g16[9]), uint64_t(g16[10]), opts ? opts->flags : 0);
      for (int a = 0; a < 3; a++) ix->bounds_hi[a] = g16[6 + a];
    } else {
      const int64_t mn[3] = {pre.mn[0], pre.mn[1], pre.mn[2]};
      const int64_t mx[3] = {pre.mx[0], pre.mx[1], pre.mx[2]};
      ix->g = make_geometry(mn, mx, pre.level_mask, n, opts ? opts->flags : 0);
      for (int a = 0; a < 3; a++) ix->bounds_hi[a] = pre.hi[a];
    }

    if (ix->g.wide) {
      if (g16 || !search)
        fail(AMRX_ERR_UNSUPPORTED, "distributed builds need keys of at most 64 bits (this "
                                   "dataset's extent needs " + std::to_string(ix->g.total) + ")");
      if (sc_ready) AMRX_CUDA(cudaStreamWaitEvent(st, sc_ready, 0));
      ix->keys.reserve(n * 16 + 256, st);
      ix->scal.reserve(n * sizeof(double), st);
      const WideBuild wb = wide_build(cells_d, sc_d, n, ix->g, ix->keys.as<ulonglong2>(),
                                      ix->scal.as<double>(), ix->rec, st);
      ix->hmask = wb.entries - 1;
      ix->info.lookup_entries = wb.entries;
      ix->info.max_probe = wb.max_probe;
      AMRX_CUDA(cudaEventRecord(e1, st));
      AMRX_CUDA(cudaStreamSynchronize(st));
      float ms = 0;
      AMRX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      finish_info(ix.get(), wb.equal_pairs, ms);
      *out = ix.release();
      return;
    }
    ix->keys.reserve((n + kKeyPad) * sizeof(uint64_t), st);
    // resident scalars travel through the sort as the payload (read in
    // input order by the first pass); arriving scalars need the positions
    uint32_t *idx = aux ? static_cast<uint32_t *>(l_idx.get(kWsIdx, n * 4, st)) : nullptr;
    // one pass over the cells: keys, the sort's digit histograms (into the
    // sort's scratch) and the order check
    void *sort_scratch = l_sort.get(kWsSort, radix_sort_scratch_bytes(n), st);
    auto *digit_hist = static_cast<unsigned int *>(sort_scratch);
    ix->scratch.reserve(16, st);
    auto *order2 = ix->scratch.as<unsigned long long>();
    nvtxRangePushA("pack + sort");
    ingest_pack(cells_d, n, ix->g, ix->keys.as<uint64_t>(), idx, st, digit_hist,
                (ix->g.total + kSortRadixBits - 1) / kSortRadixBits, order2);

    TileStarts tstarts;  // record-tile starts from the sort's last pass
    DevBuf tstarts_buf;
    uint64_t desc = 0, eq = 0;
    uint32_t *rank = nullptr;
    bool scatter_pending = false;
    {
      unsigned long long h2[2];
      AMRX_CUDA(cudaMemcpyAsync(h2, order2, 16, cudaMemcpyDeviceToHost, st));
      AMRX_CUDA(cudaStreamSynchronize(st));
      desc = h2[0];
      eq = h2[1];
    }
    ix->scal.reserve(n * sizeof(double), st);
    if (desc == 0) {
      // already in (i,j,k,level) order; stable ties mean identity
      if (sc_ready) AMRX_CUDA(cudaStreamWaitEvent(st, sc_ready, 0));
      AMRX_CUDA(cudaMemcpyAsync(ix->scal.ptr, sc_d, n * sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
    } else {
      if (opts && (opts->flags & AMRX_FLAG_PRESORTED))
        fail(AMRX_ERR_INVALID_ARG, "input flagged presorted is not sorted");
      // the sort ping-pongs with a pool buffer the size of the key array;
      // if the keys end there the two buffers trade places (no copy).  The
      // last pass writes the scalars in key order (the gather, fused)
      DevBuf keys_alt;
      keys_alt.reserve((n + kKeyPad) * sizeof(uint64_t), st);
      int passes = 0;
      bool in_alt = false;
      if (ix->searchable && ix->g.occ == kOccDense) {
        // dense records of the whole index: the last pass finds the record
        // tiles' first positions (no separate sweep over the sorted keys)
        tstarts.tiles = ((uint64_t(1) << ix->g.dir_bits) + 1 + (uint64_t(1) << kRecTileLog) - 1) >>
                        kRecTileLog;
        tstarts_buf.reserve(size_t(tstarts.tiles + 1) * 4, st);
        tstarts.starts = tstarts_buf.as<uint32_t>();
        tstarts.shift = ix->g.dir_shift;
      }
      if (aux) {
        // arriving scalars: the last pass leaves the inverse permutation
        // for the chunk scatters
        auto *idx_alt = static_cast<uint32_t *>(l_ialt.get(kWsIdxAlt, n * 4, st));
        in_alt = radix_sort_pairs(ix->keys.as<uint64_t>(), idx, keys_alt.as<uint64_t>(),
                                  idx_alt, n, ix->g.total, sort_scratch, st, &passes, nullptr,
                                  nullptr, nullptr, &rank, digit_hist, &tstarts);
      } else {
        // resident scalars: the sort's 64-bit payload from the first pass
        // on (coalesced reads in input order; no gather, no positions)
        DevBuf scal_alt;
        scal_alt.reserve(n * sizeof(double), st);
        in_alt = radix_sort_pairs_u64(ix->keys.as<uint64_t>(),
                                      reinterpret_cast<const uint64_t *>(sc_d),
                                      ix->scal.as<uint64_t>(), keys_alt.as<uint64_t>(),
                                      scal_alt.as<uint64_t>(), n, ix->g.total, sort_scratch, st,
                                      &passes, digit_hist, &tstarts);
        if (in_alt) {
          std::swap(ix->scal.ptr, scal_alt.ptr);
          std::swap(ix->scal.bytes, scal_alt.bytes);
          std::swap(ix->scal.stream, scal_alt.stream);
        }
      }
      if (in_alt) {
        std::swap(ix->keys.ptr, keys_alt.ptr);
        std::swap(ix->keys.bytes, keys_alt.bytes);
        std::swap(ix->keys.stream, keys_alt.stream);
      }
      scatter_pending = aux != nullptr;
    }
    nvtxRangePop();
    nvtxRangePushA("lookup structure");
    finalize_index(ix.get(), tstarts.filled ? tstarts.starts : nullptr);
    nvtxRangePop();
    if (scatter_pending) {
      for (int c = 0; c < kScalChunks; c++) {
        AMRX_CUDA(cudaStreamWaitEvent(st, sc_ev[c], 0));
        if (rank)
          scatter_f64(rank + sc_cut[c], sc_d + sc_cut[c], ix->scal.as<double>(),
                      sc_cut[c + 1] - sc_cut[c], st);
      }
      if (!rank)  // no pass permuted anything
        AMRX_CUDA(cudaMemcpyAsync(ix->scal.ptr, sc_d, n * sizeof(double),
                                  cudaMemcpyDeviceToDevice, st));
    }
    AMRX_CUDA(cudaEventRecord(e1, st));
    AMRX_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    AMRX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    {
      const uint64_t eq = sorted_equal_pairs(ix.get());
      ensure_search_dir(ix.get(), eq);
      finish_info(ix.get(), eq, ms);
    }
    *out = ix.release();
  }
}

}  // namespace

amrx_status amrx_index_create(const int32_t *cells4, const double *scalars,
                              uint64_t n_cells, uint64_t n_scalars,
                              const amrx_index_opts *opts, amrx_index **out)
{
  return guarded([&] { create_impl(cells4, scalars, n_cells, n_scalars, opts, nullptr, true, out); });
}

}  // extern "C"

namespace {

constexpr char kAmrMagic[8] = {'A', 'M', 'R', 'C', 'E', 'L', 'L', '1'};
constexpr uint64_t kAmrHeader = 24, kAmrRecord = 24;  // io.cpp:35-37

/// build_index errors re-raised with the path in front (io.cpp:122-125)
template <typename Fn>
void with_path(const std::string &path, Fn &&fn)
{
  try {
    fn();
  } catch (const ApiError &e) {
    if (e.code != AMRX_ERR_LOAD) throw;
    fail(AMRX_ERR_LOAD, path + ": " + e.what());
  }
}

struct Fd {
  int fd = -1;
  ~Fd()
  {
    if (fd >= 0) ::close(fd);
  }
};

constexpr int kReadThreads = 8;
constexpr uint64_t kReadChunk = uint64_t(1) << 19;  // records per chunk (12 MiB)

/// pinned chunks + their "upload done" events, kept for the process
/// (cudaHostAlloc of the ring costs more than reading a small file)
struct PinnedRing {
  int device = -1;
  std::vector<void *> host;
  std::vector<cudaEvent_t> done;
};
std::mutex g_read_ring_mu;

PinnedRing &read_ring(int dev)
{
  static PinnedRing r;
  if (r.device != dev) {
    for (void *p : r.host) cudaFreeHost(p);
    for (cudaEvent_t e : r.done) cudaEventDestroy(e);
    r.host.clear();
    r.done.clear();
    for (int b = 0; b < 2 * kReadThreads; b++) {
      void *h = nullptr;
      AMRX_CUDA(cudaHostAlloc(&h, kReadChunk * kAmrRecord, cudaHostAllocDefault));
      r.host.push_back(h);
      cudaEvent_t e;
      AMRX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      r.done.push_back(e);
    }
    r.device = dev;
  }
  return r;
}

/*! read_amr_binary (io.cpp:76-126) feeding the GPU: the header checks in
    the reference's order and wording, then the records stream through a
    ring of pinned chunks (pread on the host overlaps the upload and the
    device-side split of the previous chunk) straight into device arrays,
    which build_index then takes as device input.  No host copy of the
    dataset is ever materialised. */
void read_amr_binary(const std::string &path, const amrx_index_opts *opts, amrx_index **out)
{
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY);
  struct stat sb;
  if (f.fd < 0 || ::fstat(f.fd, &sb) != 0 || !S_ISREG(sb.st_mode))
    fail(AMRX_ERR_LOAD, path + ": cannot open file");
  const uint64_t size = uint64_t(sb.st_size);
  auto read_at = [&](void *dst, uint64_t bytes, uint64_t off) {
    auto *p = static_cast<char *>(dst);
    while (bytes) {
      const ssize_t got = ::pread(f.fd, p, bytes, off_t(off));
      if (got <= 0) fail(AMRX_ERR_LOAD, path + ": read error");
      p += got;
      off += uint64_t(got);
      bytes -= uint64_t(got);
    }
  };
  if (size < kAmrHeader) fail(AMRX_ERR_LOAD, path + ": file shorter than the 24-byte header");
  unsigned char hdr[kAmrHeader];
  read_at(hdr, kAmrHeader, 0);
  uint32_t version, fields;
  uint64_t n;
  std::memcpy(&version, hdr + 8, 4);
  std::memcpy(&n, hdr + 12, 8);
  std::memcpy(&fields, hdr + 20, 4);
  if (std::memcmp(hdr, kAmrMagic, 8) != 0)
    fail(AMRX_ERR_LOAD, path + ": bad magic, not a cell data file");
  if (version != 1) fail(AMRX_ERR_LOAD, path + ": unsupported version " + std::to_string(version));
  if (fields != 1)
    fail(AMRX_ERR_LOAD,
         path + ": expected exactly 1 field, file declares " + std::to_string(fields));
  if (n == 0) fail(AMRX_ERR_LOAD, path + ": file declares zero cells");
  const uint64_t expected = kAmrHeader + n * kAmrRecord;
  if (size < expected)
    fail(AMRX_ERR_LOAD, path + ": truncated: header declares " + std::to_string(n) +
                          " cells but only " + std::to_string((size - kAmrHeader) / kAmrRecord) +
                          " fit in the file");
  if (size > expected)
    fail(AMRX_ERR_LOAD, path + ": " + std::to_string(size - expected) +
                          " trailing bytes after the last record");

  // build_index's 32-bit CellId limit before staging 24 B per record on the
  // device (the reference would first scan the scalars of such a file)
  if (n > uint64_t(std::numeric_limits<uint32_t>::max()))
    fail(AMRX_ERR_LOAD, path + ": dataset too large for 32-bit cell ids");
  int dev = opts && opts->device >= 0 ? opts->device : -1;
  if (dev < 0) AMRX_CUDA(cudaGetDevice(&dev));
  DeviceGuard dg(dev);
  enable_pool_caching(dev);
  cudaStream_t st = nullptr;
  AMRX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamOwner {
    cudaStream_t s;
    ~StreamOwner() { cudaStreamDestroy(s); }
  } so{st};
  DevBuf cells, scal, bad, stage;
  cells.reserve(n * 16, st);
  scal.reserve(n * 8, st);
  bad.reserve(8, st);
  AMRX_CUDA(cudaMemsetAsync(bad.ptr, 0xff, 8, st));
  // two sets of T pinned chunks: the host threads pread set g % 2 while
  // the GPU uploads and splits the other one
  const int T = kReadThreads;
  const uint64_t chunks = (n + kReadChunk - 1) / kReadChunk;
  std::unique_lock<std::mutex> lock(g_read_ring_mu);
  PinnedRing &pr = read_ring(dev);
  stage.reserve(size_t(2 * T) * kReadChunk * kAmrRecord, st);
  std::vector<std::thread> pool;
  for (uint64_t g0 = 0, gi = 0; g0 < chunks; g0 += uint64_t(T), gi++) {
    const int set = int(gi & 1);
    const int m = int(std::min<uint64_t>(uint64_t(T), chunks - g0));
    for (int t = 0; t < m; t++) AMRX_CUDA(cudaEventSynchronize(pr.done[set * T + t]));
    std::atomic<bool> bad_read{false};
    pool.clear();
    for (int t = 0; t < m; t++)
      pool.emplace_back([&, t] {
        const uint64_t first = (g0 + uint64_t(t)) * kReadChunk;
        const uint64_t cnt = std::min(kReadChunk, n - first);
        auto *p = static_cast<char *>(pr.host[set * T + t]);
        uint64_t bytes = cnt * kAmrRecord, off = kAmrHeader + first * kAmrRecord;
        while (bytes) {
          const ssize_t got = ::pread(f.fd, p, bytes, off_t(off));
          if (got <= 0) {
            bad_read = true;
            return;
          }
          p += got;
          off += uint64_t(got);
          bytes -= uint64_t(got);
        }
      });
    for (auto &th : pool) th.join();
    if (bad_read) fail(AMRX_ERR_LOAD, path + ": read error");
    for (int t = 0; t < m; t++) {
      const int b = set * T + t;
      const uint64_t first = (g0 + uint64_t(t)) * kReadChunk;
      const uint64_t cnt = std::min(kReadChunk, n - first);
      void *dst = stage.as<char>() + size_t(b) * kReadChunk * kAmrRecord;
      AMRX_CUDA(cudaMemcpyAsync(dst, pr.host[b], cnt * kAmrRecord, cudaMemcpyHostToDevice, st));
      split_records(dst, cnt, first, cells.as<int4>(), scal.as<double>(),
                    bad.as<unsigned long long>(), st);
      AMRX_CUDA(cudaEventRecord(pr.done[b], st));
    }
  }
  unsigned long long first_bad = 0;
  AMRX_CUDA(cudaMemcpyAsync(&first_bad, bad.ptr, 8, cudaMemcpyDeviceToHost, st));
  AMRX_CUDA(cudaStreamSynchronize(st));
  stage.release();
  lock.unlock();
  if (first_bad != ~0ull)
    fail(AMRX_ERR_LOAD, path + ": record " + std::to_string(first_bad) + ": scalar is not finite");
  with_path(path, [&] {
    create_impl(cells.as<int32_t>(), scal.as<double>(), n, n, opts, nullptr, true, out);
  });
}

/// read_amr_text (io.cpp:128-176): one "i j k level scalar" per line, '#'
/// comments and blank lines skipped, parsed with the same stream
/// extraction so the accepted spellings are the reference's
void read_amr_text(const std::string &path, const amrx_index_opts *opts, amrx_index **out)
{
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(AMRX_ERR_LOAD, path + ": cannot open file");
  std::ostringstream buf;
  buf << in.rdbuf();
  if (!in && !in.eof()) fail(AMRX_ERR_LOAD, path + ": read error");
  std::istringstream lines(std::move(buf).str());
  std::vector<int32_t> cells;
  std::vector<double> scalars;
  std::string line;
  for (uint64_t no = 1; std::getline(lines, line); no++) {
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    if (line.find_first_not_of(" \t\r\v\f") == std::string::npos) continue;
    const std::string at = path + ": line " + std::to_string(no) + ": ";
    std::istringstream fields(line);
    long long v[4];
    double x;
    if (!(fields >> v[0] >> v[1] >> v[2] >> v[3] >> x))
      fail(AMRX_ERR_LOAD, at + "expected 'i j k level scalar'");
    std::string extra;
    if (fields >> extra) fail(AMRX_ERR_LOAD, at + "trailing characters '" + extra + "'");
    for (int a = 0; a < 3; a++)
      if (v[a] < std::numeric_limits<int32_t>::min() || v[a] > std::numeric_limits<int32_t>::max())
        fail(AMRX_ERR_LOAD, at + "anchor out of 32-bit range");
    if (v[3] < 0 || v[3] > 30)
      fail(AMRX_ERR_LOAD, at + "level " + std::to_string(v[3]) + " out of range");
    if (!std::isfinite(x)) fail(AMRX_ERR_LOAD, at + "scalar is not finite");
    for (int a = 0; a < 4; a++) cells.push_back(int32_t(v[a]));
    scalars.push_back(x);
  }
  with_path(path, [&] {
    create_impl(cells.data(), scalars.data(), scalars.size(), scalars.size(), opts, nullptr,
                true, out);
  });
}

}  // namespace

extern "C" {

amrx_status amrx_read_amr(const char *path, const amrx_index_opts *opts, amrx_index **out)
{
  return guarded([&] {
    if (!path || !out) fail(AMRX_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    const std::string p(path);
    if (std::filesystem::path(p).extension() == ".txt")
      read_amr_text(p, opts, out);
    else
      read_amr_binary(p, opts, out);
  });
}

amrx_status amrx_index_sort_part(const int32_t *cells4, const double *scalars,
                                 uint64_t n_cells, const int64_t *geometry16,
                                 const amrx_index_opts *opts, amrx_index **out)
{
  return guarded([&] {
    if (!geometry16) fail(AMRX_ERR_INVALID_ARG, "null geometry");
    create_impl(cells4, scalars, n_cells, n_cells, opts, geometry16, false, out);
  });
}

amrx_status amrx_bounds(const int32_t *cells4, uint64_t n_cells, const amrx_index_opts *opts,
                        int64_t *bounds10)
{
  return guarded([&] {
    if (!bounds10) fail(AMRX_ERR_INVALID_ARG, "null argument");
    if (n_cells == 0) fail(AMRX_ERR_LOAD, "dataset is empty");
    if (!cells4) fail(AMRX_ERR_INVALID_ARG, "null input array");
    int dev = opts && opts->device >= 0 ? opts->device : -1;
    if (dev < 0) AMRX_CUDA(cudaGetDevice(&dev));
    DeviceGuard dg(dev);
    cudaStream_t st = opts && opts->stream ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    DevIn<int4> cells(reinterpret_cast<const int4 *>(cells4), n_cells, st);
    DevBuf scratch;
    const PrepassResult pre = ingest_prepass(cells.ptr, n_cells, scratch, st);
    if (pre.first_bad != ~0ull)
      fail(AMRX_ERR_LOAD, "record " + std::to_string(pre.first_bad) +
                            ": level out of range or anchor not a multiple of the cell width");
    for (int a = 0; a < 3; a++) {
      bounds10[a] = pre.mn[a];
      bounds10[3 + a] = pre.mx[a];
      bounds10[6 + a] = pre.hi[a];
    }
    bounds10[9] = pre.level_mask;
  });
}

amrx_status amrx_index_from_keys(const void *keys_dev, const double *scalars_dev,
                                 uint64_t n_cells, const int64_t *g16,
                                 const amrx_index_opts *opts, amrx_index **out)
{
  return guarded([&] {
    if (!out || !keys_dev || !scalars_dev || !g16)
      fail(AMRX_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    if (n_cells == 0) fail(AMRX_ERR_LOAD, "dataset is empty");
    if (n_cells > uint64_t(std::numeric_limits<uint32_t>::max()))
      fail(AMRX_ERR_LOAD, "dataset too large for 32-bit cell ids");
    if (uint64_t(g16[14]) <= uint64_t(g16[13]))
      fail(AMRX_ERR_INVALID_ARG, "empty key range");
    auto ix = std::make_unique<amrx_index>();
    setup_stream(ix.get(), opts);
    cudaStream_t st = ix->stream;
    const uint64_t n = n_cells;
    ix->n = n;
    const int64_t mn[3] = {g16[0], g16[1], g16[2]};
    const int64_t mx[3] = {g16[3], g16[4], g16[5]};
    ix->g = make_geometry(mn, mx, uint32_t(g16[9]), uint64_t(g16[10]), opts ? opts->flags : 0);
    for (int a = 0; a < 3; a++) ix->bounds_hi[a] = g16[6 + a];
    if (ix->g.wide)
      fail(AMRX_ERR_UNSUPPORTED, "distributed indexes need keys of at most 64 bits");
    if (ix->g.occ == kOccNone)
      fail(AMRX_ERR_UNSUPPORTED, "a partition index needs occupancy records (dense or "
                                 "hashed), not the directory");
    ix->partition = true;
    ix->id_base = g16[12];
    ix->key_lo = uint64_t(g16[13]);
    ix->key_hi = uint64_t(g16[14]);
    if (ix->g.occ == kOccDense) {
      ix->rec_lo = ((ix->key_lo >> ix->g.dir_shift) >> kRecTileLog) << kRecTileLog;
      ix->rec_n = ((ix->key_hi - 1) >> ix->g.dir_shift) - ix->rec_lo + 1;
    }
    cudaEvent_t e0, e1;
    AMRX_CUDA(cudaEventCreate(&e0));
    AMRX_CUDA(cudaEventCreate(&e1));
    AMRX_CUDA(cudaEventRecord(e0, st));
    ix->keys.reserve((n + kKeyPad) * sizeof(uint64_t), st);
    ix->scal.reserve(n * sizeof(double), st);
    AMRX_CUDA(cudaMemcpyAsync(ix->keys.ptr, keys_dev, n * 8, cudaMemcpyDefault, st));
    uint64_t desc = 0, eq = 0;
    ingest_order_check(ix->keys.as<uint64_t>(), n, ix->scratch, &desc, &eq, st);
    if (desc == 0) {
      AMRX_CUDA(cudaMemcpyAsync(ix->scal.ptr, scalars_dev, n * 8, cudaMemcpyDefault, st));
    } else {
      // e.g. the sorted runs an all-to-all exchange delivers: one radix
      // sort, the last pass gathering the scalars
      WsLease l_idx, l_ialt, l_sort;
      auto *idx = static_cast<uint32_t *>(l_idx.get(kWsIdx, n * 4, st));
      fill_iota(idx, n, st);
      DevBuf keys_alt;
      keys_alt.reserve((n + kKeyPad) * sizeof(uint64_t), st);
      auto *idx_alt = static_cast<uint32_t *>(l_ialt.get(kWsIdxAlt, n * 4, st));
      void *sort_scratch = l_sort.get(kWsSort, radix_sort_scratch_bytes(n), st);
      int passes = 0;
      if (radix_sort_pairs(ix->keys.as<uint64_t>(), idx, keys_alt.as<uint64_t>(), idx_alt, n,
                           ix->g.total, sort_scratch, st, &passes, scalars_dev,
                           ix->scal.as<double>())) {
        std::swap(ix->keys.ptr, keys_alt.ptr);
        std::swap(ix->keys.bytes, keys_alt.bytes);
        std::swap(ix->keys.stream, keys_alt.stream);
      }
    }
    uint64_t ends[2];
    AMRX_CUDA(cudaMemcpyAsync(&ends[0], ix->keys.as<uint64_t>(), 8, cudaMemcpyDeviceToHost, st));
    AMRX_CUDA(cudaMemcpyAsync(&ends[1], ix->keys.as<uint64_t>() + n - 1, 8,
                              cudaMemcpyDeviceToHost, st));
    AMRX_CUDA(cudaStreamSynchronize(st));
    if (ends[0] < ix->key_lo || ends[1] >= ix->key_hi)
      fail(AMRX_ERR_INVALID_ARG, "keys outside the partition's key range");
    {
      // interior: a lookup of cell c has its major coordinate in
      // (m - 2 cw, m + cw] (m = c's, cw = the coarsest width: a stencil
      // point is one owner width away, then masked to a coarser level), so
      // cells two coarsest widths inside each end of the range only look
      // up keys in it (dist.halo_ranges builds ranges with that halo)
      const KeyGeom &g = ix->g;
      int msh = g.lbits;
      for (int a = 2; a >= 0; a--)
        if (g.bits[a]) msh = g.sh[a];
      const int coarsest = g.nlevels ? g.levels[g.nlevels - 1] : g.shift;
      const uint64_t hw = uint64_t(2) << (coarsest - g.shift);
      const uint64_t top = g.total >= 64 ? ~0ull : (uint64_t(1) << g.total);
      const uint64_t mlo = ix->key_lo >> msh, mhi = ix->key_hi >> msh;
      uint64_t q[2] = {ix->key_lo == 0 ? 0 : (mlo + hw) << msh,
                       ix->key_hi >= top ? ~0ull : (mhi > hw ? (mhi - hw) << msh : 0)};
      uint64_t pos[2];
      lower_bounds(ix->keys.as<uint64_t>(), n, q, 2, pos, st);
      ix->safe_lo = pos[0];
      ix->safe_hi = pos[1];
    }
    finalize_index(ix.get());
    AMRX_CUDA(cudaEventRecord(e1, st));
    AMRX_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    AMRX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const uint64_t eq2 = sorted_equal_pairs(ix.get());
    ensure_search_dir(ix.get(), eq2);
    finish_info(ix.get(), eq2, ms);
    *out = ix.release();
  });
}

amrx_status amrx_validate(amrx_index *index, uint32_t *dup_pairs, uint64_t dup_cap,
                          uint64_t *n_dup, uint32_t *overlap_pairs, uint64_t overlap_cap,
                          uint64_t *n_overlap)
{
  return guarded([&] {
    require_full(index);
    if (!index || !n_dup || !n_overlap) fail(AMRX_ERR_INVALID_ARG, "null argument");
    std::lock_guard<std::recursive_mutex> lock(index->mu);
    DeviceGuard dg(index->device);
    cudaStream_t st = index->stream;
    DevOut<uint32_t> dp(dup_pairs, dup_pairs ? 2 * dup_cap : 0, st);
    DevOut<uint32_t> op(overlap_pairs, overlap_pairs ? 2 * overlap_cap : 0, st);
    if (index->g.wide)
      wide_validate(index->wctx(), index->g, op.ptr, overlap_cap, n_overlap, dp.ptr, dup_cap,
                    n_dup, st);
    else
      run_validate(index->ctx(), index->g, op.ptr, overlap_cap, n_overlap, dp.ptr, dup_cap,
                   n_dup, st);
    if (dup_pairs && dp.staged && *n_dup)
      AMRX_CUDA(cudaMemcpyAsync(dup_pairs, dp.ptr, std::min(*n_dup, dup_cap) * 8,
                                cudaMemcpyDeviceToHost, st));
    if (overlap_pairs && op.staged && *n_overlap)
      AMRX_CUDA(cudaMemcpyAsync(overlap_pairs, op.ptr, std::min(*n_overlap, overlap_cap) * 8,
                                cudaMemcpyDeviceToHost, st));
    AMRX_CUDA(cudaStreamSynchronize(st));
    if ((dup_pairs && *n_dup > dup_cap) || (overlap_pairs && *n_overlap > overlap_cap))
      fail(AMRX_ERR_CAPACITY, "validate: " + std::to_string(*n_dup) + " duplicate and " +
                                std::to_string(*n_overlap) + " overlap pairs exceed the buffers");
  });
}

amrx_status amrx_release_cached_memory(int device)
{
  return guarded([&] {
    int dev = device;
    if (dev < 0) AMRX_CUDA(cudaGetDevice(&dev));
    DeviceGuard dg(dev);
    release_idle_memory(dev);
  });
}

amrx_status amrx_weld(const double *xyz9, uint64_t n_tris, double *verts3, uint64_t vcap,
                      uint32_t *tris3, uint64_t *n_verts, const amrx_index_opts *opts)
{
  return guarded([&] {
    NvtxRange nvtx("amrx weld");
    if (!n_verts) fail(AMRX_ERR_INVALID_ARG, "null argument");
    *n_verts = 0;
    if (n_tris == 0) return;
    if (!xyz9) fail(AMRX_ERR_INVALID_ARG, "null input array");
    if (n_tris > uint64_t(std::numeric_limits<uint32_t>::max()) / 3)
      fail(AMRX_ERR_LENGTH, "weld: too many triangles for 32-bit indices");
    int dev = opts && opts->device >= 0 ? opts->device : -1;
    if (dev < 0) AMRX_CUDA(cudaGetDevice(&dev));
    DeviceGuard dg(dev);
    enable_pool_caching(dev);
    cudaStream_t st = opts && opts->stream ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    DevIn<double> in(xyz9, n_tris * 9, st);
    DevOut<uint32_t> tris(tris3, tris3 ? n_tris * 3 : 0, st);
    // vertices: device output in place, else a device buffer of the bound
    const uint64_t vbound = std::min<uint64_t>(vcap, 3 * n_tris);
    DevOut<double> verts(verts3, verts3 ? vbound * 3 : 0, st);
    const uint64_t nv = run_weld(in.ptr, n_tris, verts.ptr, verts3 ? vbound : 0, tris.ptr, st);
    *n_verts = nv;
    if (verts3 && nv > vcap)
      fail(AMRX_ERR_CAPACITY, "vertex capacity " + std::to_string(vcap) + " < " +
                                std::to_string(nv) + " vertices");
    if (verts3 && verts.staged)
      AMRX_CUDA(cudaMemcpyAsync(verts3, verts.ptr, nv * 24, cudaMemcpyDeviceToHost, st));
    tris.finish(st);
    AMRX_CUDA(cudaStreamSynchronize(st));
  });
}

amrx_status amrx_index_destroy(amrx_index *index)
{
  return guarded([&] {
    if (!index) return;
    {
      DeviceGuard dg(index->device);
      if (index->stream) cudaStreamSynchronize(index->stream);
      index->keys.release();
      index->scal.release();
      index->dir.release();
      index->rec.release();
      index->order.release();
      index->scratch.release();
      index->out_a.release();
      index->out_b.release();
      index->mesh_v.release();
      index->mesh_t.release();
      cudaStreamSynchronize(index->stream);
      if (index->own_stream) cudaStreamDestroy(index->stream);
    }
    delete index;
  });
}

amrx_status amrx_index_get_info(const amrx_index *index, amrx_index_info *out)
{
  return guarded([&] {
    if (!index || !out) fail(AMRX_ERR_INVALID_ARG, "null argument");
    *out = index->info;
  });
}

amrx_status amrx_index_download(const amrx_index *cindex, int32_t *cells4,
                                double *scalars)
{
  return guarded([&] {
    auto *index = const_cast<amrx_index *>(cindex);
    if (!index) fail(AMRX_ERR_INVALID_ARG, "null index");
    DeviceGuard dg(index->device);
    cudaStream_t st = index->stream;
    if (cells4) {
      DevOut<int4> o(reinterpret_cast<int4 *>(cells4), index->n, st);
      if (index->g.wide)
        wide_unpack(index->keys.as<ulonglong2>(), index->n, index->g, o.ptr, st);
      else
        unpack_cells(index->keys.as<uint64_t>(), index->n, index->g, o.ptr, st);
      o.finish(st);
      AMRX_CUDA(cudaStreamSynchronize(st));
    }
    if (scalars)
      AMRX_CUDA(cudaMemcpyAsync(scalars, index->scal.ptr, index->n * sizeof(double),
                                cudaMemcpyDefault, st));
    AMRX_CUDA(cudaStreamSynchronize(st));
  });
}

amrx_status amrx_index_device_arrays(const amrx_index *index, void **keys,
                                     void **scalars)
{
  return guarded([&] {
    if (!index) fail(AMRX_ERR_INVALID_ARG, "null index");
    if (index->g.wide)
      fail(AMRX_ERR_UNSUPPORTED, "a two-word-key index has no packed 64-bit key array");
    if (keys) *keys = index->keys.ptr;
    if (scalars) *scalars = index->scal.ptr;
  });
}

amrx_status amrx_index_geometry(const amrx_index *index, int64_t *g16)
{
  return guarded([&] {
    if (!index || !g16) fail(AMRX_ERR_INVALID_ARG, "null argument");
    if (index->g.wide)
      fail(AMRX_ERR_UNSUPPORTED, "replicated / distributed indexes need keys of at most 64 bits");
    const KeyGeom &g = index->g;
    for (int a = 0; a < 3; a++) {
      g16[a] = g.mn[a];
      g16[3 + a] = g.mx[a];
      g16[6 + a] = index->bounds_hi[a];
    }
    g16[9] = g.level_mask;
    g16[10] = int64_t(index->n);
    g16[11] = int64_t(index->info.duplicate_keys);
    g16[12] = index->id_base;
    g16[13] = int64_t(index->key_lo);
    g16[14] = int64_t(index->key_hi);
    // key layout for partitioning: shift of the most significant coordinate
    // field present, finest level, coarsest level, key bits
    int major = g.lbits;
    for (int a = 2; a >= 0; a--)
      if (g.bits[a]) major = g.sh[a];
    const int coarsest = g.nlevels ? g.levels[g.nlevels - 1] : g.shift;
    g16[15] = int64_t(major) | (int64_t(g.shift) << 8) | (int64_t(coarsest) << 16) |
              (int64_t(g.total) << 24);
  });
}

amrx_status amrx_index_adopt(const void *keys_dev, const double *scalars_dev,
                             uint64_t n_cells, const int64_t *g16,
                             const amrx_index_opts *opts, amrx_index **out)
{
  return guarded([&] {
    if (!out || !keys_dev || !scalars_dev || !g16)
      fail(AMRX_ERR_INVALID_ARG, "null argument");
    if (n_cells == 0) fail(AMRX_ERR_LOAD, "dataset is empty");
    if (uint64_t(g16[10]) != n_cells)
      fail(AMRX_ERR_INVALID_ARG, "geometry describes a different cell count");
    auto ix = std::make_unique<amrx_index>();
    setup_stream(ix.get(), opts);
    cudaStream_t st = ix->stream;
    ix->n = n_cells;
    const int64_t mn[3] = {g16[0], g16[1], g16[2]};
    const int64_t mx[3] = {g16[3], g16[4], g16[5]};
    ix->g = make_geometry(mn, mx, uint32_t(g16[9]), n_cells, opts ? opts->flags : 0);
    if (ix->g.wide)
      fail(AMRX_ERR_UNSUPPORTED, "replicated indexes need keys of at most 64 bits");
    for (int a = 0; a < 3; a++) ix->bounds_hi[a] = g16[6 + a];
    cudaEvent_t e0, e1;
    AMRX_CUDA(cudaEventCreate(&e0));
    AMRX_CUDA(cudaEventCreate(&e1));
    AMRX_CUDA(cudaEventRecord(e0, st));
    ix->keys.reserve((n_cells + kKeyPad) * sizeof(uint64_t), st);
    ix->scal.reserve(n_cells * sizeof(double), st);
    AMRX_CUDA(cudaMemcpyAsync(ix->keys.ptr, keys_dev, n_cells * 8,
                              cudaMemcpyDefault, st));
    AMRX_CUDA(cudaMemcpyAsync(ix->scal.ptr, scalars_dev, n_cells * 8,
                              cudaMemcpyDefault, st));
    finalize_index(ix.get());
    AMRX_CUDA(cudaEventRecord(e1, st));
    AMRX_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    AMRX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    {
      const uint64_t eq = sorted_equal_pairs(ix.get());
      ensure_search_dir(ix.get(), eq);
      finish_info(ix.get(), eq, ms);
    }
    *out = ix.release();
  });
}

amrx_status amrx_find_exact(amrx_index *index, const int32_t *cells4,
                            uint64_t n, int64_t *out_ids)
{
  return guarded([&] {
    require_full(index);
    if (!index) fail(AMRX_ERR_INVALID_ARG, "null index");
    if (n == 0) return;
    DeviceGuard dg(index->device);
    cudaStream_t st = index->stream;
    DevIn<int4> in(reinterpret_cast<const int4 *>(cells4), n, st);
    DevOut<int64_t> o(out_ids, n, st);
    if (index->g.wide)
      wide_find_exact(index->wctx(), index->g, in.ptr, n, o.ptr, st);
    else
      run_find_exact(index->ctx(), index->g, in.ptr, n, o.ptr, st);
    o.finish(st);
    AMRX_CUDA(cudaStreamSynchronize(st));
  });
}

amrx_status amrx_snap(amrx_index *index, const int64_t *points3,
                      const int32_t *hints, int32_t hint_all, uint64_t n,
                      int64_t *out_ids)
{
  return guarded([&] {
    require_full(index);
    if (!index) fail(AMRX_ERR_INVALID_ARG, "null index");
    if (n == 0) return;
    DeviceGuard dg(index->device);
    cudaStream_t st = index->stream;
    DevIn<int64_t> p(points3, 3 * n, st);
    DevIn<int32_t> h(hints, hints ? n : 0, st);
    DevOut<int64_t> o(out_ids, n, st);
    if (index->g.wide)
      wide_snap(index->wctx(), index->g, p.ptr, h.ptr, hint_all, n, o.ptr, st);
    else
      run_snap(index->ctx(), index->g, p.ptr, h.ptr, hint_all, n, o.ptr, st);
    o.finish(st);
    AMRX_CUDA(cudaStreamSynchronize(st));
  });
}

amrx_status amrx_try_build_duals(amrx_index *index, const uint64_t *tasks,
                                 uint64_t n, uint8_t *out_reject,
                                 uint32_t *out_corners8)
{
  return guarded([&] {
    require_full(index);
    if (!index) fail(AMRX_ERR_INVALID_ARG, "null index");
    if (n == 0) return;
    DeviceGuard dg(index->device);
    cudaStream_t st = index->stream;
    DevIn<uint64_t> t(tasks, n, st);
    DevOut<uint8_t> r(out_reject, n, st);
    DevOut<uint32_t> c(out_corners8, out_corners8 ? 8 * n : 0, st);
    if (index->g.wide)
      wide_try_build(index->wctx(), index->g, t.ptr, n, r.ptr, c.ptr, st);
    else
      run_try_build(index->ctx(), index->g, t.ptr, n, r.ptr, c.ptr, st);
    r.finish(st);
    c.finish(st);
    AMRX_CUDA(cudaStreamSynchronize(st));
  });
}

amrx_status amrx_extract_dual(amrx_index *index, const amrx_range *range,
                              uint32_t *corners8, uint64_t *task_ids,
                              uint64_t cap, uint64_t *count, amrx_stats *stats)
{
  return guarded([&] {
    extract_dual_impl(index, range, corners8, task_ids, cap, count, stats, false);
  });
}

amrx_status amrx_extract_iso(amrx_index *index, const amrx_range *range,
                             const amrx_iso_params *params, void *xyz9,
                             uint64_t cap, uint64_t *count, amrx_stats *stats)
{
  return guarded([&] { extract_iso_impl(index, range, params, xyz9, cap, count, stats, false); });
}

amrx_status amrx_extract_dual_cells(amrx_index *index, const amrx_range *range, void *cells64,
                                    uint64_t cap, uint64_t *count, amrx_stats *stats)
{
  return guarded([&] {
    if (!index || !count) fail(AMRX_ERR_INVALID_ARG, "null argument");
    std::lock_guard<std::recursive_mutex> lock(index->mu);
    // the duals (corners + task ids) into the index's device arena
    extract_dual_impl(index, range, nullptr, nullptr, 0, count, stats, true);
    if (!cells64) return;  // count query
    if (*count > cap)
      fail(AMRX_ERR_CAPACITY, "output capacity " + std::to_string(cap) + " < " +
                                std::to_string(*count) + " duals");
    DeviceGuard dg(index->device);
    cudaStream_t st = index->stream;
    // converted and copied out in 1 GB chunks (two buffers, the copy of one
    // overlapping the conversion of the next)
    constexpr uint64_t kChunk = uint64_t(1) << 24;  // duals per chunk
    const uint64_t n = *count;
    DevBuf buf[2];
    for (uint64_t d0 = 0, k = 0; d0 < n; d0 += kChunk, k++) {
      const uint64_t m = std::min(kChunk, n - d0);
      DevBuf &b = buf[k & 1];
      b.reserve(m * 64, st);
      dual_cells(index->out_a.as<uint32_t>() + 8 * d0, index->out_b.as<uint64_t>() + d0, m,
                 index->keys.ptr, index->g, b.ptr, st);
      AMRX_CUDA(cudaMemcpyAsync(static_cast<char *>(cells64) + d0 * 64, b.ptr, m * 64,
                                cudaMemcpyDefault, st));
    }
    AMRX_CUDA(cudaStreamSynchronize(st));
  });
}

amrx_status amrx_extract_iso_mesh(amrx_index *index, const amrx_range *range,
                                  const amrx_iso_params *params, double *verts3, uint64_t vcap,
                                  uint32_t *tris3, uint64_t tcap, uint64_t *n_verts,
                                  uint64_t *n_tris, double *seconds_weld, amrx_stats *stats)
{
  return guarded([&] {
    if (!index || !params || !n_verts || !n_tris) fail(AMRX_ERR_INVALID_ARG, "null argument");
    if (params->xyz_is_f32)
      fail(AMRX_ERR_INVALID_ARG, "the welded mesh is built from the FP64 soup (xyz_is_f32 = 0)");
    std::lock_guard<std::recursive_mutex> lock(index->mu);
    // the soup into the index's device arena (or the cached one)
    uint64_t count = 0;
    extract_iso_impl(index, range, params, nullptr, 0, &count, stats, true);
    DeviceGuard dg(index->device);
    cudaStream_t st = index->stream;
    if (!index->mesh_valid) {
      NvtxRange nvtx("amrx weld (extract_isosurface)");
      const auto t0 = std::chrono::steady_clock::now();
      index->mesh_t.reserve(count * 12 + 16, st);
      index->mesh_v.reserve(count * 72 + 16, st);  // at most 3 vertices per triangle
      index->mesh_nv = count ? run_weld(index->out_a.as<double>(), count,
                                        index->mesh_v.as<double>(), 3 * count,
                                        index->mesh_t.as<uint32_t>(), st)
                             : 0;
      AMRX_CUDA(cudaStreamSynchronize(st));
      index->mesh_weld_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      index->mesh_valid = true;
    }
    *n_verts = index->mesh_nv;
    *n_tris = count;
    if (seconds_weld) *seconds_weld = index->mesh_weld_s;
    if (!verts3 && !tris3) return;  // count query
    if ((verts3 && vcap < index->mesh_nv) || (tris3 && tcap < count))
      fail(AMRX_ERR_CAPACITY, "mesh capacity (" + std::to_string(vcap) + " vertices, " +
                                std::to_string(tcap) + " triangles) < " +
                                std::to_string(index->mesh_nv) + " vertices, " +
                                std::to_string(count) + " triangles");
    if (verts3 && index->mesh_nv)
      AMRX_CUDA(cudaMemcpyAsync(verts3, index->mesh_v.ptr, index->mesh_nv * 24,
                                cudaMemcpyDefault, st));
    if (tris3 && count)
      AMRX_CUDA(cudaMemcpyAsync(tris3, index->mesh_t.ptr, count * 12, cudaMemcpyDefault, st));
    AMRX_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"

namespace amrx {
/// the writers (writers.cpp) report through the same thread-local message
void set_last_error(const std::string &msg, bool clear)
{
  if (clear)
    g_last_error.clear();
  else
    g_last_error = msg;
}
}  // namespace amrx
