// Host-side interfaces shared between the amrx translation units.
#pragma once

#include <cstdint>
#include <atomic>
#include <stdexcept>
#include <string>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace amrx {

/// a failure with its amrx_status code, turned into the return value (and
/// the thread's amrx_last_error text) at the C ABI
struct ApiError : std::runtime_error {
  int code;
  ApiError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string &msg) { throw ApiError(code, msg); }

/// checked builds: the OR of every translation unit's check word, cleared
unsigned int check_word_extract();
unsigned int check_word_sort();
unsigned int check_word_wide();
unsigned int check_word_ingest();
unsigned int check_word_validate();
unsigned int check_word_weld();

/// the thread-local amrx_last_error text (api.cu)
void set_last_error(const std::string &msg, bool clear);

[[noreturn]] void throw_cuda(cudaError_t e, const char *what, const char *file,
                             int line);

#define AMRX_CUDA(call)                                                  \
  do {                                                                   \
    const cudaError_t amrx_e_ = (call);                                  \
    if (amrx_e_ != cudaSuccess)                                          \
      ::amrx::throw_cuda(amrx_e_, #call, __FILE__, __LINE__);            \
  } while (0)

void note_launch();

/// an NVTX range for the duration of a scope (header-only NVTX3: a no-op
/// unless a profiler injects itself), naming the library's phases in
/// nsys / ncu timelines
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

/// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
void ensure_smem_attr(const void *kernel, size_t bytes);

#define AMRX_LAUNCH_CHECK()                                              \
  do {                                                                   \
    ::amrx::note_launch();                                               \
    AMRX_CUDA(cudaGetLastError());                                       \
  } while (0)

/*! device allocation with RAII, grows on demand.  Memory comes from the
    device's stream-ordered pool (cudaMallocAsync) whose release threshold is
    raised at index creation, so a buffer freed by one step is handed to the
    next step's allocation without touching the driver. */
struct DevBuf {
  void *ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  ~DevBuf();
  void reserve(size_t n, cudaStream_t st = nullptr);  // contents not kept
  void release();
  template <typename T> T *as() const { return static_cast<T *>(ptr); }
};

/// keep pool memory cached across frees on this device (idempotent)
void enable_pool_caching(int device);

/*! Per-device workspace: the large temporaries of ingest and extraction
    (staged inputs, sort ping-pong buffers, output staging arenas) live in
    process-wide slots that only grow, so a pipeline that builds and drops
    an index per batch allocates nothing in steady state.  A lease holds a
    slot exclusively until it is destroyed; if the slot is busy (another
    thread) the lease falls back to a private allocation. */
enum WsSlot {
  kWsCells, kWsScal, kWsIdx, kWsKeysAlt, kWsIdxAlt, kWsSort, kWsStageA,
  kWsStageB, kWsTiles, kWsBits, kWsCtl, kWsScratch, kWsOutA, kWsOutB, kWsJobs, kWsCount
};

struct WsLease {
  void *ptr = nullptr;
  size_t bytes = 0;
  WsLease() = default;
  WsLease(const WsLease &) = delete;
  WsLease &operator=(const WsLease &) = delete;
  ~WsLease();
  /// at least `bytes` from slot `slot` of the current device (contents not kept)
  void *get(int slot, size_t bytes, cudaStream_t st);
  template <typename T> T *as() const { return static_cast<T *>(ptr); }

 private:
  int device_ = -1, slot_ = -1;
  DevBuf own_;  // fallback when the shared slot is busy
};

/// a workspace lease with DevBuf's reserve/as surface
struct WsBuf {
  WsLease lease;
  int slot;
  void *ptr = nullptr;
  explicit WsBuf(int s) : slot(s) {}
  void reserve(size_t n, cudaStream_t st) { ptr = lease.get(slot, n, st); }
  template <typename T> T *as() const { return static_cast<T *>(ptr); }
};

/// the temporaries of one extraction, all from the device workspace
struct ExtractScratch {
  WsBuf ctl{kWsCtl}, tiles{kWsTiles}, stage_a{kWsStageA}, stage_b{kWsStageB},
    bits{kWsBits}, jobs{kWsJobs};
  DevBuf scan;  // unused by the pool-free scan; kept for its signature
};

// ------------------------------------------------------------ ingest.cu
struct PrepassResult {
  uint64_t first_bad;   // UINT64_MAX if every record is valid
  int32_t mn[3], mx[3];
  int64_t hi[3];        // max anchor + width per axis
  uint32_t level_mask;
};

/// validation + bounds + level mask over n input records (device pointer)
PrepassResult ingest_prepass(const int4 *cells, uint64_t n, DevBuf &scratch,
                             cudaStream_t st);

/// radix digits of the sort (sort.cu) -- also the layout of the digit
/// histograms ingest_pack can produce for it
constexpr int kSortRadixBits = 9;
constexpr int kSortDigits = 1 << kSortRadixBits;
constexpr int kSortMaxPasses = 8;

/// occupancy records are built per tile of 2^kRecTileLog buckets; a
/// partition's first bucket is a multiple of the tile
#ifndef AMRX_REC_TILE_LOG
#define AMRX_REC_TILE_LOG 12
#endif
constexpr int kRecTileLog = AMRX_REC_TILE_LOG;

/// key = pack(cell), idx = position (idx may be null).  With hist (device,
/// kSortMaxPasses x kSortDigits u32, zeroed here) the same pass counts the
/// sort's digits of the first `passes` digits, and order2 (device, 2 u64,
/// zeroed here) receives the keys' descents and equal neighbours
void ingest_pack(const int4 *cells, uint64_t n, const KeyGeom &g,
                 uint64_t *keys, uint32_t *idx, cudaStream_t st,
                 unsigned int *hist = nullptr, int passes = 0,
                 unsigned long long *order2 = nullptr);

/// number of i with key[i] > key[i+1] (0 = already sorted), and equal pairs
void ingest_order_check(const uint64_t *keys, uint64_t n, DevBuf &scratch,
                        uint64_t *descents, uint64_t *equal_pairs,
                        cudaStream_t st);

void gather_f64(const uint32_t *perm, const double *in, double *out,
                uint64_t n, cudaStream_t st);

/// p[i] = i for i in [0, n)
void fill_iota(uint32_t *p, uint64_t n, cudaStream_t st);
/// n AMRCELL1 records (24 B each, 8-byte aligned) -> cells[first..] and
/// scal[first..]; atomicMin(*bad) with the first non-finite scalar's record
void split_records(const void *rec, uint64_t n, uint64_t first, int4 *cells, double *scal,
                   unsigned long long *bad, cudaStream_t st);

/// fill kKeyPad sentinels (all ones) after the n sorted keys
void pad_keys(uint64_t *keys, uint64_t n, cudaStream_t st);

/// dir[b] = first position whose key >> g.dir_shift >= b, b in [0, 2^D];
/// or, with rec (g.occ geometry) instead, the occupancy records (dir
/// unused): rec[b - rec_lo] for buckets b in [rec_lo, rec_lo + rec_n] (all
/// 2^D + 1 when rec_n = 0; rec_lo a multiple of 4096, no key below it);
/// order2 (device, 2 x u64) receives the keys' descents and equal pairs
void build_directory(const uint64_t *keys, uint64_t n, const KeyGeom &g,
                     uint32_t *dir, uint2 *rec, unsigned long long *order2,
                     DevBuf &scratch, cudaStream_t st, uint64_t rec_lo = 0,
                     uint64_t rec_n = 0, const uint32_t *tile_starts = nullptr);

/// the record tiles' first key positions, found by the sort's last pass
/// (dense records of a whole index): starts[t] = first position whose key
/// >> shift >> kRecTileLog >= t, t in [0, tiles]; filled by the sort
struct TileStarts {
  uint32_t *starts = nullptr;  // tiles + 1 entries (device)
  int shift = 0;
  uint64_t tiles = 0;
  bool filled = false;
};

/// hashed records: distinct buckets of the sorted keys (synchronises);
/// order2 (device, 2 x u64) receives the keys' descents and equal pairs
uint64_t hash_count(const uint64_t *keys, uint64_t n, const KeyGeom &g,
                    unsigned long long *order2, DevBuf &scratch, cudaStream_t st);
/// fill the table of `buckets` (a power of two) 32-byte table buckets, two
/// entries each; *max_probe (device) = the longest displacement (buckets)
void build_hash(const uint64_t *keys, uint64_t n, const KeyGeom &g, ulonglong4 *tab,
                uint64_t buckets, unsigned int *max_probe, cudaStream_t st);

/// lower_bound of nq host keys q in the sorted device keys -> host out (synchronises)
void lower_bounds(const uint64_t *keys, uint64_t n, const uint64_t *q, int nq, uint64_t *out,
                  cudaStream_t st);

/// 64-byte DualCell records (dual.hpp:30-35) of n duals into out (device)
void dual_cells(const uint32_t *corners, const uint64_t *tasks, uint64_t n, const void *keys,
                const KeyGeom &g, void *out, cudaStream_t st);

/// unpack sorted keys into 4 x int32 cells
void unpack_cells(const uint64_t *keys, uint64_t n, const KeyGeom &g,
                  int4 *cells, cudaStream_t st);

/// exclusive scan of n u32 values (in place allowed); returns launches
int scan_exclusive_u32(const uint32_t *in, uint32_t *out, uint64_t n,
                       DevBuf &scratch, cudaStream_t st);

/// exclusive scan of n u32 counts into u64 offsets; returns launches
int scan_exclusive_u32_u64(const uint32_t *in, uint64_t *out, uint64_t n,
                           DevBuf &scratch, cudaStream_t st);

// -------------------------------------------------------------- sort.cu
/// stable LSD radix sort of (keys, vals) over bits [0, key_bits), ping-
/// ponging with the alt buffers; returns true when the sorted keys (and,
/// without gsrc, values) ended in the alt buffers.  With gsrc, the last
/// pass writes gdst[i] = gsrc[value of sorted item i] instead of the
/// values (after gsrc_ready, if set).  With rank_out instead, the last
/// pass writes the inverse permutation (rank[input position] = sorted
/// position) and *rank_out points at it (null if no pass ran: identity)
bool radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_alt,
                      uint32_t *vals_alt, uint64_t n, int key_bits,
                      void *scratch, cudaStream_t st, int *passes_run,
                      const double *gsrc = nullptr, double *gdst = nullptr,
                      cudaEvent_t gsrc_ready = nullptr, uint32_t **rank_out = nullptr,
                      const unsigned int *hist_in = nullptr, TileStarts *ts = nullptr);

/// radix_sort_pairs with a 64-bit payload that enters from vals_src (read
/// by the first pass only: e.g. the caller's scalars in input order) and
/// ping-pongs between vals and vals_alt; true when keys and values ended in
/// the alt buffers
bool radix_sort_pairs_u64(uint64_t *keys, const uint64_t *vals_src, uint64_t *vals,
                          uint64_t *keys_alt, uint64_t *vals_alt, uint64_t n, int key_bits,
                          void *scratch, cudaStream_t st, int *passes_run,
                          const unsigned int *hist_in = nullptr, TileStarts *ts = nullptr);

/// out[rank[i]] = in[i] for i in [0, n) (a payload chunk into key order)
void scatter_f64(const uint32_t *rank, const double *in, double *out, uint64_t n,
                 cudaStream_t st);

/// bytes of scratch radix_sort_pairs needs for n keys
size_t radix_sort_scratch_bytes(uint64_t n);

// ----------------------------------------------------------- extract.cu
struct ExtractRequest {
  SearchCtx s;
  KeyGeom g;
  const double *scal;
  uint64_t cell_begin, cell_end;
  bool emit_dual;
  bool emit_tri;
  bool tri_f32;
  double iso;
  // outputs: device memory, or pinned host memory (final_host) filled by
  // one bulk copy per round; at most dual_cap / tri_cap items are written
  uint32_t *corners;    // [dual_cap][8] or null
  uint64_t *tasks;      // [dual_cap] or null
  uint64_t dual_cap;
  void *xyz;            // [tri_cap][9] f64/f32 or null
  uint64_t tri_cap;
  bool final_host;
  bool unique;          // the index holds no duplicate keys
  // growable device outputs (an index's cached arena): when set, the
  // pointers above are ignored and these grow to hold the whole result
  DevBuf *grow_a = nullptr;  // corners (dual) or xyz (iso)
  DevBuf *grow_b = nullptr;  // tasks (dual)
  // host output: small first rounds (1/64, 1/32 of the tiles) so the
  // first download overlaps the rest of the extraction
  bool stream_rounds = false;
};

struct ExtractResult {
  uint64_t counters[4];  // accepted, missing, finer, lower_key
  uint64_t duals;        // emitted by the scan (== accepted)
  uint64_t tris_counted; // count phase
  uint64_t tris_written; // emit phase
  uint32_t error_flags;  // bit0 collapsed edge, bit1 undecided candidate
  float ms;              // device time of the extraction kernels (all rounds)
  float ms2;             // device time of scan + reorder into final order
  uint64_t launches;
  uint32_t rounds;       // staging rounds the call took
};

ExtractResult run_extract(const ExtractRequest &r, cudaStream_t st);

// ------------------------------------------------------------- wide.cu
struct WideCtx;
/// the extraction for wide (> 64-bit) keys: two counted passes (extract.cu)
ExtractResult run_extract_wide(const ExtractRequest &r, const WideCtx &w, cudaStream_t st);

struct WideBuild {
  uint64_t equal_pairs;  // adjacent equal keys
  uint64_t entries;      // exact-key table entries
  uint32_t max_probe;
  int passes;            // radix passes run
};
/// build_index for wide keys: pack, two stable radix sorts (lo, then hi
/// word), keys + scalars in sorted order, the exact-key table (synchronises)
WideBuild wide_build(const int4 *cells, const double *scal, uint64_t n, const KeyGeom &g,
                     ulonglong2 *keys, double *scal_out, DevBuf &table, cudaStream_t st);
void wide_unpack(const ulonglong2 *keys, uint64_t n, const KeyGeom &g, int4 *cells,
                 cudaStream_t st);
void wide_find_exact(const WideCtx &w, const KeyGeom &g, const int4 *cells, uint64_t n,
                     int64_t *out, cudaStream_t st);
void wide_snap(const WideCtx &w, const KeyGeom &g, const int64_t *points, const int32_t *hints,
               int32_t hint_all, uint64_t n, int64_t *out, cudaStream_t st);
void wide_try_build(const WideCtx &w, const KeyGeom &g, const uint64_t *tasks, uint64_t n,
                    uint8_t *reject, uint32_t *corners, cudaStream_t st);
void wide_validate(const WideCtx &w, const KeyGeom &g, uint32_t *ovl_pairs, uint64_t ovl_cap,
                   uint64_t *n_ovl, uint32_t *dup_pairs, uint64_t dup_cap, uint64_t *n_dup,
                   cudaStream_t st);

/// amrx_debug_round_limit: cap on every round's staging items (0 = default)
extern std::atomic<uint64_t> g_round_limit;

void run_find_exact(const SearchCtx &s, const KeyGeom &g, const int4 *cells,
                    uint64_t n, int64_t *out, cudaStream_t st);
void run_snap(const SearchCtx &s, const KeyGeom &g, const int64_t *points,
              const int32_t *hints, int32_t hint_all, uint64_t n,
              int64_t *out, cudaStream_t st);
void run_try_build(const SearchCtx &s, const KeyGeom &g, const uint64_t *tasks,
                   uint64_t n, uint8_t *reject, uint32_t *corners,
                   cudaStream_t st);

int device_sm_count();

// --------------------------------------------------------- validate.cu
/// validate_dataset: overlap / duplicate pairs (2 x u32 each, global ids)
/// into the buffers (device, may be null) up to their capacities; the
/// counts are returned either way
void run_validate(const SearchCtx &s, const KeyGeom &g, uint32_t *ovl_pairs, uint64_t ovl_cap,
                  uint64_t *n_ovl, uint32_t *dup_pairs, uint64_t dup_cap, uint64_t *n_dup,
                  cudaStream_t st);

// ------------------------------------------------------------- weld.cu
/// weld n_tris fat triangles (device xyz9); verts (vcap) / tris (3 per
/// triangle) may be null; returns the vertex count
uint64_t run_weld(const double *xyz9, uint64_t n_tris, double *verts, uint64_t vcap,
                  uint32_t *tris, cudaStream_t st);

}  // namespace amrx
