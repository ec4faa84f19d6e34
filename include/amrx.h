/* amrx -- B200-native dual-mesh / iso-surface extraction for structured AMR.
 *
 * The C ABI every host binding goes through (the C++ drop-in shim in
 * paper_2004_08475_b200/shim/, the Python host mirror over ctypes, and any
 * FFI a maintainer adds).  Plain pointers and sizes only.
 *
 * Which reference interface each entry point replaces (paths relative to the
 * reference checkout, /root/reference/):
 *
 *   amrx_index_create     build_index(vector<CellCoord>, vector<double>)
 *                         proj/include/amriso/locator.hpp:52-53,
 *                         proj/src/locator.cpp:26-92
 *   amrx_index_download   CellIndex.data.{cells,scalars} / .levels / bounds
 *                         proj/include/amriso/locator.hpp:38-45,
 *                         proj/include/amriso/core.hpp:143-148
 *   amrx_find_exact       find_exact   proj/src/locator.cpp:94-101
 *   amrx_snap             snap         proj/src/locator.cpp:122-134
 *   amrx_try_build_duals  try_build_dual (batched) proj/src/dual.cpp:41-72
 *   amrx_extract_dual     extract_dual_mesh  proj/include/amriso/pipeline.hpp:70-71,
 *                         proj/src/pipeline.cpp:160-194
 *   amrx_extract_iso      extract_isosurface passes 1+2 (the fat soup, before
 *                         weld) proj/include/amriso/pipeline.hpp:65-66,
 *                         proj/src/pipeline.cpp:67-146
 *   amrx_stats            ExtractionStats proj/include/amriso/pipeline.hpp:29-49
 *   amrx_status codes     LoadError / invalid_argument / length_error /
 *                         logic_error (core.hpp:62-74, locator.cpp:29-50,
 *                         pipeline.cpp:70-71,116-118)
 *
 * Memory: every pointer argument may be host memory (pageable or pinned) or
 * CUDA device memory on the index's device; the library detects which with
 * cudaPointerGetAttributes and copies as needed.  Calls are synchronous with
 * respect to the host (they run on the index's stream and synchronise it
 * before returning).  Output order is the reference's candidate order
 * (owning cell major, delta minor, table order within a hex), independent of
 * launch configuration and of the multi-GPU partition.
 */
#ifndef AMRX_H
#define AMRX_H

#include <stdint.h>

#if defined(__GNUC__)
#define AMRX_API __attribute__((visibility("default")))
#else
#define AMRX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum amrx_status {
  AMRX_OK = 0,
  AMRX_ERR_LOAD = 1,          /* malformed input -> LoadError ("record n: ...") */
  AMRX_ERR_INVALID_ARG = 2,   /* empty dataset / bad argument -> invalid_argument */
  AMRX_ERR_LENGTH = 3,        /* output too large for 32-bit indices -> length_error */
  AMRX_ERR_INTERNAL = 4,      /* internal consistency check failed -> logic_error */
  AMRX_ERR_CUDA = 5,          /* CUDA runtime failure (message names the call) */
  AMRX_ERR_CAPACITY = 6,      /* caller buffer too small; *count holds the need */
  AMRX_ERR_UNSUPPORTED = 7,   /* dataset outside this build's limits */
  AMRX_ERR_NO_DEVICE = 8,     /* no CUDA device / kernel image for this GPU */
  AMRX_ERR_IO = 9,            /* file could not be written -> runtime_error */
  AMRX_ERR_NCCL = 10          /* NCCL missing or a collective failed (amrx_comm_*) */
} amrx_status;

typedef struct amrx_index amrx_index;

/* index construction options (NULL = defaults) */
typedef struct amrx_index_opts {
  int device;        /* CUDA device ordinal; -1 = current device */
  void *stream;      /* cudaStream_t to run on; NULL = library-owned stream */
  uint32_t flags;    /* AMRX_FLAG_* */
} amrx_index_opts;

/* input is already in (i,j,k,level) order with stable ties (e.g. the arrays
 * of an existing CellIndex): the library verifies this on the device and
 * skips the radix sort */
#define AMRX_FLAG_PRESORTED 0x1u

/* lookup structure of the index (default: chosen from the key space).  The
 * reference's find_exact/snap are a binary search over the sorted cells
 * (locator.cpp:94-134); the device index answers the same queries through
 *   RECORDS    a 32-value occupancy record per bucket of the key space:
 *              one 8-byte load + popcount per lookup (dense key spaces)
 *   HASH       records of the occupied buckets only, open-addressed
 *              (sparse or deep key spaces, any key width)
 *   DIRECTORY  a bucket directory + binary search of the bucket
 * An index with duplicate cells always uses the directory (a record's
 * popcount cannot count equal keys).  The results are identical. */
#define AMRX_FLAG_LOOKUP_RECORDS 0x2u
#define AMRX_FLAG_LOOKUP_HASH 0x4u
#define AMRX_FLAG_LOOKUP_DIRECTORY 0x8u

/* amrx_index_info.lookup */
#define AMRX_LOOKUP_DIRECTORY 0
#define AMRX_LOOKUP_RECORDS 1
#define AMRX_LOOKUP_HASH 2
#define AMRX_LOOKUP_WIDE 3  /* > 64-bit keys: exact-key table, per-level probes */

typedef struct amrx_index_info {
  uint64_t cell_count;
  int32_t max_level;
  int32_t level_count;
  int32_t levels[31];       /* distinct levels present, finest first */
  int64_t bounds_lo[3];     /* hull of all cell boxes (locator.cpp:70-83) */
  int64_t bounds_hi[3];
  int32_t key_bits;         /* bits of the packed sort key in use (> 64: two-word keys) */
  int32_t directory_bits;   /* log2 of the lookup structure's entry count */
  uint64_t duplicate_keys;  /* adjacent equal keys after the sort */
  uint64_t device_bytes;    /* HBM held by the index */
  double seconds_ingest;    /* device time of pack + sort + gather + directory */
  int32_t lookup;           /* AMRX_LOOKUP_* in use */
  uint32_t max_probe;       /* HASH: longest displacement from a home slot */
  uint64_t lookup_entries;  /* records / hash slots / directory entries */
} amrx_index_info;

typedef struct amrx_stats {
  uint64_t cell_count;
  uint64_t duals_accepted;
  uint64_t duals_missing_corner;
  uint64_t duals_finer_corner;
  uint64_t duals_lower_key_corner;
  uint64_t pass1_triangle_count;  /* counted before the emit pass */
  uint64_t fat_triangle_count;    /* written by the emit pass */
  uint64_t dual_count;            /* duals emitted (== duals_accepted) */
  double seconds_pass1;           /* device time, search + count phase */
  double seconds_pass2;           /* device time, emit phase (fused: 0) */
  uint64_t kernel_launches;       /* kernels this call launched */
} amrx_stats;

/* Build a device index: pack (i,j,k,level) into 64-bit keys, radix-sort
 * them with the input position as a stable tie-break, gather the scalars,
 * build the search directory.  Errors mirror build_index: empty input,
 * length mismatch, > 2^32-1 cells, level outside [0,30], misaligned anchor
 * (message names "record n" like locator.cpp:37-49). */
AMRX_API amrx_status amrx_index_create(const int32_t *cells4, const double *scalars,
                              uint64_t n_cells, uint64_t n_scalars,
                              const amrx_index_opts *opts, amrx_index **out);

/* read_amr (proj/src/io.cpp:178-181, io.hpp:43): an AMRCELL1 file (binary,
 * 24-byte header + 24-byte records, io.cpp:76-126) or, for a ".txt" path,
 * the text form (io.cpp:128-176) -> a device index.  Binary records stream
 * through pinned chunks into device memory (no host copy of the dataset).
 * Errors are AMRX_ERR_LOAD with the reference's messages, prefixed with the
 * path ("<path>: record 1: scalar is not finite", "<path>: truncated: ..."). */
AMRX_API amrx_status amrx_read_amr(const char *path, const amrx_index_opts *opts,
                                   amrx_index **out);

AMRX_API amrx_status amrx_index_destroy(amrx_index *index);

AMRX_API amrx_status amrx_index_get_info(const amrx_index *index, amrx_index_info *out);

/* the sorted cells (4 x int32 each) and scalars; either pointer may be NULL */
AMRX_API amrx_status amrx_index_download(const amrx_index *index, int32_t *cells4,
                                double *scalars);

/* device pointers of the sorted packed keys (u64) and scalars (f64) --
 * what the multi-GPU path broadcasts */
AMRX_API amrx_status amrx_index_device_arrays(const amrx_index *index, void **keys,
                                     void **scalars);

/* Adopt already-sorted packed keys + scalars (e.g. received by NCCL
 * broadcast) with the geometry of a source index: no sort, directory only.
 * geometry: the 16 int64 words from amrx_index_geometry(). */
AMRX_API amrx_status amrx_index_geometry(const amrx_index *index, int64_t *geometry16);
AMRX_API amrx_status amrx_index_adopt(const void *keys_dev, const double *scalars_dev,
                             uint64_t n_cells, const int64_t *geometry16,
                             const amrx_index_opts *opts, amrx_index **out);

/* ---- distributed build (dist.py): every rank holds a slice of the cell
 * list; the global geometry is agreed first, each rank sorts its slice, the
 * sorted runs are exchanged by key range (plus a halo), and each rank
 * indexes the key range it received.  No reference counterpart: the
 * reference is single-process. */

/* bounds of n records: mn[3] (min anchor), mx[3] (max anchor), hi[3]
 * (max anchor + width), level mask -- to be reduced across ranks into the
 * global geometry words 0-9 of amrx_index_geometry's layout */
AMRX_API amrx_status amrx_bounds(const int32_t *cells4, uint64_t n_cells,
                                 const amrx_index_opts *opts, int64_t *bounds10);

/* sort a slice under the global geometry (words 0-10 of geometry16; word 10
 * = global cell count): sorted packed keys + scalars only, no search
 * structure (amrx_index_device_arrays reads them) */
AMRX_API amrx_status amrx_index_sort_part(const int32_t *cells4, const double *scalars,
                                          uint64_t n_cells, const int64_t *geometry16,
                                          const amrx_index_opts *opts, amrx_index **out);

/* index a partition: packed keys (any order; sorted here) + scalars on this
 * device, all inside the key range [geometry16[13], geometry16[14]); word
 * 12 = global CellId of the partition's first key.  Every id it reports is
 * global.  Needs unique cells and the occupancy-record geometry. */
AMRX_API amrx_status amrx_index_from_keys(const void *keys_dev, const double *scalars_dev,
                                          uint64_t n_cells, const int64_t *geometry16,
                                          const amrx_index_opts *opts, amrx_index **out);

/* find_exact for n cells (4 x int32 each): out_ids = CellId or -1 */
AMRX_API amrx_status amrx_find_exact(amrx_index *index, const int32_t *cells4,
                            uint64_t n, int64_t *out_ids);

/* snap for n points (3 x int64 each), one hint level per point (or a single
 * hint if hints == NULL: *hint_all) */
AMRX_API amrx_status amrx_snap(amrx_index *index, const int64_t *points3,
                      const int32_t *hints, int32_t hint_all, uint64_t n,
                      int64_t *out_ids);

/* try_build_dual for n candidates given as task ids (cell*8 + delta):
 * reject codes (0 accepted, 1 missing, 2 finer, 3 lower key) and, when
 * accepted, the 8 corner CellIds */
AMRX_API amrx_status amrx_try_build_duals(amrx_index *index, const uint64_t *tasks,
                                 uint64_t n, uint8_t *out_reject,
                                 uint32_t *out_corners8);

/* Cell range [cell_begin, cell_end) of the candidate order; {0, UINT64_MAX}
 * = all cells.  Used by the multi-GPU range partition. */
typedef struct amrx_range {
  uint64_t cell_begin;
  uint64_t cell_end;
} amrx_range;

/* extract_dual_mesh: the accepted duals in candidate order.  corners8 gets
 * 8 CellIds per dual; task_ids (optional) gets owner*8+delta, from which
 * DualCell.{owner,base,level} follow (dual.hpp:61-67).  If the caller's cap
 * is too small returns AMRX_ERR_CAPACITY with *count = the total. */
AMRX_API amrx_status amrx_extract_dual(amrx_index *index, const amrx_range *range,
                              uint32_t *corners8, uint64_t *task_ids,
                              uint64_t cap, uint64_t *count,
                              amrx_stats *stats);

/* extract_isosurface passes 1+2: the fat triangle soup (9 coordinates per
 * triangle, FP64 bit-exact with the reference; xyz_is_f32 = 1 rounds the
 * FP64 results to float after the FP64 sliver test).  Also fills the dual
 * counters.  AMRX_ERR_CAPACITY as above; AMRX_ERR_LENGTH when the total
 * exceeds UINT32_MAX/3 (pipeline.cpp:116-118) and check_length is set. */
typedef struct amrx_iso_params {
  double iso;
  int32_t xyz_is_f32;
  int32_t check_length;
} amrx_iso_params;

AMRX_API amrx_status amrx_extract_iso(amrx_index *index, const amrx_range *range,
                             const amrx_iso_params *params, void *xyz9,
                             uint64_t cap, uint64_t *count,
                             amrx_stats *stats);

/* extract_dual_mesh as the reference returns it (pipeline.cpp:160-194):
 * 64-byte DualCell records (dual.hpp:30-35: 8 corner CellIds, the query base
 * dual_base_of(owner, delta) as 3 x int64, the owner's level, the owner) in
 * candidate order, built on the device.  cells64 NULL = count query (the
 * duals stay on the device for the copy call). */
AMRX_API amrx_status amrx_extract_dual_cells(amrx_index *index, const amrx_range *range,
                                             void *cells64, uint64_t cap, uint64_t *count,
                                             amrx_stats *stats);

/* extract_isosurface as the reference returns it (pipeline.cpp:67-158):
 * passes 1+2 and the weld (weld.cpp:31-64) on the device, only the indexed
 * mesh crosses to the caller -- verts3 (3 f64 per vertex, position-sorted
 * like the reference) and tris3 (3 u32 per triangle, candidate order).  Both
 * NULL = count query (*n_verts, *n_tris; the mesh stays on the device for
 * the copy call).  *seconds_weld = host time of the weld.  FP64 only. */
AMRX_API amrx_status amrx_extract_iso_mesh(amrx_index *index, const amrx_range *range,
                                           const amrx_iso_params *params, double *verts3,
                                           uint64_t vcap, uint32_t *tris3, uint64_t tcap,
                                           uint64_t *n_verts, uint64_t *n_tris,
                                           double *seconds_weld, amrx_stats *stats);

/* validate_dataset (proj/src/locator.cpp:136-161): duplicate pairs (n,
 * n+1) of equal adjacent cells and overlap pairs (n, coarser cell holding
 * cell n's anchor), 2 x uint32 CellIds each, in the reference's order.
 * Either buffer may be NULL (count only); AMRX_ERR_CAPACITY when a cap is
 * too small (the counts are still set). */
AMRX_API amrx_status amrx_validate(amrx_index *index, uint32_t *dup_pairs, uint64_t dup_cap,
                                   uint64_t *n_dup, uint32_t *overlap_pairs,
                                   uint64_t overlap_cap, uint64_t *n_overlap);

/* weld (proj/src/weld.cpp:31-64, replaces amriso::weld): merge bitwise-
 * identical corner positions of n_tris fat triangles (9 FP64 each, host or
 * device) into shared vertices, position-sorted like the reference.
 * verts3 gets 3 FP64 per vertex (capacity vcap vertices; vcap = 3 * n_tris
 * always suffices), tris3 3 vertex ids per triangle; *n_verts the vertex
 * count.  AMRX_ERR_LENGTH when n_tris > UINT32_MAX/3 (weld.cpp:36-37);
 * AMRX_ERR_CAPACITY when vcap is too small (*n_verts = the need). */
AMRX_API amrx_status amrx_weld(const double *xyz9, uint64_t n_tris, double *verts3,
                               uint64_t vcap, uint32_t *tris3, uint64_t *n_verts,
                               const amrx_index_opts *opts);

/* give back the device memory the library keeps cached between calls (idle
 * workspace buffers, the stream-ordered pool's free blocks) on `device`
 * (-1 = current); indexes stay valid */
AMRX_API amrx_status amrx_release_cached_memory(int device);

/* Writers (proj/src/io.cpp:212-305): write_obj (obj_string, shortest
 * round-trip decimals, 1-based faces), write_ply (binary little-endian,
 * float32 positions, uchar 3 + uint32 x3 faces) and write_dual_mesh
 * (dual_mesh_string: 8 corner cell centres then 8 scalars per line) with
 * byte-identical output, formatted by `threads` host threads (0 = all
 * cores) and written through "<path>.tmp" + rename like write_file_atomic
 * (io.cpp:307-333).  Host pointers; vertices are (x,y,z) f64 triples,
 * triangles u32 triples, corners8 the 8 CellIds of each dual, cells4 /
 * scalars the sorted arrays of the index (amrx_index_download). */
AMRX_API amrx_status amrx_write_obj(const char *path, const double *verts3, uint64_t n_verts,
                                    const uint32_t *tris3, uint64_t n_tris, int threads);
AMRX_API amrx_status amrx_write_ply(const char *path, const double *verts3, uint64_t n_verts,
                                    const uint32_t *tris3, uint64_t n_tris, int threads);
AMRX_API amrx_status amrx_write_dual_mesh(const char *path, const uint32_t *corners8,
                                          uint64_t n_duals, const int32_t *cells4,
                                          const double *scalars, uint64_t n_cells,
                                          int threads);

/* ---- single-process multi-GPU (one host thread per device, NCCL over
 * NVLink / NVSwitch).  The reference's parallelism is a thread pool over
 * candidate chunks (proj/include/amriso/parallel.hpp:49-85); its output is
 * candidate order (proj/src/pipeline.cpp:40-57), so device d extracting the
 * sorted cells [n d / N, n (d+1) / N) and the parts concatenated in device
 * order give exactly the single-GPU output. */
typedef struct amrx_comm amrx_comm;
typedef struct amrx_comm_index amrx_comm_index;

/* one NCCL communicator over `ndev` devices (ncclCommInitAll); devices =
 * NULL means 0..ndev-1, ndev <= 0 every visible device.  NCCL is loaded on
 * first use (AMRX_ERR_NCCL if it is missing). */
AMRX_API amrx_status amrx_comm_init(int ndev, const int *devices, amrx_comm **out);
/* CUDA devices visible to this process */
AMRX_API amrx_status amrx_device_count(int *n);
AMRX_API amrx_status amrx_comm_destroy(amrx_comm *comm);
AMRX_API amrx_status amrx_comm_size(const amrx_comm *comm, int *ndev);

/* build_index on the first device, the sorted keys + scalars broadcast to
 * the others (ncclBroadcast), each of which builds its own lookup
 * structure: a replicated index.  flags: AMRX_FLAG_* as in
 * amrx_index_opts.  The comm must outlive the index. */
AMRX_API amrx_status amrx_comm_index_create(amrx_comm *comm, const int32_t *cells4,
                                            const double *scalars, uint64_t n_cells,
                                            uint64_t n_scalars, uint32_t flags,
                                            amrx_comm_index **out);
AMRX_API amrx_status amrx_comm_index_destroy(amrx_comm_index *index);

/* amrx_extract_iso / amrx_extract_dual over every device: each extracts
 * its share, the parts land in the caller's buffer (host or device memory)
 * at their candidate-order offsets; xyz9 / corners8 NULL = count only.
 * Stats are summed (device times: the slowest device). */
AMRX_API amrx_status amrx_comm_extract_iso(amrx_comm_index *index,
                                           const amrx_iso_params *params, void *xyz9,
                                           uint64_t cap, uint64_t *count, amrx_stats *stats);
AMRX_API amrx_status amrx_comm_extract_dual(amrx_comm_index *index, uint32_t *corners8,
                                            uint64_t *task_ids, uint64_t cap, uint64_t *count,
                                            amrx_stats *stats);

/* testing hook: cap every extraction round's staging at `items` outputs
 * (0 = the default), so small inputs exercise the multi-round path; the
 * results are identical for every value */
AMRX_API void amrx_debug_round_limit(uint64_t items);

/* kernels this process has launched through the library so far */
AMRX_API uint64_t amrx_kernel_launches(void);

/* thread-local text of the last error on this thread */
AMRX_API const char *amrx_last_error(void);

/* library version string */
AMRX_API const char *amrx_version(void);

#ifdef __cplusplus
}
#endif

#endif /* AMRX_H */
