/* TEST ORACLE -- CPU restatement of the reference's dual-mesh / iso-surface
 * path, in plain C.  Test infrastructure only: tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product never does.
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/).  It is pinned against the reference itself
 * (oracle/_ref, tests/test_oracle.py) and the committed golden vectors
 * (tests/golden/). */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_index orc_index;

enum { ORC_ACCEPTED = 0, ORC_MISSING = 1, ORC_FINER = 2, ORC_LOWER_KEY = 3 };

/* build_index (proj/src/locator.cpp:26-92). NULL on LoadError with the
 * message available from orc_last_error(). */
orc_index *orc_build_index(const int32_t *cells4, const double *scalars,
                           uint64_t n, uint64_t n_scalars);
void orc_index_free(orc_index *idx);
uint64_t orc_index_size(const orc_index *idx);
void orc_index_get(const orc_index *idx, int32_t *cells4, double *scalars);
int orc_index_levels(const orc_index *idx, int32_t *out);
void orc_index_bounds(const orc_index *idx, int64_t *out7);
const char *orc_last_error(void);

/* find_exact / snap (locator.cpp:94-134); -1 = miss */
int64_t orc_find_exact(const orc_index *idx, const int32_t *c4);
int64_t orc_snap(const orc_index *idx, const int64_t *p3, int32_t hint);

/* try_build_dual (proj/src/dual.cpp:41-72): returns the reject code */
int orc_try_build_dual(const orc_index *idx, const int64_t *base3,
                       int32_t level, uint32_t self, uint32_t *corners8);

/* contour_hex (proj/src/contour.cpp:52-87): triangle count, -1 on the
 * collapsed-edge logic_error */
int orc_contour_hex(const uint32_t *cells8, const double *pos24,
                    const double *value8, double iso, double *out45);

/* extract_dual_mesh (proj/src/pipeline.cpp:160-194), serial.  Writes up to
 * cap duals; returns the total count.  counters4 (accepted, missing, finer,
 * lower_key) optional. */
uint64_t orc_extract_dual(const orc_index *idx, uint32_t *corners8,
                          uint32_t *owner, int64_t *base3, int32_t *level,
                          uint64_t cap, uint64_t *counters4);

/* the same over cells [cell_begin, cell_end) (sampled parity at scale) */
uint64_t orc_extract_dual_range(const orc_index *idx, uint64_t cell_begin,
                                uint64_t cell_end, uint32_t *corners8,
                                uint32_t *owner, int64_t *base3, int32_t *level,
                                uint64_t cap, uint64_t *counters4);

/* extract_isosurface passes 1+2 (pipeline.cpp:67-146) without the weld,
 * serial: the fat triangle soup in emission order, 9 doubles/triangle.
 * Writes up to cap triangles; returns the total, -1 (as UINT64_MAX) on a
 * logic_error.  counters4 as above. */
uint64_t orc_extract_iso(const orc_index *idx, double iso, double *xyz9,
                         uint64_t cap, uint64_t *counters4);

/* cells [cell_begin, cell_end) only: the candidate-order slice a range
 * partition computes (sampled parity at scale) */
uint64_t orc_extract_iso_range(const orc_index *idx, double iso,
                               uint64_t cell_begin, uint64_t cell_end,
                               double *xyz9, uint64_t cap,
                               uint64_t *counters4);

/* weld (proj/src/weld.cpp:31-64): returns the vertex count; verts3 (may be
 * NULL to count) receives position-sorted vertices, tris3 the indices */
uint64_t orc_weld(const double *xyz9, uint64_t n_tris, double *verts3,
                  uint32_t *tris3);

#ifdef __cplusplus
}
#endif
