"""ctypes access to the two CPU oracles (TEST INFRASTRUCTURE ONLY).

* ``Restatement`` -- oracle/liboracle.so, the plain-C restatement of the
  reference path (oracle/amrx_oracle.c).  Always built by ``build()``.
* ``Reference``   -- oracle/_ref/libamriso_ref.so, the unmodified reference
  sources compiled in place plus C glue (oracle/ref_harness.cpp).  Built
  where /root/reference exists; the prebuilt .so travels to the GPU box.

Both expose the same numpy-level surface so tests can run one against the
other and against the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RESTATEMENT_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REFERENCE_SO = os.path.join(ROOT, "oracle", "_ref", "libamriso_ref.so")

P = C.c_void_p
U64 = C.c_uint64
I64 = C.c_int64
I32 = C.c_int32
U32 = C.c_uint32
F64 = C.c_double


def _ptr(a):
    return a.ctypes.data_as(P) if a is not None else None


class Dataset:
    """Sorted cells (n,4) int32 + scalars (n,) f64 + levels + bounds."""

    def __init__(self, cells, scalars, levels, bounds, max_level):
        self.cells = cells
        self.scalars = scalars
        self.levels = levels
        self.bounds = bounds
        self.max_level = max_level

    def __len__(self):
        return len(self.cells)


class _Lib:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        self._fn(p + "build_index", P, [P, P, U64, U64])
        self._fn(p + "index_free", None, [P])
        self._fn(p + "index_size", U64, [P])
        self._fn(p + "index_get", None, [P, P, P])
        self._fn(p + "index_levels", C.c_int, [P, P])
        self._fn(p + "index_bounds", None, [P, P])
        self._fn(p + "last_error", C.c_char_p, [])
        self._fn(p + "find_exact", I64, [P, P])
        self._fn(p + "snap", I64, [P, P, I32])
        self._fn(p + "try_build_dual", C.c_int, [P, P, I32, U32, P])
        self._fn(p + "contour_hex", C.c_int, [P, P, P, F64, P])
        del L

    def _fn(self, name, res, args):
        f = getattr(self.lib, name)
        f.restype = res
        f.argtypes = args

    def f(self, name):
        return getattr(self.lib, self.prefix + name)

    # ------------------------------------------------------------ index
    def build(self, cells, scalars):
        cells = np.ascontiguousarray(cells, dtype=np.int32).reshape(-1, 4)
        scalars = np.ascontiguousarray(scalars, dtype=np.float64)
        h = self.f("build_index")(_ptr(cells), _ptr(scalars), len(cells), len(scalars))
        if not h:
            raise LoadErrorOracle(self.f("last_error")().decode())
        return h

    def free(self, h):
        self.f("index_free")(h)

    def dataset(self, h):
        n = self.f("index_size")(h)
        cells = np.empty((n, 4), np.int32)
        scal = np.empty(n, np.float64)
        self.f("index_get")(h, _ptr(cells), _ptr(scal))
        lv = np.empty(32, np.int32)
        nl = self.f("index_levels")(h, _ptr(lv))
        b = np.empty(7, np.int64)
        self.f("index_bounds")(h, _ptr(b))
        return Dataset(cells, scal, [int(x) for x in lv[:nl]], b[:6].copy(), int(b[6]))

    def snap(self, h, p, hint=-1):
        p = np.asarray(p, np.int64)
        return int(self.f("snap")(h, _ptr(p), hint))

    def find_exact(self, h, c):
        c = np.asarray(c, np.int32)
        return int(self.f("find_exact")(h, _ptr(c)))

    def try_build_dual(self, h, base, level, self_id):
        b = np.asarray(base, np.int64)
        out = np.zeros(8, np.uint32)
        r = self.f("try_build_dual")(h, _ptr(b), level, self_id, _ptr(out))
        return r, out

    def contour_hex(self, cells8, pos24, val8, iso):
        cells8 = np.ascontiguousarray(cells8, np.uint32)
        pos24 = np.ascontiguousarray(pos24, np.float64)
        val8 = np.ascontiguousarray(val8, np.float64)
        out = np.zeros(45, np.float64)
        k = self.f("contour_hex")(_ptr(cells8), _ptr(pos24), _ptr(val8), iso, _ptr(out))
        if k < 0:
            raise LogicErrorOracle(self.f("last_error")().decode())
        return out[: 9 * k].reshape(k, 9)


class LoadErrorOracle(Exception):
    pass


class LogicErrorOracle(Exception):
    pass


class Restatement(_Lib):
    prefix = "orc_"

    def __init__(self, path=RESTATEMENT_SO):
        super().__init__(path)
        self._fn("orc_extract_dual", U64, [P, P, P, P, P, U64, P])
        self._fn("orc_extract_dual_range", U64, [P, U64, U64, P, P, P, P, U64, P])
        self._fn("orc_extract_iso", U64, [P, F64, P, U64, P])
        self._fn("orc_extract_iso_range", U64, [P, F64, U64, U64, P, U64, P])
        self._fn("orc_weld", U64, [P, U64, P, P])

    def extract_dual(self, h):
        cnt = np.zeros(4, np.uint64)
        total = self.lib.orc_extract_dual(h, None, None, None, None, 0, _ptr(cnt))
        corners = np.empty((total, 8), np.uint32)
        owner = np.empty(total, np.uint32)
        base = np.empty((total, 3), np.int64)
        level = np.empty(total, np.int32)
        self.lib.orc_extract_dual(h, _ptr(corners), _ptr(owner), _ptr(base), _ptr(level),
                                  total, _ptr(cnt))
        return dict(corners=corners, owner=owner, base=base, level=level, counters=cnt)

    def extract_dual_range(self, h, cell_begin, cell_end):
        cnt = np.zeros(4, np.uint64)
        total = self.lib.orc_extract_dual_range(h, cell_begin, cell_end, None, None, None,
                                                None, 0, _ptr(cnt))
        corners = np.empty((total, 8), np.uint32)
        owner = np.empty(total, np.uint32)
        self.lib.orc_extract_dual_range(h, cell_begin, cell_end, _ptr(corners), _ptr(owner),
                                        None, None, total, _ptr(cnt))
        return dict(corners=corners, owner=owner, counters=cnt)

    def extract_iso(self, h, iso, cell_begin=None, cell_end=None):
        cnt = np.zeros(4, np.uint64)
        if cell_begin is None:
            cell_begin, cell_end = 0, 2**63
        total = self.lib.orc_extract_iso_range(h, iso, cell_begin, cell_end, None, 0, _ptr(cnt))
        if total == 2**64 - 1:
            raise LogicErrorOracle("collapsed edge")
        fat = np.empty((total, 9), np.float64)
        self.lib.orc_extract_iso_range(h, iso, cell_begin, cell_end, _ptr(fat), total, _ptr(cnt))
        return dict(fat=fat, counters=cnt)

    def weld(self, fat):
        fat = np.ascontiguousarray(fat, np.float64)
        n = len(fat)
        nv = self.lib.orc_weld(_ptr(fat), n, None, None)
        verts = np.empty((nv, 3), np.float64)
        tris = np.empty((n, 3), np.uint32)
        self.lib.orc_weld(_ptr(fat), n, _ptr(verts), _ptr(tris))
        return verts, tris


class Reference(_Lib):
    prefix = "ref_"

    def __init__(self, path=REFERENCE_SO):
        super().__init__(path)
        L = self.lib
        self._fn("ref_gen_uniform", P, [I32, C.c_int, P])
        self._fn("ref_gen_octree", P, [I32, C.c_int, P, F64])
        self._fn("ref_gen_blocks", P, [P, C.c_int, C.c_int, P, P, C.c_int])
        self._fn("ref_gen_slots", P, [U32, C.c_int, C.c_int, F64])
        self._fn("ref_acceptance_fixture", P, [C.c_int, P])
        self._fn("ref_validate", I64, [P, P, P])
        self._fn("ref_validate_pairs", None, [P, P, P, U64])
        self._fn("ref_extract_dual", P, [P, C.c_int, P])
        self._fn("ref_duals_count", U64, [P])
        self._fn("ref_duals_get", None, [P, P, P, P, P])
        self._fn("ref_duals_free", None, [P])
        self._fn("ref_exhaustive_duals", P, [P])
        self._fn("ref_keys_count", U64, [P])
        self._fn("ref_keys_get", None, [P, P])
        self._fn("ref_keys_free", None, [P])
        self._fn("ref_extract_iso", P, [P, F64, C.c_int, C.c_int])
        self._fn("ref_iso_stats", None, [P, P, P])
        self._fn("ref_iso_fat", None, [P, P])
        self._fn("ref_iso_mesh", None, [P, P, P])
        self._fn("ref_iso_obj", P, [P])
        self._fn("ref_iso_free", None, [P])
        self._fn("ref_weld", P, [P, U64])
        self._fn("ref_mesh_sizes", U64, [P, P])
        self._fn("ref_degenerate_hexes", None, [U32, C.c_int, P, P, P, P])
        self._fn("ref_write_mesh", C.c_int, [C.c_char_p, C.c_int, P, U64, P, U64])
        self._fn("ref_write_dual_mesh", C.c_int, [C.c_char_p, P, U64, P, P, U64])
        self._libc = C.CDLL(None)
        self._libc.free.argtypes = [P]
        del L

    def _check(self, h):
        if not h:
            raise LoadErrorOracle(self.lib.ref_last_error().decode())
        return h

    @staticmethod
    def _field(kind, params):
        kinds = {"sphere": 0, "linear": 1, "rsine": 2}
        return kinds[kind], np.asarray(params, np.float64)

    def gen_uniform(self, n, kind, params):
        k, f = self._field(kind, params)
        return self._check(self.lib.ref_gen_uniform(n, k, _ptr(f)))

    def gen_octree(self, depth, kind, params, threshold):
        k, f = self._field(kind, params)
        return self._check(self.lib.ref_gen_octree(depth, k, _ptr(f), threshold))

    def gen_blocks(self, blocks, kind, params, holes=()):
        k, f = self._field(kind, params)
        b = np.ascontiguousarray(blocks, np.int32).reshape(-1, 7)
        ho = np.ascontiguousarray(holes, np.int64).reshape(-1, 6)
        return self._check(self.lib.ref_gen_blocks(_ptr(b), len(b), k, _ptr(f), _ptr(ho), len(ho)))

    def gen_slots(self, seed, slots, max_level, hole_prob=0.15):
        return self._check(self.lib.ref_gen_slots(seed, slots, max_level, hole_prob))

    def acceptance_fixture(self, n):
        iso = C.c_double(0)
        h = self._check(self.lib.ref_acceptance_fixture(n, C.byref(iso)))
        return h, iso.value

    def validate(self, h):
        d, o = C.c_uint64(0), C.c_uint64(0)
        self.lib.ref_validate(h, C.byref(d), C.byref(o))
        return d.value, o.value

    def validate_pairs(self, h):
        nd, no = self.validate(h)
        dup = np.empty((nd, 2), np.uint32)
        ovl = np.empty((no, 2), np.uint32)
        self.lib.ref_validate_pairs(h, _ptr(dup), _ptr(ovl), max(nd, no))
        return dup, ovl

    def extract_dual(self, h, threads=0):
        secs = C.c_double(0)
        r = self._check(self.lib.ref_extract_dual(h, threads, C.byref(secs)))
        n = self.lib.ref_duals_count(r)
        corners = np.empty((n, 8), np.uint32)
        base = np.empty((n, 3), np.int64)
        level = np.empty(n, np.int32)
        owner = np.empty(n, np.uint32)
        self.lib.ref_duals_get(r, _ptr(corners), _ptr(base), _ptr(level), _ptr(owner))
        self.lib.ref_duals_free(r)
        return dict(corners=corners, base=base, level=level, owner=owner, seconds=secs.value)

    def exhaustive_duals(self, h):
        r = self._check(self.lib.ref_exhaustive_duals(h))
        n = self.lib.ref_keys_count(r)
        keys = np.empty((n, 8), np.uint32)
        self.lib.ref_keys_get(r, _ptr(keys))
        self.lib.ref_keys_free(r)
        return keys

    def extract_iso(self, h, iso, threads=0, emit_dual=False, want_obj=False):
        r = self._check(self.lib.ref_extract_iso(h, iso, threads, int(emit_dual)))
        u = np.empty(9, np.uint64)
        t = np.empty(4, np.float64)
        self.lib.ref_iso_stats(r, _ptr(u), _ptr(t))
        stats = dict(zip(["cell_count", "duals_accepted", "duals_missing_corner",
                          "duals_finer_corner", "duals_lower_key_corner",
                          "pass1_triangle_count", "fat_triangle_count",
                          "welded_vertex_count", "welded_triangle_count"],
                         [int(x) for x in u]))
        stats.update(dict(zip(["seconds_sort", "seconds_pass1", "seconds_pass2",
                               "seconds_weld"], [float(x) for x in t])))
        fat = np.empty((stats["welded_triangle_count"], 9), np.float64)
        self.lib.ref_iso_fat(r, _ptr(fat))
        verts = np.empty((stats["welded_vertex_count"], 3), np.float64)
        tris = np.empty((stats["welded_triangle_count"], 3), np.uint32)
        self.lib.ref_iso_mesh(r, _ptr(verts), _ptr(tris))
        out = dict(stats=stats, fat=fat, verts=verts, tris=tris)
        if want_obj:
            s = self.lib.ref_iso_obj(r)
            out["obj"] = C.string_at(s).decode()
            self._libc.free(s)
        self.lib.ref_iso_free(r)
        return out

    def weld(self, fat):
        fat = np.ascontiguousarray(fat, np.float64)
        r = self._check(self.lib.ref_weld(_ptr(fat), len(fat)))
        nt = C.c_uint64(0)
        nv = self.lib.ref_mesh_sizes(r, C.byref(nt))
        verts = np.empty((nv, 3), np.float64)
        tris = np.empty((nt.value, 3), np.uint32)
        self.lib.ref_iso_mesh(r, _ptr(verts), _ptr(tris))
        self.lib.ref_iso_free(r)
        return verts, tris

    def degenerate_hexes(self, seed, count):
        cells = np.empty((count, 8), np.uint32)
        pos = np.empty((count, 24), np.float64)
        val = np.empty((count, 8), np.float64)
        iso = np.empty(count, np.float64)
        self.lib.ref_degenerate_hexes(seed, count, _ptr(cells), _ptr(pos), _ptr(val), _ptr(iso))
        return cells, pos, val, iso


def restatement():
    return Restatement()


def reference():
    """The compiled reference, or None where oracle/_ref was not built."""
    if not os.path.exists(REFERENCE_SO):
        return None
    return Reference()
