"""Python host mirror of the reference's operator API over the amrx C ABI.

Names, argument meaning and error behaviour follow the reference's free
functions in namespace ``amriso`` (paths under /root/reference/):

  build_index(cells, scalars)          proj/include/amriso/locator.hpp:52-53
  find_exact(index, coord)             proj/include/amriso/locator.hpp:55-57
  snap(index, p, hint_level=-1)        proj/include/amriso/locator.hpp:59-66
  try_build_dual(index, base...)       proj/include/amriso/dual.hpp:78-81
  extract_dual_mesh(index, threads=0)  proj/include/amriso/pipeline.hpp:70-71
  extract_isosurface(index, params)    proj/include/amriso/pipeline.hpp:65-66

Errors map to the reference's exception types: ``LoadError`` (a
RuntimeError, core.hpp:62-65), ``ValueError`` for std::invalid_argument,
``OverflowError`` for std::length_error and ``InternalError`` (a
RuntimeError standing for std::logic_error).

Everything computes on the GPU through libamrx.so.  There is no CPU
fallback: importing works anywhere, but any call raises if the library or a
CUDA device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# AMRX_LIB selects an alternate in-tree build (A/B experiments)
LIB_PATH = os.environ.get("AMRX_LIB") or os.path.join(_HERE, "libamrx.so")

AMRX_OK = 0
AMRX_ERR_LOAD = 1
AMRX_ERR_INVALID_ARG = 2
AMRX_ERR_LENGTH = 3
AMRX_ERR_INTERNAL = 4
AMRX_ERR_CUDA = 5
AMRX_ERR_CAPACITY = 6
AMRX_ERR_UNSUPPORTED = 7
AMRX_ERR_NO_DEVICE = 8
AMRX_ERR_IO = 9
AMRX_ERR_NCCL = 10

MAX_LEVEL = 30

# DualReject (dual.hpp:38-43)
ACCEPTED, MISSING_CORNER, FINER_CORNER, LOWER_KEY_CORNER = 0, 1, 2, 3


class LoadError(RuntimeError):
    """malformed input (core.hpp:62-65)"""


class InternalError(RuntimeError):
    """internal consistency failure (std::logic_error, core.hpp:67-74)"""


class CudaError(RuntimeError):
    pass


class CapacityError(RuntimeError):
    def __init__(self, msg, count):
        super().__init__(msg)
        self.count = count


class UnsupportedError(RuntimeError):
    pass


class _IndexInfo(C.Structure):
    _fields_ = [("cell_count", C.c_uint64), ("max_level", C.c_int32),
                ("level_count", C.c_int32), ("levels", C.c_int32 * 31),
                ("bounds_lo", C.c_int64 * 3), ("bounds_hi", C.c_int64 * 3),
                ("key_bits", C.c_int32), ("directory_bits", C.c_int32),
                ("duplicate_keys", C.c_uint64), ("device_bytes", C.c_uint64),
                ("seconds_ingest", C.c_double), ("lookup", C.c_int32),
                ("max_probe", C.c_uint32), ("lookup_entries", C.c_uint64)]


# index lookup structures (amrx.h AMRX_FLAG_LOOKUP_* / AMRX_LOOKUP_*)
_LOOKUP_FLAGS = {None: 0, "auto": 0, "records": 0x2, "hash": 0x4, "directory": 0x8}
_LOOKUP_NAMES = {0: "directory", 1: "records", 2: "hash", 3: "wide"}


def _flags(presorted=False, lookup=None):
    if lookup not in _LOOKUP_FLAGS:
        raise ValueError(f"lookup must be one of {sorted(k for k in _LOOKUP_FLAGS if k)}")
    return (1 if presorted else 0) | _LOOKUP_FLAGS[lookup]


class _Opts(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("flags", C.c_uint32)]


class _Stats(C.Structure):
    _fields_ = [("cell_count", C.c_uint64), ("duals_accepted", C.c_uint64),
                ("duals_missing_corner", C.c_uint64), ("duals_finer_corner", C.c_uint64),
                ("duals_lower_key_corner", C.c_uint64),
                ("pass1_triangle_count", C.c_uint64), ("fat_triangle_count", C.c_uint64),
                ("dual_count", C.c_uint64), ("seconds_pass1", C.c_double),
                ("seconds_pass2", C.c_double), ("kernel_launches", C.c_uint64)]


class _Range(C.Structure):
    _fields_ = [("cell_begin", C.c_uint64), ("cell_end", C.c_uint64)]


class _IsoParams(C.Structure):
    _fields_ = [("iso", C.c_double), ("xyz_is_f32", C.c_int32), ("check_length", C.c_int32)]


_lib = None


def library():
    """Load libamrx.so (raises if it was never built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P, U64, I64, I32 = C.c_void_p, C.c_uint64, C.c_int64, C.c_int32
    sig = {
        "amrx_index_create": [P, P, U64, U64, P, P],
        "amrx_read_amr": [C.c_char_p, P, P],
        "amrx_write_obj": [C.c_char_p, P, U64, P, U64, I32],
        "amrx_write_ply": [C.c_char_p, P, U64, P, U64, I32],
        "amrx_write_dual_mesh": [C.c_char_p, P, U64, P, P, U64, I32],
        "amrx_index_destroy": [P],
        "amrx_index_get_info": [P, P],
        "amrx_index_download": [P, P, P],
        "amrx_index_device_arrays": [P, P, P],
        "amrx_index_geometry": [P, P],
        "amrx_index_adopt": [P, P, U64, P, P, P],
        "amrx_bounds": [P, U64, P, P],
        "amrx_index_sort_part": [P, P, U64, P, P, P],
        "amrx_index_from_keys": [P, P, U64, P, P, P],
        "amrx_weld": [P, U64, P, U64, P, P, P],
        "amrx_validate": [P, P, U64, P, P, U64, P],
        "amrx_release_cached_memory": [I32],
        "amrx_find_exact": [P, P, U64, P],
        "amrx_snap": [P, P, P, I32, U64, P],
        "amrx_try_build_duals": [P, P, U64, P, P],
        "amrx_extract_dual": [P, P, P, P, U64, P, P],
        "amrx_extract_iso": [P, P, P, P, U64, P, P],
        "amrx_device_count": [P],
        "amrx_extract_iso_mesh": [P, P, P, P, U64, P, U64, P, P, P, P],
        "amrx_extract_dual_cells": [P, P, P, U64, P, P],
        "amrx_comm_init": [C.c_int, P, P],
        "amrx_comm_destroy": [P],
        "amrx_comm_size": [P, P],
        "amrx_comm_index_create": [P, P, P, U64, U64, C.c_uint32, P],
        "amrx_comm_index_destroy": [P],
        "amrx_comm_extract_iso": [P, P, P, U64, P, P],
        "amrx_comm_extract_dual": [P, P, P, U64, P, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    lib.amrx_last_error.restype = C.c_char_p
    lib.amrx_last_error.argtypes = []
    lib.amrx_version.restype = C.c_char_p
    lib.amrx_debug_round_limit.restype = None
    lib.amrx_debug_round_limit.argtypes = [C.c_uint64]
    lib.amrx_kernel_launches.restype = C.c_uint64
    lib.amrx_kernel_launches.argtypes = []
    _lib = lib
    return lib


def _check(status, count=None):
    if status == AMRX_OK:
        return
    msg = library().amrx_last_error().decode()
    if status == AMRX_ERR_LOAD:
        raise LoadError(msg)
    if status == AMRX_ERR_INVALID_ARG:
        raise ValueError(msg)
    if status == AMRX_ERR_LENGTH:
        raise OverflowError(msg)
    if status == AMRX_ERR_INTERNAL:
        raise InternalError(msg)
    if status == AMRX_ERR_CAPACITY:
        raise CapacityError(msg, count)
    if status == AMRX_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == AMRX_ERR_IO:
        raise OSError(msg)
    raise CudaError(msg)


def _ptr(a):
    """ctypes pointer of a numpy array or a torch tensor (host or CUDA)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())


@dataclass
class IndexInfo:
    cell_count: int
    max_level: int
    levels: list
    bounds_lo: tuple
    bounds_hi: tuple
    key_bits: int
    directory_bits: int
    duplicate_keys: int
    device_bytes: int
    seconds_ingest: float
    lookup: str = "records"
    max_probe: int = 0
    lookup_entries: int = 0


class CellIndex:
    """Device-resident search structure (CellIndex, locator.hpp:38-45).

    ``cells``/``scalars`` (sorted, like CellIndex.data) are downloaded
    lazily on first access."""

    def __init__(self, handle, lib):
        self._h = C.c_void_p(handle)
        self._lib = lib
        self._cells = None
        self._scalars = None
        info = _IndexInfo()
        _check(lib.amrx_index_get_info(self._h, C.byref(info)))
        self.info = IndexInfo(
            info.cell_count, info.max_level, list(info.levels[: info.level_count]),
            tuple(info.bounds_lo), tuple(info.bounds_hi), info.key_bits,
            info.directory_bits, info.duplicate_keys, info.device_bytes,
            info.seconds_ingest, _LOOKUP_NAMES.get(info.lookup, str(info.lookup)),
            info.max_probe, info.lookup_entries)

    # -- CellIndex surface
    def size(self):
        return self.info.cell_count

    def __len__(self):
        return self.info.cell_count

    @property
    def levels(self):
        return self.info.levels

    @property
    def max_level(self):
        return self.info.max_level

    @property
    def bounds(self):
        return self.info.bounds_lo, self.info.bounds_hi

    def _download(self):
        n = self.size()
        cells = np.empty((n, 4), np.int32)
        scal = np.empty(n, np.float64)
        _check(self._lib.amrx_index_download(self._h, _ptr(cells), _ptr(scal)))
        self._cells, self._scalars = cells, scal

    @property
    def cells(self):
        if self._cells is None:
            self._download()
        return self._cells

    @property
    def scalars(self):
        if self._scalars is None:
            self._download()
        return self._scalars

    def device_arrays(self):
        k, s = C.c_void_p(), C.c_void_p()
        _check(self._lib.amrx_index_device_arrays(self._h, C.byref(k), C.byref(s)))
        return k.value, s.value

    def geometry(self):
        g = np.zeros(16, np.int64)
        _check(self._lib.amrx_index_geometry(self._h, _ptr(g)))
        return g

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            self._lib.amrx_index_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def release_cached_memory(device=-1):
    """return the device memory the library caches between calls (idle
    workspace buffers, pool free blocks) -- e.g. before a large torch
    allocation in the same process"""
    _check(library().amrx_release_cached_memory(device))


def debug_round_limit(items=0):
    """testing hook: cap every extraction round's staging at ``items``
    outputs (0 = default) -- results are identical for every value"""
    library().amrx_debug_round_limit(int(items))


def kernel_launches():
    """kernels launched through libamrx.so by this process so far"""
    return int(library().amrx_kernel_launches())


def build_index(cells, scalars, device=-1, presorted=False, stream=None, lookup=None):
    """Sort cells (with their scalars) into a device CellIndex
    (build_index, locator.cpp:26-92).  ``cells`` is (n,4) int32 (i,j,k,level),
    numpy or torch (host or CUDA).  ``lookup`` forces the index's lookup
    structure ("records", "hash" or "directory"; default: chosen from the
    key space) -- every choice gives identical results."""
    lib = library()
    if isinstance(cells, np.ndarray) or not hasattr(cells, "data_ptr"):
        cells = np.ascontiguousarray(np.asarray(cells, dtype=np.int32).reshape(-1, 4))
        n_cells = len(cells)
    else:
        n_cells = cells.shape[0] if cells.numel() else 0
    if isinstance(scalars, np.ndarray) or not hasattr(scalars, "data_ptr"):
        scalars = np.ascontiguousarray(np.asarray(scalars, dtype=np.float64).reshape(-1))
        n_s = len(scalars)
    else:
        n_s = scalars.numel()
    opts = _Opts(device, C.c_void_p(stream) if stream else None, _flags(presorted, lookup))
    h = C.c_void_p()
    _check(lib.amrx_index_create(_ptr(cells) if n_cells else C.c_void_p(1),
                                 _ptr(scalars) if n_s else C.c_void_p(1),
                                 n_cells, n_s, C.byref(opts), C.byref(h)))
    return CellIndex(h.value, lib)


def read_amr(path, device=-1, stream=None, lookup=None):
    """Read an AMRCELL1 cell file (binary, or text for a ``.txt`` path) into
    a device CellIndex (read_amr, io.cpp:76-181).  Binary records stream
    through pinned chunks straight to the GPU; errors raise LoadError with
    the reference's messages, prefixed with the path."""
    lib = library()
    opts = _Opts(device, C.c_void_p(stream) if stream else None, _flags(False, lookup))
    h = C.c_void_p()
    _check(lib.amrx_read_amr(os.fsencode(os.fspath(path)), C.byref(opts), C.byref(h)))
    return CellIndex(h.value, lib)


def write_amr(path, cells, scalars):
    """Write cells + scalars as an AMRCELL1 binary file (write_amr's binary
    branch, io.cpp:194-208; host-side, for producing inputs)."""
    cells = np.ascontiguousarray(np.asarray(cells, np.int32).reshape(-1, 4))
    scalars = np.ascontiguousarray(np.asarray(scalars, np.float64).reshape(-1))
    rec = np.empty(len(cells), dtype=[("c", "<i4", 4), ("s", "<f8")])
    rec["c"] = cells
    rec["s"] = scalars
    with open(path, "wb") as f:
        f.write(b"AMRCELL1")
        f.write(np.array([1], "<u4").tobytes())
        f.write(np.array([len(cells)], "<u8").tobytes())
        f.write(np.array([1], "<u4").tobytes())
        f.write(rec.tobytes())


def adopt_index(keys_dev_ptr, scalars_dev_ptr, n_cells, geometry, device=-1, stream=None,
                lookup=None):
    """Index over already-sorted packed keys + scalars on this device (the
    multi-GPU replica path: no sort, directory only)."""
    lib = library()
    g = np.ascontiguousarray(geometry, np.int64)
    opts = _Opts(device, C.c_void_p(stream) if stream else None, _flags(False, lookup))
    h = C.c_void_p()
    _check(lib.amrx_index_adopt(C.c_void_p(keys_dev_ptr), C.c_void_p(scalars_dev_ptr),
                                n_cells, _ptr(g), C.byref(opts), C.byref(h)))
    return CellIndex(h.value, lib)


def _cells_arg(cells):
    if isinstance(cells, np.ndarray) or not hasattr(cells, "data_ptr"):
        cells = np.ascontiguousarray(np.asarray(cells, dtype=np.int32).reshape(-1, 4))
        return cells, len(cells)
    return cells, (cells.shape[0] if cells.numel() else 0)


def cell_bounds(cells, device=-1, stream=None):
    """(10,) int64: min anchor[3], max anchor[3], max anchor + width[3],
    level mask of a slice of the cell list -- reduced across ranks into the
    global geometry of a distributed build (dist.build_distributed)"""
    lib = library()
    cells, n = _cells_arg(cells)
    out = np.zeros(10, np.int64)
    opts = _Opts(device, C.c_void_p(stream) if stream else None, 0)
    _check(lib.amrx_bounds(_ptr(cells) if n else C.c_void_p(1), n, C.byref(opts), _ptr(out)))
    return out


def sort_part(cells, scalars, geometry, device=-1, stream=None):
    """a slice sorted under the global geometry: sorted keys + scalars only
    (device_arrays()), no search structure"""
    lib = library()
    cells, n = _cells_arg(cells)
    if isinstance(scalars, np.ndarray) or not hasattr(scalars, "data_ptr"):
        scalars = np.ascontiguousarray(np.asarray(scalars, dtype=np.float64).reshape(-1))
    g = np.ascontiguousarray(geometry, np.int64)
    opts = _Opts(device, C.c_void_p(stream) if stream else None, 0)
    h = C.c_void_p()
    _check(lib.amrx_index_sort_part(_ptr(cells) if n else C.c_void_p(1), _ptr(scalars), n,
                                    _ptr(g), C.byref(opts), C.byref(h)))
    return CellIndex(h.value, lib)


def index_from_keys(keys_dev_ptr, scalars_dev_ptr, n_cells, geometry, device=-1, stream=None,
                    lookup=None):
    """index of one partition of a distributed index: packed keys (any
    order) + scalars on this device inside the key range geometry[13:15];
    geometry[12] = global CellId of its first key; every id it reports is
    global"""
    lib = library()
    g = np.ascontiguousarray(geometry, np.int64)
    opts = _Opts(device, C.c_void_p(stream) if stream else None, _flags(False, lookup))
    h = C.c_void_p()
    _check(lib.amrx_index_from_keys(C.c_void_p(keys_dev_ptr), C.c_void_p(scalars_dev_ptr),
                                    n_cells, _ptr(g), C.byref(opts), C.byref(h)))
    return CellIndex(h.value, lib)


@dataclass
class ValidationReport:
    """ValidationReport (locator.hpp:70-78): (n, n+1) duplicate pairs and
    (finer, coarser) overlap pairs of CellIds"""
    duplicates: np.ndarray  # (D, 2) uint32
    overlaps: np.ndarray    # (O, 2) uint32

    def ok(self):
        return len(self.duplicates) == 0 and len(self.overlaps) == 0

    def describe(self, index):
        """the reference's text (locator.cpp:163-185)"""
        cells = index.cells

        def cell(i):
            c = cells[int(i)]
            return f"({c[0]} {c[1]} {c[2]} level {c[3]})"

        out = f"{len(self.duplicates)} duplicate pair(s), {len(self.overlaps)} overlap pair(s)"
        for a, _ in self.duplicates[:8]:
            out += "\n  duplicate cell " + cell(a)
        for a, b in self.overlaps[:8]:
            out += "\n  cell " + cell(a) + " lies inside " + cell(b)
        return out


def validate_dataset(index: CellIndex):
    """validate_dataset (locator.cpp:136-161) on the GPU"""
    lib = index._lib
    nd, no = C.c_uint64(), C.c_uint64()
    _check(lib.amrx_validate(index.handle, None, 0, C.byref(nd), None, 0, C.byref(no)))
    dup = np.empty((nd.value, 2), np.uint32)
    ovl = np.empty((no.value, 2), np.uint32)
    _check(lib.amrx_validate(index.handle, _ptr(dup) if nd.value else None, nd.value,
                             C.byref(nd), _ptr(ovl) if no.value else None, no.value,
                             C.byref(no)))
    return ValidationReport(dup, ovl)


@dataclass
class IndexedMesh:
    """IndexedMesh (weld.hpp:28-31): shared vertices + triangle indices"""
    vertices: object   # (V, 3) float64, position-sorted
    triangles: object  # (T, 3) uint32


def weld(triangles, device=-1, stream=None):
    """weld (weld.cpp:31-64) on the GPU: merge bitwise-identical corner
    positions of a fat triangle soup ((T, 9) float64, numpy or torch host or
    CUDA) into an IndexedMesh with the reference's vertex order."""
    lib = library()
    on_gpu = hasattr(triangles, "is_cuda") and triangles.is_cuda
    if isinstance(triangles, np.ndarray) or not hasattr(triangles, "data_ptr"):
        tri = np.ascontiguousarray(np.asarray(triangles, np.float64).reshape(-1, 9))
        n = len(tri)
    else:
        tri = triangles.contiguous()
        n = tri.shape[0] if tri.numel() else 0
    if on_gpu:  # CUDA tensor in: the mesh stays on the device
        import torch
        verts = torch.empty((3 * n, 3), dtype=torch.float64, device=tri.device)
        idx = torch.empty((n, 3), dtype=torch.int32, device=tri.device)
    else:
        verts = np.empty((3 * n, 3), np.float64)
        idx = np.empty((n, 3), np.uint32)
    nv = C.c_uint64()
    opts = _Opts(device, C.c_void_p(stream) if stream else None, 0)
    _check(lib.amrx_weld(_ptr(tri) if n else None, n, _ptr(verts), 3 * n, _ptr(idx),
                         C.byref(nv), C.byref(opts)))
    if on_gpu:
        return IndexedMesh(verts[: nv.value], idx)  # ids as int32 (torch has no uint32 ops)
    return IndexedMesh(verts[: nv.value].copy(), idx)


def find_exact(index: CellIndex, coords):
    """CellId per (i,j,k,level) row, -1 = absent (locator.cpp:94-101)."""
    c = np.ascontiguousarray(np.asarray(coords, np.int32).reshape(-1, 4))
    out = np.empty(len(c), np.int64)
    _check(index._lib.amrx_find_exact(index.handle, _ptr(c), len(c), _ptr(out)))
    return out


def snap(index: CellIndex, points, hint_level=-1):
    """CellId containing each int64 point, -1 = none (locator.cpp:122-134).
    ``hint_level`` is one int or one per point."""
    p = np.ascontiguousarray(np.asarray(points, np.int64).reshape(-1, 3))
    out = np.empty(len(p), np.int64)
    if np.ndim(hint_level) == 0:
        _check(index._lib.amrx_snap(index.handle, _ptr(p), None, int(hint_level),
                                    len(p), _ptr(out)))
    else:
        h = np.ascontiguousarray(np.asarray(hint_level, np.int32).reshape(-1))
        _check(index._lib.amrx_snap(index.handle, _ptr(p), _ptr(h), -1, len(p), _ptr(out)))
    return out


def try_build_duals(index: CellIndex, tasks):
    """try_build_dual for candidate tasks (cell*8+delta): (reject codes,
    corners[n,8]) (dual.cpp:41-72)."""
    t = np.ascontiguousarray(np.asarray(tasks, np.uint64).reshape(-1))
    rej = np.empty(len(t), np.uint8)
    cor = np.empty((len(t), 8), np.uint32)
    _check(index._lib.amrx_try_build_duals(index.handle, _ptr(t), len(t), _ptr(rej), _ptr(cor)))
    return rej, cor


@dataclass
class ExtractionStats:
    """ExtractionStats (pipeline.hpp:29-49); times are device seconds."""
    cell_count: int = 0
    duals_accepted: int = 0
    duals_missing_corner: int = 0
    duals_finer_corner: int = 0
    duals_lower_key_corner: int = 0
    pass1_triangle_count: int = 0
    fat_triangle_count: int = 0
    dual_count: int = 0
    seconds_pass1: float = 0.0
    seconds_pass2: float = 0.0
    kernel_launches: int = 0

    @staticmethod
    def _from(s: _Stats):
        return ExtractionStats(*[getattr(s, f) for f, _ in _Stats._fields_])


@dataclass
class IsoParams:
    """IsoParams (pipeline.hpp:23-27); thread_count is accepted and ignored."""
    iso: float = 0.0
    emit_dual_mesh: bool = False
    thread_count: int = 0
    f32: bool = False


@dataclass
class DualMesh:
    """extract_dual_mesh's result as arrays: corners[n,8] CellIds and the
    candidate task id owner*8+delta (owner/base/level follow)."""
    corners: np.ndarray
    tasks: np.ndarray
    stats: ExtractionStats = None

    @property
    def owner(self):
        return (self.tasks >> np.uint64(3)).astype(np.uint32)

    @property
    def delta(self):
        return (self.tasks & np.uint64(7)).astype(np.int32)

    def __len__(self):
        return len(self.corners)


@dataclass
class ExtractionResult:
    fat: np.ndarray                      # [n,9] triangle soup (emission order)
    stats: ExtractionStats
    duals: DualMesh = None
    extra: dict = field(default_factory=dict)


def _range(r):
    if r is None:
        return None
    return C.byref(_Range(int(r[0]), int(r[1])))


def extract_dual_mesh(index: CellIndex, thread_count=0, cell_range=None, out=None):
    """The accepted duals in candidate order (pipeline.cpp:160-194).
    ``out`` = (corners, tasks) preallocated device tensors to write into."""
    lib = index._lib
    st = _Stats()
    cnt = C.c_uint64(0)
    if out is not None:
        corners, tasks = out
        cap = corners.shape[0]
        rc = lib.amrx_extract_dual(index.handle, _range(cell_range), _ptr(corners), _ptr(tasks),
                                   cap, C.byref(cnt), C.byref(st))
        _check(rc, cnt.value)
        return DualMesh(corners[: cnt.value], tasks[: cnt.value], ExtractionStats._from(st))
    _check(lib.amrx_extract_dual(index.handle, _range(cell_range), None, None, 0,
                                 C.byref(cnt), C.byref(st)))
    n = cnt.value
    corners = np.empty((n, 8), np.uint32)
    tasks = np.empty(n, np.uint64)
    if n:
        _check(lib.amrx_extract_dual(index.handle, _range(cell_range), _ptr(corners), _ptr(tasks),
                                     n, C.byref(cnt), C.byref(st)))
    return DualMesh(corners, tasks, ExtractionStats._from(st))


def extract_isosurface(index: CellIndex, params: IsoParams = None, cell_range=None,
                       out=None, check_length=True):
    """Passes 1+2 of extract_isosurface (pipeline.cpp:67-146): the fat
    triangle soup in emission order plus ExtractionStats.  The weld
    (weld.cpp:31-64) is not part of this path; see DESIGN.md."""
    if params is None:
        params = IsoParams()
    elif isinstance(params, (int, float)):
        params = IsoParams(iso=float(params))
    lib = index._lib
    p = _IsoParams(float(params.iso), 1 if params.f32 else 0, 1 if check_length else 0)
    st = _Stats()
    cnt = C.c_uint64(0)
    dtype = np.float32 if params.f32 else np.float64
    if out is not None:
        rc = lib.amrx_extract_iso(index.handle, _range(cell_range), C.byref(p), _ptr(out),
                                  out.shape[0], C.byref(cnt), C.byref(st))
        _check(rc, cnt.value)
        fat = out[: cnt.value]
    else:
        _check(lib.amrx_extract_iso(index.handle, _range(cell_range), C.byref(p), None, 0,
                                    C.byref(cnt), C.byref(st)))
        fat = np.empty((cnt.value, 9), dtype)
        if cnt.value:
            _check(lib.amrx_extract_iso(index.handle, _range(cell_range), C.byref(p),
                                        _ptr(fat), cnt.value, C.byref(cnt), C.byref(st)))
    res = ExtractionResult(fat, ExtractionStats._from(st))
    if params.emit_dual_mesh:
        res.duals = extract_dual_mesh(index, cell_range=cell_range)
    return res


DUAL_CELL = np.dtype([("corners", "<u4", 8), ("base", "<i8", 3), ("level", "<i4"),
                      ("owner", "<u4")])  # DualCell, dual.hpp:30-35 (64 bytes)


def extract_dual_cells(index: CellIndex, cell_range=None):
    """extract_dual_mesh as the reference returns it (pipeline.cpp:160-194):
    DualCell records (corners, base, level, owner) built on the device"""
    lib = index._lib
    st = _Stats()
    cnt = C.c_uint64(0)
    _check(lib.amrx_extract_dual_cells(index.handle, _range(cell_range), None, 0, C.byref(cnt),
                                       C.byref(st)))
    out = np.empty(cnt.value, DUAL_CELL)
    if cnt.value:
        _check(lib.amrx_extract_dual_cells(index.handle, _range(cell_range), _ptr(out), cnt.value,
                                           C.byref(cnt), C.byref(st)))
    return out


def extract_isosurface_mesh(index: CellIndex, params: IsoParams = None, cell_range=None):
    """extract_isosurface as the reference returns it (pipeline.cpp:67-158):
    passes 1+2 and the weld on the device, only the IndexedMesh crosses to the
    host (vertices position-sorted, triangles in candidate order); returns
    (IndexedMesh, ExtractionStats, seconds_weld)"""
    if params is None:
        params = IsoParams()
    elif isinstance(params, (int, float)):
        params = IsoParams(iso=float(params))
    lib = index._lib
    p = _IsoParams(float(params.iso), 0, 1)
    st = _Stats()
    nv, nt, tw = C.c_uint64(0), C.c_uint64(0), C.c_double(0)
    _check(lib.amrx_extract_iso_mesh(index.handle, _range(cell_range), C.byref(p), None, 0, None,
                                     0, C.byref(nv), C.byref(nt), C.byref(tw), C.byref(st)))
    verts = np.empty((nv.value, 3), np.float64)
    tris = np.empty((nt.value, 3), np.uint32)
    if nv.value or nt.value:
        _check(lib.amrx_extract_iso_mesh(index.handle, _range(cell_range), C.byref(p),
                                         _ptr(verts), nv.value, _ptr(tris), nt.value,
                                         C.byref(nv), C.byref(nt), C.byref(tw), C.byref(st)))
    return IndexedMesh(verts, tris), ExtractionStats._from(st), tw.value


def dual_bases(index: CellIndex, tasks):
    """DualCell.base / .level for task ids (dual_base_of, dual.hpp:61-67)."""
    t = np.asarray(tasks, np.uint64)
    owner = (t >> np.uint64(3)).astype(np.int64)
    delta = (t & np.uint64(7)).astype(np.int64)
    c = index.cells[owner].astype(np.int64)
    w = np.left_shift(np.int64(1), c[:, 3])
    base = np.stack([c[:, a] - np.where((delta >> a) & 1, 0, w) for a in range(3)], axis=1)
    return base, c[:, 3].astype(np.int32)


def _host(a, dtype, cols):
    """host, contiguous, ``dtype`` (int32 CellIds/indices are viewed as u32)"""
    if hasattr(a, "is_cuda"):
        a = a.cpu().numpy()
    a = np.asarray(a)
    if a.dtype != dtype and a.dtype.kind in "iu" and a.dtype.itemsize == np.dtype(dtype).itemsize:
        a = a.view(dtype)
    return np.ascontiguousarray(a, dtype).reshape(-1, cols)


def _mesh_arrays(mesh):
    v = _host(mesh.vertices, np.float64, 3)
    t = _host(mesh.triangles, np.uint32, 3)
    return v, t


def write_obj(path, mesh, threads=0):
    """write_obj (io.cpp:219-239): Wavefront OBJ, shortest round-trip decimals,
    byte-identical to the reference; formatted by host threads."""
    v, t = _mesh_arrays(mesh)
    _check(library().amrx_write_obj(os.fsencode(os.fspath(path)), _ptr(v), len(v), _ptr(t),
                                    len(t), threads))


def write_ply(path, mesh, threads=0):
    """write_ply (io.cpp:241-272): binary little-endian PLY, float32 positions."""
    v, t = _mesh_arrays(mesh)
    _check(library().amrx_write_ply(os.fsencode(os.fspath(path)), _ptr(v), len(v), _ptr(t),
                                    len(t), threads))


def write_dual_mesh(path, duals, index, threads=0):
    """write_dual_mesh (io.cpp:274-305): per dual, the 8 corner cell centres
    then the 8 scalars.  ``duals`` is a DualMesh (or (n, 8) corner CellIds),
    ``index`` the CellIndex they came from."""
    corners = duals.corners if hasattr(duals, "corners") else duals
    corners = _host(corners, np.uint32, 8)
    cells = np.ascontiguousarray(index.cells)
    scal = np.ascontiguousarray(index.scalars)
    _check(library().amrx_write_dual_mesh(os.fsencode(os.fspath(path)), _ptr(corners),
                                          len(corners), _ptr(cells), _ptr(scal), len(cells),
                                          threads))



# ---------------------------------------------------------------------------
# single-process multi-GPU (amrx_comm_*: NCCL over NVLink, one host thread
# per device)

def device_count():
    n = C.c_int(0)
    _check(library().amrx_device_count(C.byref(n)))
    return n.value


class Comm:
    """one NCCL communicator over several GPUs of this process
    (amrx_comm_init); ``devices`` = list of ordinals, None = all visible"""

    def __init__(self, devices=None):
        lib = library()
        self._lib = lib
        self._h = C.c_void_p()
        if devices is None:
            _check(lib.amrx_comm_init(0, None, C.byref(self._h)))
        else:
            d = (C.c_int * len(devices))(*devices)
            _check(lib.amrx_comm_init(len(devices), d, C.byref(self._h)))

    def size(self):
        n = C.c_int(0)
        _check(self._lib.amrx_comm_size(self._h, C.byref(n)))
        return n.value

    def build_index(self, cells, scalars, presorted=False, lookup=None):
        """build_index on the first device, broadcast to the others"""
        cells = np.ascontiguousarray(np.asarray(cells, np.int32).reshape(-1, 4)) \
            if not hasattr(cells, "data_ptr") else cells
        scalars = np.ascontiguousarray(np.asarray(scalars, np.float64).reshape(-1)) \
            if not hasattr(scalars, "data_ptr") else scalars
        n = cells.shape[0]
        ns = scalars.shape[0]
        h = C.c_void_p()
        _check(self._lib.amrx_comm_index_create(self._h, _ptr(cells), _ptr(scalars), n, ns,
                                                _flags(presorted, lookup), C.byref(h)))
        return CommIndex(h.value, self)

    def close(self):
        if self._h:
            self._lib.amrx_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CommIndex:
    """a replicated index over a Comm's devices; extraction splits the
    cells across them and concatenates in candidate order"""

    def __init__(self, handle, comm):
        self._h = C.c_void_p(handle)
        self._comm = comm

    def extract_isosurface(self, params=None, out=None):
        if params is None:
            params = IsoParams()
        elif isinstance(params, (int, float)):
            params = IsoParams(iso=float(params))
        lib = self._comm._lib
        p = _IsoParams(float(params.iso), 1 if params.f32 else 0, 1)
        st = _Stats()
        cnt = C.c_uint64(0)
        if out is None:
            _check(lib.amrx_comm_extract_iso(self._h, C.byref(p), None, 0, C.byref(cnt),
                                             C.byref(st)))
            out = np.empty((cnt.value, 9), np.float32 if params.f32 else np.float64)
        rc = lib.amrx_comm_extract_iso(self._h, C.byref(p), _ptr(out), out.shape[0],
                                       C.byref(cnt), C.byref(st))
        _check(rc, cnt.value)
        return ExtractionResult(out[: cnt.value], ExtractionStats._from(st))

    def extract_dual_mesh(self):
        lib = self._comm._lib
        st = _Stats()
        cnt = C.c_uint64(0)
        _check(lib.amrx_comm_extract_dual(self._h, None, None, 0, C.byref(cnt), C.byref(st)))
        corners = np.empty((cnt.value, 8), np.uint32)
        tasks = np.empty(cnt.value, np.uint64)
        if cnt.value:
            _check(lib.amrx_comm_extract_dual(self._h, _ptr(corners), _ptr(tasks), cnt.value,
                                              C.byref(cnt), C.byref(st)))
        return DualMesh(corners, tasks, ExtractionStats._from(st))

    def close(self):
        if self._h:
            self._comm._lib.amrx_comm_index_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
