"""paper_2004_08475_b200 -- B200-native dual-mesh / iso-surface extraction
for structured AMR (arxiv 2004.08475), a drop-in for the reference amriso
hot path: AMR cell list in, dual cells and/or fat triangle soup out.

The compute path is libamrx.so (sm_100a CUDA behind the C ABI in
include/amrx.h).  This package is the Python mirror of the reference's
operator API (see amrx.py) plus the multi-GPU range partition (dist.py).
"""
from .amrx import (  # noqa: F401
    ACCEPTED, FINER_CORNER, LOWER_KEY_CORNER, MISSING_CORNER, MAX_LEVEL,
    CapacityError, CellIndex, CudaError, DualMesh, ExtractionResult,
    ExtractionStats, InternalError, IsoParams, LoadError, UnsupportedError,
    adopt_index, build_index, cell_bounds, dual_bases, extract_dual_mesh,
    extract_isosurface, find_exact, index_from_keys, kernel_launches, library, snap,
    debug_round_limit, Comm, CommIndex, device_count, extract_isosurface_mesh, extract_dual_cells,
    sort_part, try_build_duals, weld, IndexedMesh, validate_dataset, ValidationReport,
    release_cached_memory, read_amr, write_amr,
    write_obj, write_ply, write_dual_mesh,
)

__all__ = [
    "build_index", "find_exact", "snap", "try_build_duals", "extract_dual_mesh",
    "extract_isosurface", "IsoParams", "ExtractionStats", "ExtractionResult",
    "CellIndex", "DualMesh", "LoadError", "InternalError", "CapacityError",
    "UnsupportedError", "CudaError", "adopt_index", "dual_bases", "library",
    "cell_bounds", "sort_part", "index_from_keys", "weld", "IndexedMesh",
    "validate_dataset", "ValidationReport", "release_cached_memory",
    "read_amr", "write_amr", "write_obj", "write_ply", "write_dual_mesh",
]
