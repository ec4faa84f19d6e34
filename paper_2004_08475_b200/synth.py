"""Synthetic AMR inputs for tests and the benchmark (libamrx_synth.so).

Small configurations reproduce the reference's own generators record for
record (host C++, same libstdc++ <random>): ``octree_sphere`` = gen_octree
with a sphere field (proj/src/synth.cpp:141-181), ``uniform_sphere`` =
gen_uniform (synth.cpp:122-137), ``slots`` = random_slot_dataset
(proj/tests/fixtures.hpp:38-69).  They return the generator's record order,
i.e. the cell list a caller hands to build_index.

``bricks`` is the GPU generator for the large configurations (SURVEY §8(d)
C4/C5): a 4-level block-structured AMR around Gaussian vortex tubes with
"aircraft body" holes and a vorticity-magnitude scalar, optionally in a
bijective-hash "soup" order.  Its arrays stay on the device.

Config registry: ``CONFIGS`` names every BASELINE.json configuration.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libamrx_synth.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make -C {_HERE}`")
        L = C.CDLL(LIB_PATH)
        P, U64, D, I32 = C.c_void_p, C.c_uint64, C.c_double, C.c_int32
        L.amrxs_octree_sphere.restype = P
        L.amrxs_octree_sphere.argtypes = [I32, D, D, D, D, D]
        L.amrxs_uniform_sphere.restype = P
        L.amrxs_uniform_sphere.argtypes = [I32, D, D, D, D]
        L.amrxs_slots.restype = P
        L.amrxs_slots.argtypes = [C.c_uint32, C.c_int, C.c_int, D]
        L.amrxs_size.restype = U64
        L.amrxs_size.argtypes = [P]
        L.amrxs_get.argtypes = [P, P, P]
        L.amrxs_free.argtypes = [P]
        L.amrxs_bricks.restype = C.c_int
        L.amrxs_bricks.argtypes = [P, U64, C.c_int, P, C.c_int, P, P, P, P, P]
        L.amrxs_device_free.argtypes = [P]
        L.amrxs_memcpy.restype = C.c_int
        L.amrxs_memcpy.argtypes = [P, P, U64]
        _lib = L
    return _lib


def _take(h):
    L = lib()
    n = L.amrxs_size(h)
    cells = np.empty((n, 4), np.int32)
    scal = np.empty(n, np.float64)
    L.amrxs_get(h, cells.ctypes.data_as(C.c_void_p), scal.ctypes.data_as(C.c_void_p))
    L.amrxs_free(h)
    return cells, scal


def octree_sphere(depth, centre, radius, threshold):
    return _take(lib().amrxs_octree_sphere(depth, *map(float, centre), float(radius),
                                           float(threshold)))


def uniform_sphere(n, centre, radius):
    return _take(lib().amrxs_uniform_sphere(n, *map(float, centre), float(radius)))


def slots(seed, n_slots, max_level, hole_prob=0.15):
    return _take(lib().amrxs_slots(seed, n_slots, max_level, hole_prob))


class DeviceDataset:
    """cells (n,4) int32 and scalars (n,) f64 as torch CUDA tensors."""

    def __init__(self, cells, scalars, level_cells, ptrs):
        self.cells = cells
        self.scalars = scalars
        self.level_cells = level_cells
        self._ptrs = ptrs

    def __len__(self):
        return self.cells.shape[0]


def bricks(bricks3, seed=1, shuffle=True, knobs=None, holes=()):
    """Generate on the current CUDA device; returns torch tensors that own
    copies of the generated arrays (the raw buffers are freed)."""
    import torch
    L = lib()
    if knobs is None:
        knobs = C4_KNOBS
    b3 = np.asarray(bricks3, np.int32)
    k8 = np.asarray(knobs, np.float64)
    ho = np.ascontiguousarray(np.asarray(holes, np.int64).reshape(-1, 6))
    cp, sp, n = C.c_void_p(), C.c_void_p(), C.c_uint64()
    lc = np.zeros(4, np.uint64)
    rc = L.amrxs_bricks(b3.ctypes.data_as(C.c_void_p), seed, int(shuffle),
                        k8.ctypes.data_as(C.c_void_p), len(ho),
                        ho.ctypes.data_as(C.c_void_p) if len(ho) else None,
                        C.byref(cp), C.byref(sp), C.byref(n),
                        lc.ctypes.data_as(C.c_void_p))
    if rc != 0:
        raise RuntimeError(f"amrxs_bricks failed ({rc})")
    nn = n.value
    cells = torch.empty((nn, 4), dtype=torch.int32, device="cuda")
    scal = torch.empty(nn, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    if L.amrxs_memcpy(C.c_void_p(cells.data_ptr()), cp, nn * 16) or \
            L.amrxs_memcpy(C.c_void_p(scal.data_ptr()), sp, nn * 8):
        raise RuntimeError("amrxs_memcpy failed")
    L.amrxs_device_free(cp)
    L.amrxs_device_free(sp)
    return DeviceDataset(cells, scal, [int(x) for x in lc], None)


# knobs: ntubes, core radius min, max, indicator reach (core radii), level
# thresholds t0 t1 t2, noise amplitude
C4_KNOBS = [14, 24.0, 48.0, 1.41, 0.30, 0.08, 0.01, 8.0]
C4_ISO = 4.0
# C5: the same field with a narrower level-0 band (t0 0.53): 250M cells
C5_KNOBS = [14, 24.0, 48.0, 1.41, 0.53, 0.08, 0.01, 8.0]

# "aircraft body": fuselage + wing boxes (finest units), scaled to the domain
def body_holes(bricks3):
    X, Y, Z = (8 * b for b in bricks3)
    fus = [int(0.10 * X), int(0.46 * Y), int(0.46 * Z), int(0.55 * X), int(0.54 * Y), int(0.54 * Z)]
    wing = [int(0.28 * X), int(0.20 * Y), int(0.49 * Z), int(0.38 * X), int(0.80 * Y), int(0.51 * Z)]
    return [fus, wing]


def value_noise(p, seed, octaves=5, base=0.02):
    """fixed-seed fractal value noise at FP64 positions p (n, 3): per octave
    a lattice of pseudo-random values in [-1, 1) from an integer hash of the
    lattice point, blended trilinearly with smoothstep weights; octave o has
    frequency base * 2^o and amplitude 2^-o (hashed-lattice
    value noise, >= 5 octaves, FP64 evaluation)"""
    import torch
    f = torch.zeros(len(p), dtype=torch.float64, device=p.device)
    amp, freq = 1.0, base
    for o in range(octaves):
        q = p * freq
        i0 = torch.floor(q)
        t = q - i0
        s = t * t * (3.0 - 2.0 * t)
        i0 = i0.to(torch.int64)
        v = torch.zeros_like(f)
        for d in range(8):
            dx, dy, dz = d & 1, (d >> 1) & 1, (d >> 2) & 1
            h = ((i0[:, 0] + dx) * 73856093) ^ ((i0[:, 1] + dy) * 19349663) ^ \
                ((i0[:, 2] + dz) * 83492791) ^ ((seed * 131 + o) * 2654435761)
            h = h ^ (h >> 13)
            h = h * 0x5BD1E995
            h = h ^ (h >> 15)
            lat = (h & 0xFFFFFF).to(torch.float64) / float(1 << 23) - 1.0
            w = (s[:, 0] if dx else 1.0 - s[:, 0]) * (s[:, 1] if dy else 1.0 - s[:, 1]) * \
                (s[:, 2] if dz else 1.0 - s[:, 2])
            v += w * lat
        f += amp * v
        amp *= 0.5
        freq *= 2.0
    return f


def octree_noise(root=(48, 48, 48), levels=6, seed=3, k=0.45, base=0.02, shuffle=True,
                 device="cuda", octaves=5):
    """C3: a 6-level octree (levels 0..levels-1) over a root grid of
    coarsest cells, refined toward the zero set of a turbulent field --
    fixed-seed hashed-lattice value noise, `octaves` octaves (value_noise) --
    a cell being split while |f(centre)| < k w base; the field at the cell
    centre is the scalar (iso 0 = its median by symmetry); optionally
    shuffled into a soup.  Built with torch on the GPU (no reference
    counterpart: the reference's own generators are CPU, synth.cpp).
    Returns (cells int32[n,4], scalars f64[n]) on `device`."""
    import torch
    L = levels - 1
    W = 1 << L
    r = [torch.arange(n, device=device, dtype=torch.int64) * W for n in root]
    cur = torch.stack(torch.meshgrid(*r, indexing="ij"), -1).reshape(-1, 3)
    off = torch.tensor([[(d >> 0) & 1, (d >> 1) & 1, (d >> 2) & 1] for d in range(8)],
                       device=device, dtype=torch.int64)
    cells, scal = [], []
    while True:
        w = 1 << L
        f = value_noise(cur.to(torch.float64) + 0.5 * w, seed, octaves, base)
        refine = (f.abs() < k * w * base) if L > 0 else torch.zeros_like(f, dtype=torch.bool)
        keep = ~refine
        cells.append(torch.cat([cur[keep], torch.full((int(keep.sum()), 1), L, device=device,
                                                      dtype=torch.int64)], 1).to(torch.int32))
        scal.append(f[keep])
        if L == 0 or not bool(refine.any()):
            break
        cur = (cur[refine][:, None, :] + off[None] * (w // 2)).reshape(-1, 3)
        L -= 1
    cells = torch.cat(cells)
    scal = torch.cat(scal)
    if shuffle:
        gp = torch.Generator(device=device).manual_seed(seed)
        perm = torch.randperm(len(cells), device=device, generator=gp)
        cells, scal = cells[perm].contiguous(), scal[perm].contiguous()
    return cells, scal


def landing_gear_sdf(c, scale, size=1.0):
    """signed distance (finest units, FP64) to a landing-gear-like body: a
    main strut, a side brace, an axle and two wheels (tori) -- the shape
    class of the paper's 13-level NASA landing gear.
    ``scale`` = the domain's finest-unit extent along y."""
    import torch
    S = float(scale)
    x, y, z = c[:, 0], c[:, 1], c[:, 2]
    # the body scaled by `size` about the domain's centre line
    x = 0.5 * S + (x - 0.5 * S) / size
    y = 0.5 * S + (y - 0.5 * S) / size
    z = 0.5 * S + (z - 0.5 * S) / size

    def capsule(ax, ay, az, bx, by, bz, r):
        px, py, pz = x - ax, y - ay, z - az
        dx, dy, dz = bx - ax, by - ay, bz - az
        h = ((px * dx + py * dy + pz * dz) / (dx * dx + dy * dy + dz * dz)).clamp(0.0, 1.0)
        return torch.sqrt((px - h * dx) ** 2 + (py - h * dy) ** 2 + (pz - h * dz) ** 2) - r

    def torus_y(cx, cy, cz, R, r):  # axis along y
        q = torch.sqrt((x - cx) ** 2 + (z - cz) ** 2) - R
        return torch.sqrt(q * q + (y - cy) ** 2) - r

    cx, cy = 0.5 * S, 0.5 * S
    d = capsule(cx, cy, 0.62 * S, cx, cy, 0.30 * S, 0.035 * S)           # strut
    d = torch.minimum(d, capsule(cx, cy, 0.55 * S, cx + 0.16 * S, cy, 0.78 * S, 0.018 * S))
    d = torch.minimum(d, capsule(cx, cy - 0.17 * S, 0.30 * S, cx, cy + 0.17 * S, 0.30 * S,
                                 0.022 * S))                             # axle
    for sy in (-0.15, 0.15):                                             # wheels
        d = torch.minimum(d, torus_y(cx, cy + sy * S, 0.30 * S, 0.10 * S, 0.045 * S))
    return d * size


def octree_sdf(root=(3, 2, 2), levels=13, k=0.9, seed=13, shuffle=True, device="cuda",
               noise=0.0, size=1.0):
    """DEEP config: an octree of `levels` levels (0..levels-1) over a root
    grid of coarsest cells, refined toward a landing-gear surface
    (landing_gear_sdf) -- a cell is split while its centre lies within k
    cell widths of the surface -- with the signed distance (plus optional
    value noise) at the cell centre as the scalar, iso 0.  Built with torch
    on the GPU; optionally shuffled into a soup.  Returns (cells int32[n,4],
    scalars f64[n]) on `device`."""
    import torch
    L = levels - 1
    W = 1 << L
    scale = root[1] * W
    r = [torch.arange(n, device=device, dtype=torch.int64) * W for n in root]
    cur = torch.stack(torch.meshgrid(*r, indexing="ij"), -1).reshape(-1, 3)
    off = torch.tensor([[(d >> 0) & 1, (d >> 1) & 1, (d >> 2) & 1] for d in range(8)],
                       device=device, dtype=torch.int64)
    g = torch.Generator(device="cpu").manual_seed(seed)
    ph = (torch.rand(3, generator=g, dtype=torch.float64) * 6.283185307179586).tolist()
    cells, scal = [], []
    while True:
        w = 1 << L
        ctr = cur.to(torch.float64) + 0.5 * w
        f = landing_gear_sdf(ctr, scale, size)
        if noise:
            f = f + noise * torch.sin(ctr[:, 0] * 0.013 + ph[0]) * \
                torch.sin(ctr[:, 1] * 0.011 + ph[1]) * torch.sin(ctr[:, 2] * 0.017 + ph[2])
        refine = (f.abs() < k * w) if L > 0 else torch.zeros_like(f, dtype=torch.bool)
        keep = ~refine
        cells.append(torch.cat([cur[keep], torch.full((int(keep.sum()), 1), L, device=device,
                                                      dtype=torch.int64)], 1).to(torch.int32))
        scal.append(f[keep])
        if L == 0 or not bool(refine.any()):
            break
        cur = (cur[refine][:, None, :] + off[None] * (w // 2)).reshape(-1, 3)
        L -= 1
    cells = torch.cat(cells)
    scal = torch.cat(scal)
    if shuffle:
        gp = torch.Generator(device=device).manual_seed(seed)
        perm = torch.randperm(len(cells), device=device, generator=gp)
        cells, scal = cells[perm].contiguous(), scal[perm].contiguous()
    return cells, scal


CONFIGS = {
    # C1: SURVEY §8(d): gen_octree(6, sphere((25,27.5,30), 20), 3.2), iso 0
    "c1": dict(kind="octree_sphere", args=(6, (25.0, 27.5, 30.0), 20.0, 3.2), iso=0.0),
    # C2: random_slot_dataset(mt19937(seed), 23, 4, 0.15), iso 0.1
    "c2": dict(kind="slots", args=(2026, 23, 4, 0.15), iso=0.1),
    # C3: ~100M-cell 6-level octree refined toward the zero set of 5-octave
    # hashed-lattice value noise, the noise as scalar, iso 0 (its median by
    # symmetry) (GPU generator, soup order)
    "c3": dict(kind="octree_noise", args=((48, 48, 48), 6, 3, 0.7), iso=0.0),
    # C4: 626M-cell 4-level soup (bricks 512 x 256 x 256 -> tuned knobs)
    "c4": dict(kind="bricks", bricks=(512, 256, 256), seed=1, shuffle=True, iso=None),
    # C5: ~250M-cell mixed-level AMR, dual mesh only
    "c5": dict(kind="bricks", bricks=(384, 192, 192), seed=5, shuffle=False, iso=None,
               dual_only=True, knobs=C5_KNOBS),
    # DEEP: a 13-level octree (levels 0..12) refined toward a landing-gear
    # surface (the paper's 13-level NASA landing gear shape class), soup
    # order, iso 0 on the signed distance -- a sparse 44-bit key space; a
    # cell splits within 2 widths of the surface (AMR codes keep a buffer of
    # a few cells per level band)
    "deep": dict(kind="octree_sdf", args=((6, 4, 4), 13, 2.0), kwargs=dict(size=0.335), iso=0.0),
    # the same with a one-cell band per level (k = 0.9): nearly every cell
    # at a level transition -- the lookup stress case
    "deep_thin": dict(kind="octree_sdf", args=((3, 2, 2), 13, 0.9), iso=0.0),
}
