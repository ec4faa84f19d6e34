"""GPU weld timing on the C4 soup (device-resident triangles).

python tools/weld_probe.py [scale]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_08475_b200 as P  # noqa: E402
from paper_2004_08475_b200 import synth  # noqa: E402


def main():
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    b3 = [max(1, int(round(x * scale))) for x in (512, 256, 256)]
    k = list(synth.C4_KNOBS)
    k[1] *= scale
    k[2] *= scale
    ds = synth.bricks(b3, seed=1, shuffle=True, knobs=k, holes=synth.body_holes(b3))
    idx = P.build_index(ds.cells, ds.scalars)
    r = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO))
    n = len(r.fat)
    fat = torch.empty((n, 9), dtype=torch.float64, device="cuda")
    r2 = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO), out=fat)
    idx.close()
    del ds, r
    verts = torch.empty((3 * n, 3), dtype=torch.float64, device="cuda")
    tris = torch.empty((n, 3), dtype=torch.int32, device="cuda")
    lib = P.library()
    import ctypes as C
    nv = C.c_uint64()
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = lib.amrx_weld(C.c_void_p(fat.data_ptr()), n, C.c_void_p(verts.data_ptr()), 3 * n,
                           C.c_void_p(tris.data_ptr()), C.byref(nv), None)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        assert st == 0, lib.amrx_last_error()
        v = verts[:nv.value].contiguous().view(torch.int64)
        chk = (int(v.sum()), int((v * torch.arange(1, nv.value + 1, device="cuda")[:, None]).sum()),
               int((tris.to(torch.int64) * torch.arange(1, n + 1, device="cuda")[:, None]).sum()))
        print(f"weld {n} triangles -> {nv.value} vertices: {1000 * dt:.1f} ms  checksum {chk}",
              flush=True)


if __name__ == "__main__":
    main()
