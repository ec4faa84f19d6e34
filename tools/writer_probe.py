"""OBJ / PLY writer throughput on a welded scaled-C4 mesh: amrx_write_* (host
threads) against the reference's write_obj / write_ply (oracle/_ref), bytes
compared.  python tools/writer_probe.py [scale] [dir]"""
import filecmp
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2004_08475_b200 as P  # noqa: E402
from paper_2004_08475_b200 import synth  # noqa: E402
import oracles  # noqa: E402


def main():
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
    d = sys.argv[2] if len(sys.argv) > 2 else "/tmp"
    b3 = [max(1, int(round(x * scale))) for x in (512, 256, 256)]
    k = list(synth.C4_KNOBS)
    k[1] *= scale
    k[2] *= scale
    ds = synth.bricks(b3, seed=1, shuffle=True, knobs=k, holes=synth.body_holes(b3))
    idx = P.build_index(ds.cells, ds.scalars)
    r = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO))
    mesh = P.weld(r.fat)
    v = np.ascontiguousarray(np.asarray(mesh.vertices.cpu() if hasattr(mesh.vertices, "cpu") else mesh.vertices, np.float64))
    t = np.ascontiguousarray(np.asarray(mesh.triangles.cpu() if hasattr(mesh.triangles, "cpu") else mesh.triangles).view(np.uint32))
    m = type("M", (), {})()
    m.vertices, m.triangles = v, t
    R = oracles.reference()
    for ply in (0, 1):
        a, b = os.path.join(d, f"mine{ply}"), os.path.join(d, f"ref{ply}")
        t0 = time.perf_counter()
        (P.write_ply if ply else P.write_obj)(a, m)
        t1 = time.perf_counter()
        rc = R.lib.ref_write_mesh(os.fsencode(b), ply, oracles._ptr(v), len(v), oracles._ptr(t), len(t)) if R else -1
        t2 = time.perf_counter()
        same = filecmp.cmp(a, b, shallow=False) if R else None
        print(f"{'ply' if ply else 'obj'}: {len(v)} vertices {len(t)} triangles "
              f"{os.path.getsize(a) / 1e9:.2f} GB  amrx {1000 * (t1 - t0):.0f} ms  "
              f"reference {1000 * (t2 - t1):.0f} ms  identical {same}")
        for f in (a, b):
            if os.path.exists(f):
                os.remove(f)


if __name__ == "__main__":
    main()
