"""Randomised GPU-vs-reference sweep (not part of the pytest suite): datasets
from the reference's own generators (slots with level jumps up to 5, octrees
of several fields), shuffled, built on the GPU; the dual mesh, the fat soup
bits, the four counters and the welded mesh must equal the reference library's.

python tools/fuzz_parity.py [count] [seed0] [records|hash|directory]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2004_08475_b200 as P  # noqa: E402
import oracles  # noqa: E402


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    lookup = sys.argv[3] if len(sys.argv) > 3 else None  # forced lookup structure
    R = oracles.reference()
    kinds = ["sphere", "linear", "rsine"]
    bad = 0
    total_duals = total_tris = 0
    for s in range(seed0, seed0 + count):
        rng = np.random.default_rng(s)
        if s % 2:
            h = R.gen_slots(int(rng.integers(1, 1 << 30)), int(rng.integers(2, 9)),
                            int(rng.integers(1, 6)), float(rng.uniform(0, 0.4)))
            what = "slots"
        else:
            kind = kinds[int(rng.integers(0, len(kinds)))]
            depth = int(rng.integers(3, 7))
            side = float(1 << depth)
            params = np.concatenate([rng.uniform(0.1 * side, 0.9 * side, 3),
                                     [rng.uniform(0.1 * side, 0.5 * side)]])
            try:
                h = R.gen_octree(depth, kind, params, float(rng.uniform(0.5, 4)))
            except Exception:  # noqa: BLE001 - a field this generator rejects
                continue
            what = "octree-" + kind
        ds = R.dataset(h)
        cells, scal = ds.cells, ds.scalars
        perm = rng.permutation(len(cells))
        # an iso that ties with stored scalars half of the time (strict > rule)
        iso = float(scal[rng.integers(0, len(scal))]) if s % 4 < 2 else float(rng.normal())
        idx = P.build_index(cells[perm], scal[perm], lookup=lookup)
        d = P.extract_dual_mesh(idx)
        rd = R.extract_dual(h)
        r = P.extract_isosurface(idx, P.IsoParams(iso=iso))
        ri = R.extract_iso(h, iso)
        ok = d.corners.shape == rd["corners"].shape and (d.corners == rd["corners"]).all()
        ok &= r.fat.shape == ri["fat"].shape and (r.fat.view(np.uint64) == ri["fat"].view(np.uint64)).all()
        st = ri["stats"]
        ok &= [r.stats.duals_accepted, r.stats.duals_missing_corner, r.stats.duals_finer_corner,
               r.stats.duals_lower_key_corner] == [st["duals_accepted"], st["duals_missing_corner"],
                                                   st["duals_finer_corner"], st["duals_lower_key_corner"]]
        if len(r.fat):
            m = P.weld(r.fat)
            ok &= m.vertices.shape == ri["verts"].shape and \
                (np.ascontiguousarray(m.vertices).view(np.uint64) == ri["verts"].view(np.uint64)).all()
            ok &= (np.asarray(m.triangles).view(np.uint32) == ri["tris"]).all()
        idx.close()
        R.free(h)
        total_duals += len(d.corners)
        total_tris += len(r.fat)
        if not ok:
            bad += 1
            print(f"MISMATCH seed {s} {what} cells {len(cells)} iso {iso!r}", flush=True)
    print(f"{count} datasets from seed {seed0}: {total_duals} duals, {total_tris} triangles, "
          f"{bad} mismatching", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
