"""Small end-to-end run of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run): golden cases through
build_index (shuffled input: pack + radix sort + scatter), every lookup
structure, extraction (dual + iso, several staging rounds), weld, validate,
point queries, a two-word-key dataset and the read_amr reader.

compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_08475_b200 as P  # noqa: E402


def main():
    z = np.load(os.path.join(ROOT, "tests", "golden", "cases.npz"))
    names = ["slots_l4_s3", "octree_sphere", "blocks_jump2"]
    for name in names:
        cells, scal, iso = z[name + "/in_cells"], z[name + "/in_scalars"], float(z[name + "/iso"])
        for lookup in (None, "hash", "directory"):
            idx = P.build_index(cells, scal, lookup=lookup)
            d = P.extract_dual_mesh(idx)
            r = P.extract_isosurface(idx, P.IsoParams(iso=iso))
            P.debug_round_limit(200)
            r2 = P.extract_isosurface(idx, P.IsoParams(iso=iso + 1e-3))
            P.debug_round_limit(0)
            assert len(d) == len(z[name + "/dual_corners"])
            assert r.fat.shape == z[name + "/fat"].shape
            rep = P.validate_dataset(idx)
            assert rep.ok()
            pts = idx.cells[::7, :3].astype(np.int64) + 1
            P.snap(idx, pts, 0)
            P.find_exact(idx, idx.cells[::5])
            P.try_build_duals(idx, np.arange(0, 8 * len(idx), 13, dtype=np.uint64))
            idx.close()
            del r2
        mesh = P.weld(r.fat)
        assert len(mesh.vertices) > 0
    # two-word keys
    c = z["octree_sphere/in_cells"].astype(np.int64)
    c2 = c + np.array([(1 << 30) - 64, (1 << 30) - 128, (1 << 30) - 192, 0])
    wc = np.concatenate([c, c2]).astype(np.int32)
    ws = np.concatenate([z["octree_sphere/in_scalars"]] * 2)
    widx = P.build_index(wc, ws)
    assert widx.info.lookup == "wide"
    P.extract_dual_mesh(widx)
    P.extract_isosurface(widx, 0.0)
    P.validate_dataset(widx)
    # the AMRCELL1 reader
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "c.amr")
        P.write_amr(path, z["slots_l4_s3/in_cells"], z["slots_l4_s3/in_scalars"])
        ridx = P.read_amr(path)
        P.extract_dual_mesh(ridx)
    print("sanitize probe ok")


if __name__ == "__main__":
    main()
