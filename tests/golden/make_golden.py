"""Generate the committed golden vectors from the reference itself.

Runs the UNMODIFIED reference library (oracle/_ref/libamriso_ref.so, built by
`make -C oracle ref` from /root/reference/proj/src) and writes:

  sphere16.obj          extract_isosurface + obj_string on
                        gen_uniform(16, sphere(8,8,8;5)), iso 0 -- checked
                        byte-for-byte against the reference's own shipped
                        golden (proj/tests/golden/sphere16.obj) when present
  cases.npz             small datasets: the input cell list (generator order,
                        then shuffled), scalars, the reference's sorted
                        arrays, dual mesh (corners + owner*8+delta), the four
                        dual counters and the fat triangle soup (f64 bits)
  known_answers.json    aggregate counts for larger reference runs

Usage: python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracles  # noqa: E402

REF_GOLDEN = "/root/reference/proj/tests/golden/sphere16.obj"


def dataset_cases(R):
    """(name, handle, iso) for the committed small cases"""
    cases = []
    cases.append(("sphere8", R.gen_uniform(8, "sphere", [4, 4, 4, 2.5]), 0.0))
    cases.append(("octree_sphere", R.gen_octree(4, "sphere", [5, 6, 7, 3.5], 3.0), 0.0))
    cases.append(("slots_s11", R.gen_slots(11, 3, 2, 0.15), 0.1))
    cases.append(("slots_l4_s3", R.gen_slots(3, 3, 4, 0.15), 0.1))
    cases.append(("slots_l1_s11", R.gen_slots(11, 3, 1, 0.15), 0.0))
    blocks = [[0, 0, 0, 2, 4, 4, 2], [8, 0, 0, 8, 16, 16, 0]]
    holes = [[10, 3, 3, 13, 6, 6]]
    cases.append(("blocks_jump2", R.gen_blocks(blocks, "linear", [0.3, -0.2, 0.1, -1.0], holes), 0.0))
    # acceptance pool members with each generator kind
    for n in (0, 1, 2, 34, 101):
        h, iso = R.acceptance_fixture(n)
        cases.append((f"acceptance_{n}", h, iso))
    return cases


def main():
    R = oracles.reference()
    if R is None:
        raise SystemExit("oracle/_ref not built: run `make -C oracle ref` first")
    out = {}
    known = {}
    rng = np.random.default_rng(20261018)
    for name, h, iso in dataset_cases(R):
        ds = R.dataset(h)
        n = len(ds)
        perm = rng.permutation(n)
        # the shuffled list must rebuild to the identical index
        h2 = R.build(ds.cells[perm], ds.scalars[perm])
        ds2 = R.dataset(h2)
        assert (ds2.cells == ds.cells).all() and (ds2.scalars == ds.scalars).all()
        R.free(h2)
        duals = R.extract_dual(h, 1)
        res = R.extract_iso(h, iso, 1)
        st = res["stats"]
        tasks = duals["owner"].astype(np.uint64) * 8 + np.array(
            [int(np.nonzero([(duals["base"][i] == b).all() for b in _bases(ds.cells[o])])[0][0])
             for i, o in enumerate(duals["owner"])], np.uint64) if len(duals["owner"]) else np.zeros(0, np.uint64)
        out[f"{name}/in_cells"] = ds.cells[perm]
        out[f"{name}/in_scalars"] = ds.scalars[perm]
        out[f"{name}/cells"] = ds.cells
        out[f"{name}/scalars"] = ds.scalars
        out[f"{name}/levels"] = np.array(ds.levels, np.int32)
        out[f"{name}/bounds"] = ds.bounds
        out[f"{name}/iso"] = np.array(iso)
        out[f"{name}/dual_corners"] = duals["corners"]
        out[f"{name}/dual_tasks"] = tasks
        out[f"{name}/counters"] = np.array([st["duals_accepted"], st["duals_missing_corner"],
                                            st["duals_finer_corner"], st["duals_lower_key_corner"]],
                                           np.uint64)
        out[f"{name}/fat"] = res["fat"]
        known[name] = {k: v for k, v in st.items() if not k.startswith("seconds")}
        known[name]["duals"] = int(len(duals["corners"]))
        R.free(h)

    # the reference's own golden mesh
    h = R.gen_uniform(16, "sphere", [8, 8, 8, 5.0])
    obj = R.extract_iso(h, 0.0, 1, want_obj=True)["obj"]
    R.free(h)
    if os.path.exists(REF_GOLDEN):
        with open(REF_GOLDEN) as f:
            assert f.read() == obj, "reference output differs from its shipped golden"
    with open(os.path.join(HERE, "sphere16.obj"), "w") as f:
        f.write(obj)

    # larger known answers (aggregates only)
    big = [("octree7", R.gen_octree(7, "sphere", [50, 55, 60, 40.0], 3.2), 0.0),
           ("c1_octree6", R.gen_octree(6, "sphere", [25, 27.5, 30, 20.0], 3.2), 0.0),
           ("slots_l4_s6_n6", R.gen_slots(6, 6, 4, 0.15), 0.1)]
    for name, h, iso in big:
        res = R.extract_iso(h, iso, 0)
        d = R.extract_dual(h, 0)
        known[name] = {k: v for k, v in res["stats"].items() if not k.startswith("seconds")}
        known[name]["duals"] = int(len(d["corners"]))
        known[name]["fat_sum"] = float(np.sum(res["fat"]))
        R.free(h)
    # acceptance pool totals (acceptance.cpp:182-203, 260-284, 343-360)
    tot_d = tot_t = 0
    for n in range(102):
        h, iso = R.acceptance_fixture(n)
        tot_d += len(R.extract_dual(h, 1)["corners"])
        tot_t += R.extract_iso(h, iso, 1)["stats"]["fat_triangle_count"]
        R.free(h)
    known["acceptance_pool"] = {"datasets": 102, "duals": tot_d, "triangles": tot_t}

    np.savez_compressed(os.path.join(HERE, "cases.npz"), **out)
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(known, f, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays;", known["acceptance_pool"])


def _bases(c):
    w = 1 << int(c[3])
    return [np.array([c[0] - (0 if d & 1 else w), c[1] - (0 if d & 2 else w),
                      c[2] - (0 if d & 4 else w)]) for d in range(8)]


if __name__ == "__main__":
    main()
