"""Tune the C4 brick generator: cells, level mix and triangles/cell for a
set of knob choices and iso values, plus first timings.  GPU only.

python tools/tune_c4.py --scale 0.5
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_08475_b200 as P  # noqa: E402
from paper_2004_08475_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.5, help="linear scale of the C4 brick grid")
    ap.add_argument("--isos", default="20,30,40,50")
    ap.add_argument("--knobs", default=None, help="json list of knob vectors")
    args = ap.parse_args()
    b3 = [max(1, int(round(x * args.scale))) for x in (512, 256, 256)]
    knob_sets = json.loads(args.knobs) if args.knobs else [synth.C4_KNOBS]
    for knobs in knob_sets:
        # scale tube radii with the domain so ratios carry over to full size
        k = list(knobs)
        k[1] *= args.scale
        k[2] *= args.scale
        t0 = time.time()
        ds = synth.bricks(b3, seed=1, shuffle=True, knobs=k, holes=synth.body_holes(b3))
        gen_s = time.time() - t0
        n = len(ds)
        torch.cuda.synchronize()
        t0 = time.time()
        idx = P.build_index(ds.cells, ds.scalars)
        torch.cuda.synchronize()
        build_s = time.time() - t0
        out = dict(knobs=knobs, bricks=b3, cells=n, level_cells=ds.level_cells,
                   gen_s=round(gen_s, 3), build_s=round(build_s, 3),
                   ingest_device_s=idx.info.seconds_ingest, key_bits=idx.info.key_bits,
                   dir_bits=idx.info.directory_bits)
        del ds
        for iso in [float(x) for x in args.isos.split(",")]:
            t0 = time.time()
            r = P.extract_isosurface(idx, P.IsoParams(iso=iso))
            wall = time.time() - t0
            s = r.stats
            out[f"iso{iso:g}"] = dict(tris=len(r.fat), tris_per_cell=len(r.fat) / n,
                                      duals=s.duals_accepted, kernel_s=s.seconds_pass1,
                                      wall_s=round(wall, 3))
        t0 = time.time()
        d = P.extract_dual_mesh(idx)
        out["dual"] = dict(duals=len(d), duals_per_cell=len(d) / n,
                           kernel_s=d.stats.seconds_pass1, wall_s=round(time.time() - t0, 3))
        print(json.dumps(out), flush=True)
        idx.close()


if __name__ == "__main__":
    main()
