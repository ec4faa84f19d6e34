"""One build_index + one extraction of a scaled C4 workload, for ncu.

python tools/profile_extract.py --scale 0.5 [--dual]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_08475_b200 as P  # noqa: E402
from paper_2004_08475_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.5)
    ap.add_argument("--dual", action="store_true")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    b3 = [max(1, int(round(x * args.scale))) for x in (512, 256, 256)]
    k = list(synth.C4_KNOBS)
    k[1] *= args.scale
    k[2] *= args.scale
    ds = synth.bricks(b3, seed=1, shuffle=True, knobs=k, holes=synth.body_holes(b3))
    idx = P.build_index(ds.cells, ds.scalars)
    for _ in range(args.reps):
        if args.dual:
            r = P.extract_dual_mesh(idx)
            print("cells", len(ds), "duals", len(r), "kernel_s", r.stats.seconds_pass1)
        else:
            r = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO))
            print("cells", len(ds), "tris", len(r.fat), "kernel_s", r.stats.seconds_pass1,
                  "ingest_s", idx.info.seconds_ingest)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
