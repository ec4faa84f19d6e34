"""One build_index + one extraction of a benchmark configuration, for ncu
and the debug counters (AMRX_LIB=.../libamrx_dbg.so AMRX_DEBUG_COUNTERS=1).

python tools/profile_extract.py --config deep [--lookup hash] [--dual] [--scale 0.5]
(--scale applies to the c4 bricks only)
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_08475_b200 as P  # noqa: E402
from paper_2004_08475_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--lookup", default=None)
    ap.add_argument("--dual", action="store_true")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    if args.config == "c4" and args.scale != 1.0:
        b3 = [max(1, int(round(x * args.scale))) for x in (512, 256, 256)]
        k = list(synth.C4_KNOBS)
        k[1] *= args.scale
        k[2] *= args.scale
        ds = synth.bricks(b3, seed=1, shuffle=True, knobs=k, holes=synth.body_holes(b3))
        cells, scal, iso = ds.cells, ds.scalars, synth.C4_ISO
    else:
        sys.path.insert(0, ROOT)
        import bench
        cells, scal, _ = bench.make_workload(args.config, torch.device("cuda", 0))
        iso = bench.iso_of(args.config)
    idx = P.build_index(cells, scal, lookup=args.lookup)
    print("index", idx.info.lookup, idx.info.key_bits, "bits, max probe", idx.info.max_probe,
          "entries", idx.info.lookup_entries, "ingest_s", idx.info.seconds_ingest)
    for _ in range(args.reps):
        if args.dual:
            r = P.extract_dual_mesh(idx)
            print("cells", len(cells), "duals", len(r), "kernel_s", r.stats.seconds_pass1)
        else:
            r = P.extract_isosurface(idx, P.IsoParams(iso=iso))
            print("cells", len(cells), "tris", len(r.fat), "kernel_s", r.stats.seconds_pass1,
                  "launches", r.stats.kernel_launches)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
