"""The reference CLI's flow (read_amr -> validate_dataset ->
extract_isosurface -> extract_dual_mesh, proj/src/cli.cpp:76-118) through
the reference's C++ API: the GPU drop-in (oracle/_ref/amriso_dropin_bench,
the shim + libamrx.so) and the unmodified reference (amriso_ref_bench) on
the same AMRCELL1 file of a benchmark configuration.

python tools/dropin_bench.py c2 [--no-ref]   (GPU box; writes /tmp/<cfg>.amr)
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch
    import bench
    import paper_2004_08475_b200 as P
    cells, scal, _ = bench.make_workload(args.config, torch.device("cuda", 0))
    iso = bench.iso_of(args.config)
    path = f"/tmp/{args.config}.amr"
    P.write_amr(path, cells.cpu().numpy(), scal.cpu().numpy())
    n = cells.shape[0]
    del cells, scal
    torch.cuda.empty_cache()
    out = {"config": args.config, "cells": n, "iso": iso}
    for name, exe in (("dropin_gpu", "amriso_dropin_bench"), ("reference", "amriso_ref_bench")):
        if name == "reference" and args.no_ref:
            continue
        r = subprocess.run([os.path.join(ROOT, "oracle", "_ref", exe), path, str(iso),
                            str(args.reps)], capture_output=True, text=True)
        out[name] = json.loads(r.stdout) if r.returncode == 0 else {"error": r.stderr[-500:]}
    os.unlink(path)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
