"""Steady-state ingest (pack + radix sort + gather + directory) timing on a
scaled C4 soup, device-resident input.  GPU only.

python tools/ingest_probe.py [scale]
"""
import os
import sys

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
    times = []
    for rep in range(5):
        idx = P.build_index(ds.cells, ds.scalars)
        times.append(idx.info.seconds_ingest)
        idx.close()
    torch.cuda.synchronize()
    print(f"cells {len(ds)} ingest_ms " + " ".join(f"{1000 * t:.1f}" for t in times)
          + f" best {1000 * min(times[1:]):.1f}")


if __name__ == "__main__":
    main()
