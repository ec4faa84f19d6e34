"""read_amr throughput: an AMRCELL1 file of a scaled C4 soup (page-cached
after the write) -> device index, against build_index from pinned host
arrays of the same data.  GPU only.

python tools/read_probe.py [scale] [dir]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_08475_b200 as P  # noqa: E402
from paper_2004_08475_b200 import synth  # noqa: E402


def main():
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
    d = sys.argv[2] if len(sys.argv) > 2 else "/tmp"
    b3 = [max(1, int(round(x * scale))) for x in (512, 256, 256)]
    k = list(synth.C4_KNOBS)
    k[1] *= scale
    k[2] *= scale
    ds = synth.bricks(b3, seed=1, shuffle=True, knobs=k, holes=synth.body_holes(b3))
    cells = ds.cells.cpu().numpy()
    scal = ds.scalars.cpu().numpy()
    del ds
    path = os.path.join(d, "probe.amr")
    P.write_amr(path, cells, scal)
    size = os.path.getsize(path)
    hc = torch.from_numpy(cells).pin_memory()
    hs = torch.from_numpy(scal).pin_memory()
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        a = P.read_amr(path)
        torch.cuda.synchronize()
        tr = time.perf_counter() - t
        t = time.perf_counter()
        b = P.build_index(hc, hs)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t
        print(f"cells {len(cells)} file {size / 1e9:.2f} GB read_amr {1000 * tr:.0f} ms "
              f"({size / tr / 1e9:.1f} GB/s) build_index(pinned host) {1000 * tb:.0f} ms")
        a.close()
        b.close()
    os.remove(path)


if __name__ == "__main__":
    main()
