"""Break down the host-buffer (e2e) path: build_index from pinned host arrays,
extract into a pinned host buffer.  GPU only.

python tools/e2e_probe.py [scale]          C4 bricks at a scale
python tools/e2e_probe.py --config NAME    a bench configuration"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_08475_b200 as P  # noqa: E402
from paper_2004_08475_b200 import synth  # noqa: E402


def main():
    iso = synth.C4_ISO
    if len(sys.argv) > 2 and sys.argv[1] == "--config":
        import bench
        cells, scal, _ = bench.make_workload(sys.argv[2], torch.device("cuda", 0))
        iso = bench.iso_of(sys.argv[2])
    else:
        scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
        b3 = [max(1, int(round(x * scale))) for x in (512, 256, 256)]
        k = list(synth.C4_KNOBS)
        k[1] *= scale
        k[2] *= scale
        ds = synth.bricks(b3, seed=1, shuffle=True, knobs=k, holes=synth.body_holes(b3))
        cells, scal = ds.cells, ds.scalars
    n = len(cells)
    hc = torch.empty(cells.shape, dtype=torch.int32, pin_memory=True)
    hs = torch.empty(scal.shape, dtype=torch.float64, pin_memory=True)
    hc.copy_(cells)
    hs.copy_(scal)
    t = time.perf_counter()
    torch.cuda.synchronize()
    probe = P.build_index(cells, scal)
    ntri = len(P.extract_isosurface(probe, P.IsoParams(iso=iso)).fat)
    probe.close()
    hout = torch.empty((int(ntri * 1.05) + 1024, 9), dtype=torch.float64, pin_memory=True)
    print(f"cells {n} tris {ntri} setup {time.perf_counter() - t:.2f}s", flush=True)
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ix = P.build_index(hc, hs)
        t1 = time.perf_counter()
        r = P.extract_isosurface(ix, P.IsoParams(iso=iso), out=hout)
        t2 = time.perf_counter()
        ix.close()
        t3 = time.perf_counter()
        print(f"rep {rep}: build {t1 - t0:.3f}s (device ingest {ix.info.seconds_ingest:.3f}) "
              f"extract {t2 - t1:.3f}s (kernel {r.stats.seconds_pass1:.3f} reorder "
              f"{r.stats.seconds_pass2:.3f}) close {t3 - t2:.3f}s", flush=True)
    # raw copy bandwidths for reference
    dev = torch.empty(hc.numel() * 4 // 8, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(hc.view(torch.float64).view(-1), non_blocking=True)
    torch.cuda.synchronize()
    h2d = hc.numel() * 4 / (time.perf_counter() - t0) / 1e9
    t0 = time.perf_counter()
    hc.view(torch.float64).view(-1).copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    d2h = hc.numel() * 4 / (time.perf_counter() - t0) / 1e9
    print(f"pinned copy bandwidth: H2D {h2d:.1f} GB/s, D2H {d2h:.1f} GB/s")
    print(torch.cuda.memory_summary(abbreviated=True)[:0])


if __name__ == "__main__":
    main()
