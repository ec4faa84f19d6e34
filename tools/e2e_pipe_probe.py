"""Timeline of the pipelined e2e (bench.e2e_single): when each build_index
and extract_isosurface of a stream of C4 steps starts and ends on the host,
with device memory in use -- python tools/e2e_pipe_probe.py [config] [steps]"""
import os
import queue
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2004_08475_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cells, scal, _ = bench.make_workload(cfg, torch.device("cuda", 0))
iso = bench.iso_of(cfg)
hc = torch.empty(cells.shape, dtype=torch.int32, pin_memory=True)
hs = torch.empty(scal.shape, dtype=torch.float64, pin_memory=True)
hc.copy_(cells)
hs.copy_(scal)
del cells, scal
torch.cuda.empty_cache()
probe = P.build_index(hc, hs)
nt = len(P.extract_isosurface(probe, P.IsoParams(iso=iso)).fat)
probe.close()
hout = torch.empty((int(nt * 1.05) + 1024, 9), dtype=torch.float64, pin_memory=True)
T0 = time.perf_counter()
log = []


def mark(what, t0):
    free, total = torch.cuda.mem_get_info()
    log.append((what, t0 - T0, time.perf_counter() - T0, (total - free) / 2**30))


def run(k):
    slots = threading.Semaphore(2)
    q = queue.Queue()

    def producer():
        for i in range(k):
            slots.acquire()
            t = time.perf_counter()
            ix = P.build_index(hc, hs)
            mark(f"build {i}", t)
            q.put(ix)
        q.put(None)

    th = threading.Thread(target=producer)
    th.start()
    i = 0
    while True:
        ix = q.get()
        if ix is None:
            break
        t = time.perf_counter()
        P.extract_isosurface(ix, P.IsoParams(iso=iso), out=hout)
        mark(f"extract {i}", t)
        ix.close()
        slots.release()
        i += 1
    th.join()


for s in range(2):
    log.clear()
    T0 = time.perf_counter()
    run(k)
    tot = time.perf_counter() - T0
    print(f"--- pass {s}: {k} steps in {tot:.3f} s = {1000 * tot / k:.1f} ms/step")
    for what, a, b, gb in log:
        print(f"{what:12s} {1000 * a:8.1f} -> {1000 * b:8.1f} ms ({1000 * (b - a):7.1f}) mem {gb:6.1f} GB")
# sequential for comparison
T0 = time.perf_counter()
for i in range(2):
    t = time.perf_counter()
    ix = P.build_index(hc, hs)
    mark("seq build", t)
    t = time.perf_counter()
    P.extract_isosurface(ix, P.IsoParams(iso=iso), out=hout)
    mark("seq extract", t)
    ix.close()
for what, a, b, gb in log[-4:]:
    print(f"{what:12s} {1000 * a:8.1f} -> {1000 * b:8.1f} ms ({1000 * (b - a):7.1f}) mem {gb:6.1f} GB")
