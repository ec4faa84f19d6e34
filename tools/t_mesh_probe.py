import time, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_2004_08475_b200 as P
import bench
cells, scal, _ = bench.make_workload("c2", torch.device("cuda", 0))
c, s = cells.cpu().numpy(), scal.cpu().numpy()
idx = P.build_index(c, s)
for i in range(3):
    t = time.perf_counter(); m, st, tw = P.extract_isosurface_mesh(idx, 0.1); t1 = time.perf_counter() - t
    t = time.perf_counter(); d = P.extract_dual_mesh(idx); t2 = time.perf_counter() - t
    print(f"mesh {t1:.3f} s (weld {tw:.3f}, pass1 {st.seconds_pass1:.4f}) tris {len(m.triangles)} dual {t2:.3f}", flush=True)
