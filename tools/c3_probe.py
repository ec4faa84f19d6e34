import sys, time, torch
sys.path.insert(0, '.')
from paper_2004_08475_b200 import synth
for k in [float(x) for x in sys.argv[1:]]:
    t=time.time(); c, s = synth.octree_noise(k=k); torch.cuda.synchronize()
    lv = torch.bincount(c[:,3].long()).tolist()
    print(k, len(c), lv, f"{time.time()-t:.1f}s", flush=True)
    del c, s; torch.cuda.empty_cache()
