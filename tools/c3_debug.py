import sys, torch
sys.path.insert(0, '.')
import paper_2004_08475_b200 as P
from paper_2004_08475_b200 import synth
root = tuple(int(x) for x in sys.argv[1].split(',')) if len(sys.argv) > 1 else (12, 12, 12)
c, s = synth.octree_noise(root=root)
print("cells", len(c), torch.bincount(c[:,3].long()).tolist(), flush=True)
idx = P.build_index(c, s)
print("levels", idx.levels, idx.info.key_bits, idx.info.directory_bits, flush=True)
d = P.extract_dual_mesh(idx)
print("duals", len(d.corners), flush=True)
r = P.extract_isosurface(idx, P.IsoParams(iso=0.0))
print("tris", len(r.fat), flush=True)
