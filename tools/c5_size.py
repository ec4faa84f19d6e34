"""cell counts of candidate C5 shapes (GPU): python tools/c5_size.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2004_08475_b200 import synth  # noqa: E402

for b3, t0 in [((384, 192, 192), 0.45), ((384, 192, 192), 0.5), ((384, 192, 192), 0.55),
               ((352, 176, 176), 0.45), ((336, 168, 168), 0.40)]:
    k = list(synth.C4_KNOBS)
    k[4] = t0
    ds = synth.bricks(b3, seed=5, shuffle=False, knobs=k, holes=synth.body_holes(b3))
    print(b3, t0, len(ds), ds.level_cells, flush=True)
    del ds
    torch.cuda.empty_cache()
