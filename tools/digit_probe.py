"""Per radix pass digit statistics of a benchmark configuration's keys (for
choosing the ranking per pass): largest digit share, the mean number of lanes
of a 32-lane warp sharing a lane's digit in the pass's input order (sorted by
the lower digits) and from the global histogram.  GPU only.

python tools/digit_probe.py c5 deep c4
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2004_08475_b200 as P  # noqa: E402
from paper_2004_08475_b200 import dist as D  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for cfg in sys.argv[1:] or ["c4"]:
        cells, scal, _ = bench.make_workload(cfg, dev)
        ix = P.build_index(cells, scal)
        keys, _ = D.sorted_arrays(ix, dev)
        bits = ix.info.key_bits if hasattr(ix.info, "key_bits") else 64
        k = keys.clone()
        ix.close()
        del cells, scal
        passes = (int(bits) + 8) // 9
        for p in range(passes):
            d = ((k >> (9 * p)) & 511)
            h = torch.bincount(d, minlength=512).double()
            q = h / h.sum()
            glob = 1 + 31 * float((q * q).sum())
            # the pass's input order: sorted by the digits below p (stable),
            # i.e. by (key mod 2^(9p)); original order within ties unknown
            # here, approximate with the sorted order of the low bits
            if p:
                low = k & ((1 << (9 * p)) - 1)
                order = torch.sort(low, stable=True).indices
                dd = d[order]
            else:
                dd = d  # first pass: the input order is the (shuffled) soup: use a random sample
                dd = dd[torch.randperm(len(dd), device=dev)]
            n = (len(dd) // 32) * 32
            w = dd[:n].view(-1, 32)
            w = w[torch.randperm(w.shape[0], device=dev)[: 1 << 20]]  # a sample of warps
            same = (w.unsqueeze(2) == w.unsqueeze(1)).sum(2).double().mean().item()
            print(f"{cfg} pass {p}: max share {float(q.max()):.3f}  lanes sharing a digit: "
                  f"in order {same:.2f}, from histogram {glob:.2f}")
        del k, keys
        torch.cuda.empty_cache()
        P.release_cached_memory()


if __name__ == "__main__":
    main()
