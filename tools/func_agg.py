"""Aggregate tools/sass_lines.py output by enclosing function (rough: by the
last function header above each line).  python tools/func_agg.py lines.txt extract.cu common.cuh"""
import re
import sys
from collections import defaultdict


def funcs(lines):
    starts = []
    for i, l in enumerate(lines):
        m = re.match(r'^(?:__device__|__global__|static __device__|template|__host__|[a-z_]+\().*?(\w+)\(', l)
        if m and not l.strip().endswith(';'):
            starts.append((i + 1, m.group(1)))
    return starts


def owner(starts, n):
    best = '?'
    for s, name in starts:
        if s <= n:
            best = name
    return best


rows = []
for ln in open(sys.argv[1]).read().splitlines()[1:]:
    m = re.match(r'\s*(\S+):(\d+)\s+inst\s+([\d.]+)%\s+stall\s+([\d.]+)%', ln)
    if m:
        rows.append((m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4))))
srcs = {}
for path in sys.argv[2:]:
    srcs[path.split('/')[-1].replace('_head', '')] = funcs(open(path).read().splitlines())
agg = defaultdict(lambda: [0.0, 0.0])
for f, n, i, s in rows:
    k = f + ':' + owner(srcs[f], n) if f in srcs else f
    agg[k][0] += i
    agg[k][1] += s
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:45} inst {v[0]:5.1f}  stall {v[1]:5.1f}")
