"""Join an ncu SASS source-page export with nvdisasm line info.

ncu -i rep --page source --csv --print-source sass > sass.csv
nvdisasm -g -c extract.sm_100a.cubin > dis.txt
python tools/sass_lines.py sass.csv dis.txt <function-substring> [top]
Prints instructions executed and stall samples per (file, line), inlined
call sites attributed to the innermost line.
"""
import csv
import re
import sys
from collections import defaultdict


def parse_dis(path, fun):
    addr2line = {}
    cur = None
    on = False
    for ln in open(path):
        if ln.startswith("//---") and ".text." in ln:
            on = fun in ln
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            addr2line[int(m.group(1), 16)] = cur
    return addr2line


def main():
    sass, dis, fun = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    a2l = parse_dis(dis, fun)
    lines = open(sass).read().splitlines()
    hdr_i = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(lines[hdr_i:]))
    base = None
    inst = defaultdict(float)
    stall = defaultdict(float)
    tot_i = tot_s = 0.0
    miss = 0
    for r in rows:
        try:
            a = int(r["Address"], 16)
        except ValueError:
            continue
        if base is None:
            base = a  # the export starts at the kernel entry
        a -= base
        ie = float(r["Instructions Executed"] or 0)
        ss = float(r["Warp Stall Sampling (All Samples)"] or 0)
        key = a2l.get(a)
        if key is None:
            miss += ie
            key = ("?", 0)
        inst[key] += ie
        stall[key] += ss
        tot_i += ie
        tot_s += ss
    print(f"total inst {tot_i:.3e}  stall samples {tot_s:.0f}  unmapped inst {miss:.3e}")
    for k in sorted(inst, key=lambda k: -inst[k])[:top]:
        print(f"{k[0]:>14}:{k[1]:<5} inst {100*inst[k]/tot_i:5.1f}%  stall {100*stall[k]/max(tot_s,1):5.1f}%")


if __name__ == "__main__":
    main()
