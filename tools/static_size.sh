#!/bin/bash
# tools/static_size.sh [lib] [kernel-substring]: SASS instruction count of a
# kernel by enclosing source function (nvdisasm line info)
LIB=${1:-paper_2004_08475_b200/libamrx.so}; K=${2:-extract_kernelILb0ELb1ELb0E}
D=$(mktemp -d); (cd $D && cuobjdump -xelf all $OLDPWD/$LIB >/dev/null)
nvdisasm -g -c $D/extract.sm_100a.cubin 2>/dev/null | awk -v k="$K" '/^\.text\./{on=index($0,k)>0} on' |
  awk '/\/\/## File/{split($0,a,"\""); f=a[2]; sub(/.*\//,"",f); match($0,/line [0-9]+/); l=substr($0,RSTART+5,RLENGTH-5)} /\/\*[0-9a-f]+\*\//{print f":"l}' > $D/lines.txt
wc -l < $D/lines.txt
python3 - $D/lines.txt <<'PY'
import re, sys, collections
src = {'extract.cu': 'paper_2004_08475_b200/csrc/extract.cu', 'common.cuh': 'paper_2004_08475_b200/csrc/common.cuh'}
def funcs(path):
    st = []
    for i, l in enumerate(open(path).read().splitlines()):
        m = re.match(r'^(?:__device__|__global__|static __device__|template|__host__|[a-z_]+\().*?(\w+)\(', l)
        if m and not l.strip().endswith(';'): st.append((i + 1, m.group(1)))
    return st
F = {k: funcs(v) for k, v in src.items()}
cnt = collections.Counter()
for ln in open(sys.argv[1]):
    f, l = ln.strip().rsplit(':', 1)
    l = int(l) if l else 0
    name = f
    if f in F:
        for s, nm in F[f]:
            if s <= l: name = f + ':' + nm
    cnt[name] += 1
for k, v in cnt.most_common(20): print(v, k)
PY
rm -rf $D
