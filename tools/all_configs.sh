#!/bin/bash
# run bench.py on every BASELINE configuration + the deep one (one GPU) and
# collect the lines: tools/all_configs.sh > gpurun_out/configs.jsonl
for c in c1 c2 c3 c4 c5 deep deep_thin; do
  python bench.py --config $c --steps 5 --warmup 3 2>/dev/null | tail -1
done
