#!/bin/bash
# A/B harness: tools/ab.sh "label|LIBTAG|ENV=..." ...   (run on the GPU box)
# prints the best of 2 runs of the iso and dual-only extraction kernels on C4
for spec in "$@"; do
  IFS='|' read -r label tag envs <<< "$spec"
  if [ -n "$tag" ]; then lib="AMRX_LIB=$PWD/paper_2004_08475_b200/libamrx_$tag.so"; else lib=""; fi
  best_i=9; best_d=9
  for rep in 1 2; do
    ti=$(env $lib $envs python tools/profile_extract.py --scale ${SCALE:-1.0} | awk '{print $6}')
    td=$(env $lib $envs python tools/profile_extract.py --scale ${SCALE:-1.0} --dual | awk '{print $6}')
    best_i=$(python -c "print(min($best_i,$ti))"); best_d=$(python -c "print(min($best_d,$td))")
  done
  echo "$label iso_ms=$(python -c "print(round($best_i*1000,1))") dual_ms=$(python -c "print(round($best_d*1000,1))")"
done
