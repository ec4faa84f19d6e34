# parity (all lookup structures + the general path) and an A/B of the regular-tile path
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_edge_gpu.py tests/test_rounds_gpu.py tests/test_deep_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -4
for cfg in ${CONFIGS:-c4 c3 c5}; do
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r_$cfg.json 2> gpurun_out/r_$cfg.err; echo "$cfg rc=$?"
  AMRX_NO_REGULAR=1 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g_$cfg.json 2> gpurun_out/g_$cfg.err; echo "$cfg general rc=$?"
done
