# quick GPU round: the parity subset that exercises every lookup structure, then benches
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_deep_gpu.py tests/test_rounds_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -5
for cfg in ${CONFIGS:-c4 deep}; do
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err; echo "$cfg rc=$?"
done
for cfg in ${HASH_CONFIGS:-c3 c4}; do
  python bench.py --config $cfg --lookup hash --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_${cfg}_hash.json 2>&1; echo "${cfg}h rc=$?"
done
