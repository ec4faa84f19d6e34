cd $GRAFT_REPO_ROOT
python -m pytest tests/test_weld_gpu.py tests/test_dropin_gpu.py tests/test_comm_gpu.py -q -p no:cacheprovider 2>&1 | tail -3
python tools/dropin_bench.py c2 > gpurun_out/dropin_c2.json 2>&1; cat gpurun_out/dropin_c2.json
python tools/dropin_bench.py c3 --no-ref --reps 2 > gpurun_out/dropin_c3.json 2>&1; cat gpurun_out/dropin_c3.json
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_c4.json
