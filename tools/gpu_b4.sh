cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_weld_gpu.py tests/test_dropin_gpu.py -q -p no:cacheprovider -k "dual_cells or mesh or dropin or golden_case" 2>&1 | tail -3
for c in c2 c3; do python tools/dropin_bench.py $c $( [ $c = c3 ] && echo --no-ref ) > gpurun_out/dropin_$c.json 2>&1; cat gpurun_out/dropin_$c.json; done
python tools/dropin_bench.py c4 --no-ref --reps 1 > gpurun_out/dropin_c4.json 2>&1; cat gpurun_out/dropin_c4.json
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"; python tools/summ.py gpurun_out/bench_c4.json
