# full GPU verification: the suite on the product library, the checked
# library over the parity-heavy modules, debug counters of the big configs
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "suite rc=$?"; tail -25 gpurun_out/gpu_tests.log
AMRX_LIB=$PWD/paper_2004_08475_b200/libamrx_chk.so python tools/sanitize_probe.py 2>&1 | tail -1
AMRX_LIB=$PWD/paper_2004_08475_b200/libamrx_chk.so python -m pytest tests/test_dist_gpu.py tests/test_gpu_parity.py tests/test_wide_gpu.py tests/test_deep_gpu.py tests/test_rounds_gpu.py tests/test_edge_gpu.py tests/test_validate_gpu.py -q -p no:cacheprovider > gpurun_out/gpu_tests_checked.log 2>&1; echo "checked rc=$?"; tail -3 gpurun_out/gpu_tests_checked.log
for cfg in deep c4; do
AMRX_LIB=$PWD/paper_2004_08475_b200/libamrx_dbg.so AMRX_DEBUG_COUNTERS=1 python tools/profile_extract.py --config $cfg 2>&1 | tail -3
done
