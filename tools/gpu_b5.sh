cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_edge_gpu.py tests/test_rounds_gpu.py tests/test_deep_gpu.py tests/test_wide_gpu.py tests/test_dist_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
VARIANTS="libamrx_nc.so libamrx.so" CONFIGS="c4 c3 deep deep_thin c5 c2" bash tools/ab.sh
python tools/summ.py gpurun_out/ab_*.json
