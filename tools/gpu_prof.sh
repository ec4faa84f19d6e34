cd $GRAFT_REPO_ROOT
AMRX_LIB=$PWD/paper_2004_08475_b200/libamrx_dbg.so AMRX_DEBUG_COUNTERS=1 python tools/profile_extract.py --config deep 2>&1 | tail -4
AMRX_LIB=$PWD/paper_2004_08475_b200/libamrx_dbg.so AMRX_DEBUG_COUNTERS=1 python tools/profile_extract.py --config c4 2>&1 | tail -4
python tools/profile_extract.py --config deep > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:extract_kernel -c 1 -o gpurun_out/prof_deep python tools/profile_extract.py --config deep > gpurun_out/ncu_deep.log 2>&1; echo ncu rc=$?
