cd $GRAFT_REPO_ROOT
for cfg in ${CONFIGS:-c4}; do
AMRX_LIB=$PWD/paper_2004_08475_b200/libamrx_dbg.so AMRX_DEBUG_COUNTERS=1 python tools/profile_extract.py --config $cfg 2>&1 | tail -3
done
