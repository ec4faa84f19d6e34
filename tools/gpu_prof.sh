cd $GRAFT_REPO_ROOT
CFG=${CFG:-c4}
python tools/profile_extract.py --config $CFG > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"extract_kernel|mc_jobs" -c 2 -o gpurun_out/prof_$CFG python tools/profile_extract.py --config $CFG > gpurun_out/ncu_$CFG.log 2>&1; echo ncu rc=$?
