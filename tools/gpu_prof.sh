cd $GRAFT_REPO_ROOT
CFG=${CFG:-c4}
python tools/profile_extract.py --config $CFG > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"extract_kernel" -c 1 -o gpurun_out/prof2_$CFG python tools/profile_extract.py --config $CFG > gpurun_out/ncu2_$CFG.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on --replay-mode application -k regex:"mc_jobs" -c 1 -o gpurun_out/prof2_mc_$CFG python tools/profile_extract.py --config $CFG > gpurun_out/ncu2_mc_$CFG.log 2>&1; echo ncu2 rc=$?
