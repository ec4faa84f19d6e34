cd $GRAFT_REPO_ROOT
python tools/ingest_probe.py 1.0 > gpurun_out/sort_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"onesweep|rec_build|pack_kernel|prepass" -s 8 -c 8 -o gpurun_out/prof_sort python tools/ingest_probe.py 1.0 > gpurun_out/ncu_sort.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/sort_plain.log
