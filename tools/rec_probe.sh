# record-build timing of library variants (ncu launch durations), C4 soup:
# VARIANTS="libamrx.so libamrx_x.so" bash tools/rec_probe.sh -> gpurun_out/rec_<variant>.csv
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS}; do
  AMRX_LIB=$PWD/paper_2004_08475_b200/$v ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_write.sum \
    -k regex:"rec_build|rec_tile" -s 2 -c 2 --csv --log-file gpurun_out/rec_${v%.so}.csv \
    python tools/ingest_probe.py 1.0 > /dev/null 2>&1
  echo "$v rc=$?"
done
