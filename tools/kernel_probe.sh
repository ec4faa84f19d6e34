# launch durations (ncu, clocks unlocked) of the kernels matching KREGEX for
# library variants, one C4 build + extraction each:
# VARIANTS="libamrx.so libamrx_x.so" KREGEX="sign_bits|reorder" bash tools/kernel_probe.sh
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS}; do
  AMRX_LIB=$PWD/paper_2004_08475_b200/$v ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:"${KREGEX}" --csv --log-file gpurun_out/kp_${v%.so}.csv \
    python tools/profile_extract.py --config ${CFG:-c4} > /dev/null 2>&1
  echo "$v rc=$?"
done
