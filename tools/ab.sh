# A/B of in-tree library variants on one box: VARIANTS="libamrx.so libamrx_x.so" CONFIGS="c4 deep"
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-libamrx.so}; do
  for cfg in ${CONFIGS:-c4}; do
    AMRX_LIB=$PWD/paper_2004_08475_b200/$v python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/ab_${v%.so}_$cfg.json 2> gpurun_out/ab_${v%.so}_$cfg.err
    echo "$v $cfg rc=$?"
  done
done
