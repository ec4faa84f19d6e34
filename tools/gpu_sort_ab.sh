# ingest A/B over in-tree library variants (VARIANTS), C4 soup
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS}; do
  echo "$v: $(AMRX_LIB=$PWD/paper_2004_08475_b200/$v python tools/ingest_probe.py 1.0 2>&1 | tail -1)"
done
