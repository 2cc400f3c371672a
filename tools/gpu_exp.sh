# Quick experiment round on one GPU: build, kernel times (forward / back) and MLEM us/iteration for the
# paper configs, then a fast parity subset.  TAG names the output files under gpurun_out/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-exp}
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1 || { cat gpurun_out/${TAG}_build.txt; exit 1; }
{
for c in C4 C3 C2; do timeout 120 python tools/kernel_times.py $c; done
for c in C4 C3; do timeout 120 python tools/mlem_time.py $c 100; done
} > gpurun_out/${TAG}_times.txt 2>&1
if [ "${PARITY:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "paper_configs or random_wrapping or C4_headline or many_items or stale or large_tap" > gpurun_out/${TAG}_parity.txt 2>&1; echo "exit $?" >> gpurun_out/${TAG}_parity.txt
fi
cat gpurun_out/${TAG}_times.txt; tail -2 gpurun_out/${TAG}_parity.txt 2>/dev/null
