# In-place ratio with two alternating accumulators, the next one cleared on a forked graph branch beside
# the forward (CTIS_FORK_CLEAR=1) vs the memset node in line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/fork_times.txt; : > $O
make -j8 all > gpurun_out/fork_build.txt 2>&1 || { tail -20 gpurun_out/fork_build.txt; exit 1; }
for rep in 1 2 3; do
  for fk in 0 1; do
    echo "C4 fork=$fk $(CTIS_FORK_CLEAR=$fk timeout 120 python tools/step_time.py C4 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
  done
done
CTIS_FORK_CLEAR=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fork_pytest.txt 2>&1
echo "pytest fork=1: $(tail -1 gpurun_out/fork_pytest.txt)" >> $O
cat $O
