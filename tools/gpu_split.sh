cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -j8 all > /dev/null 2>&1 || exit 1
for c in T1w3 T1w24 T1w75 C3 C2 tiny C4; do
  echo "split  $(timeout 200 python tools/mlem_time.py $c 100)  $(timeout 200 python tools/kernel_times.py $c | cut -c1-60)"
  echo "nosplit $(CTIS_BACK_SPLIT=1 timeout 200 python tools/mlem_time.py $c 100)"
done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
