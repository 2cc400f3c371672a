# In-place reachable-box ratio (CTIS_INPLACE_BOX=1: every plan, 2: single-frame calls only) vs two buffers
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/inbox_times.txt; : > $O
make -j8 all > gpurun_out/inbox_build.txt 2>&1 || { tail -20 gpurun_out/inbox_build.txt; exit 1; }
for rep in 1 2; do
 for w in C3 T1w75 T1w24; do
  for ib in 0 1; do
    echo "$w inbox=$ib $(CTIS_INPLACE_BOX=$ib timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
  done
 done
done
for ib in 0 1; do echo "C5 inbox=$ib $(CTIS_INPLACE_BOX=$ib timeout 300 python tools/c5_batch.py 20 256 2>&1 | tail -1)" >> $O; done
for ib in 0 1; do echo "C5 inbox=$ib $(CTIS_INPLACE_BOX=$ib timeout 300 python tools/c5_batch.py 20 256 2>&1 | tail -1)" >> $O; done
CTIS_INPLACE_BOX=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/inbox_pytest.txt 2>&1
echo "pytest inbox=1: $(tail -1 gpurun_out/inbox_pytest.txt)" >> $O
cat $O
