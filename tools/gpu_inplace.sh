# In-place ratio (r overwrites g_hat, memset node clears it after the back projection) vs ratio + reset
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/inplace_times.txt; : > $O
make -j8 all > gpurun_out/inplace_build.txt 2>&1 || { tail -20 gpurun_out/inplace_build.txt; exit 1; }
for rep in 1 2; do
 for w in C4 C3 C2; do
  for ip in 0 1; do
    echo "$w inplace=$ip $(CTIS_INPLACE_RATIO=$ip timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
  done
 done
done
for ip in 0 1; do echo "C5 inplace=$ip $(CTIS_INPLACE_RATIO=$ip timeout 300 python tools/c5_batch.py 20 256 2>&1 | tail -1)" >> $O; done
CTIS_INPLACE_RATIO=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/inplace_pytest.txt 2>&1
echo "pytest inplace: $(tail -1 gpurun_out/inplace_pytest.txt)" >> $O
cat $O
