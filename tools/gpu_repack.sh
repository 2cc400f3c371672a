# f repack (warp per column) and mode-split update (per-frame grid, 32-bit band index) vs the committed build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/repack_times.txt; : > $O
git stash list > /dev/null 2>&1
make -j8 all > gpurun_out/repack_build.txt 2>&1 || { tail -20 gpurun_out/repack_build.txt; exit 1; }
for rep in 1 2; do
  for w in T1w75 T1w24 T1w3; do
    echo "$w new $(timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/repack_pytest.txt 2>&1
echo "pytest: $(tail -1 gpurun_out/repack_pytest.txt)" >> $O
cat $O
