# Back projection on 16 warps per 32 x 32 tile (CTIS_BACK_WIDE=1, ctis_back8_*) vs 8 warps (ctis_back4_*)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/wide_times.txt; : > $O
make -j8 all > gpurun_out/wide_build.txt 2>&1 || { tail -20 gpurun_out/wide_build.txt; exit 1; }
for w in C4 C3 T1w75 C2; do
  for wd in 0 1; do
    echo "$w wide=$wd $(CTIS_BACK_WIDE=$wd timeout 120 python tools/kernel_times.py $w 2>&1 | tail -1 | cut -c1-60)" >> $O
    echo "$w wide=$wd $(CTIS_BACK_WIDE=$wd timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
  done
done
for wd in 0 1; do
  echo "C5/64 wide=$wd $(CTIS_BACK_WIDE=$wd timeout 300 python tools/kernel_times.py C5 64 2>&1 | tail -1 | cut -c1-110)" >> $O
done
for nb in 8 16; do echo "C4 wide=1 nb$nb $(CTIS_BACK_WIDE=1 CTIS_BACK_NB=$nb timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)" >> $O; done
CTIS_BACK_WIDE=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/wide_pytest.txt 2>&1
echo "pytest wide: $(tail -1 gpurun_out/wide_pytest.txt)" >> $O
cat $O
