# Back projection on 32 x 64 tiles, eight voxels per thread (CTIS_BACK_TC=64, ctis_backw_*) vs 32 x 32
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/tc64_times.txt; : > $O
make -j8 all > gpurun_out/tc64_build.txt 2>&1 || { tail -20 gpurun_out/tc64_build.txt; exit 1; }
echo "C4 def $(timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)" >> $O
for nb in 4 6 8; do echo "C4 tc64 nb$nb $(CTIS_BACK_TC=64 CTIS_BACK_NB=$nb timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)" >> $O; done
echo "C3 def $(timeout 120 python tools/kernel_times.py C3 2>&1 | tail -1 | cut -c1-60)" >> $O
for nb in 2 4 6; do echo "C3 tc64 nb$nb $(CTIS_BACK_TC=64 CTIS_BACK_NB=$nb timeout 120 python tools/kernel_times.py C3 2>&1 | tail -1 | cut -c1-60)" >> $O; done
echo "T1w75 def $(timeout 120 python tools/kernel_times.py T1w75 2>&1 | tail -1 | cut -c1-60)" >> $O
for nb in 2 4 6; do echo "T1w75 tc64 nb$nb $(CTIS_BACK_TC=64 CTIS_BACK_NB=$nb timeout 120 python tools/kernel_times.py T1w75 2>&1 | tail -1 | cut -c1-60)" >> $O; done
echo "C5/64 def $(timeout 300 python tools/kernel_times.py C5 64 2>&1 | tail -1 | cut -c1-110)" >> $O
for nb in 4 6 8; do echo "C5/64 tc64 nb$nb $(CTIS_BACK_TC=64 CTIS_BACK_NB=$nb timeout 300 python tools/kernel_times.py C5 64 2>&1 | tail -1 | cut -c1-110)" >> $O; done
CTIS_BACK_TC=64 CTIS_BACK_NB=6 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tc64_pytest.txt 2>&1
echo "pytest tc64 nb6: $(tail -1 gpurun_out/tc64_pytest.txt)" >> $O
cat $O
