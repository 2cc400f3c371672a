# Reachable-box ratio with per-frame 2-D grid and 32-bit index math (CTIS_RATIO_BOX2D=1) vs 64-bit divisions
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/box2d_times.txt; : > $O
make -j8 all > gpurun_out/box2d_build.txt 2>&1 || { tail -20 gpurun_out/box2d_build.txt; exit 1; }
make BUILD=build_b2d EXTRA="-DCTIS_RATIO_BOX2D=1" LIBOUT=build_b2d/libctis.so build_b2d/libctis.so >> gpurun_out/box2d_build.txt 2>&1
B=$PWD/build_b2d/libctis.so
for rep in 1 2; do
  for w in C3 T1w75 T1w24; do
    echo "$w def $(timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
    echo "$w b2d $(CTIS_LIB_PATH=$B timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
  done
  echo "C5 def $(timeout 300 python tools/c5_batch.py 20 256 2>&1 | tail -1)" >> $O
  echo "C5 b2d $(CTIS_LIB_PATH=$B timeout 300 python tools/c5_batch.py 20 256 2>&1 | tail -1)" >> $O
done
CTIS_LIB_PATH=$B timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/box2d_pytest.txt 2>&1
echo "pytest b2d: $(tail -1 gpurun_out/box2d_pytest.txt)" >> $O
cat $O
