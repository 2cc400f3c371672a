# Back kernel: 32 x 32 tiles at 3 resident CTAs per SM (CTIS_BACK4_MINB=3 build, 80 registers) vs 2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/back3_times.txt; : > $O
make -j8 all > gpurun_out/back3_build.txt 2>&1 || { tail -20 gpurun_out/back3_build.txt; exit 1; }
make BUILD=build_b4m3 EXTRA="-DCTIS_BACK4_MINB=3" LIBOUT=build_b4m3/libctis.so build_b4m3/libctis.so >> gpurun_out/back3_build.txt 2>&1
B=$PWD/build_b4m3/libctis.so
for nb in 12 8 4; do
  echo "C4 def nb$nb $(CTIS_BACK_NB=$nb timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-70)" >> $O
  echo "C4 m3 nb$nb $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 CTIS_BACK_NB=$nb timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-70)" >> $O
done
echo "C4 m3 step $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 timeout 120 python tools/step_time.py C4 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
echo "C4 m3 nb8 step $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 CTIS_BACK_NB=8 timeout 120 python tools/step_time.py C4 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
echo "C4 m2 compiled, 3 resident $(CTIS_BACK_PER_SM=3 timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-70)" >> $O
echo "C5/64 def $(timeout 300 python tools/kernel_times.py C5 64 2>&1 | tail -1 | cut -c1-110)" >> $O
echo "C5/64 m3 $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 timeout 300 python tools/kernel_times.py C5 64 2>&1 | tail -1 | cut -c1-110)" >> $O
echo "C3 m3 $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 timeout 120 python tools/kernel_times.py C3 2>&1 | tail -1 | cut -c1-70)" >> $O
cat $O
