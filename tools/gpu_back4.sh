# Back kernel: 32 x 32 tiles at 3 resident CTAs per SM without spills (CTIS_BACK4_MINB=3, CTIS_BACK_EG=2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/back4_times.txt; : > $O
make -j8 all > gpurun_out/back4_build.txt 2>&1 || { tail -20 gpurun_out/back4_build.txt; exit 1; }
make BUILD=build_e2 EXTRA="-DCTIS_BACK4_MINB=3 -DCTIS_BACK_EG=2" LIBOUT=build_e2/libctis.so build_e2/libctis.so >> gpurun_out/back4_build.txt 2>&1
make BUILD=build_e2m2 EXTRA="-DCTIS_BACK_EG=2" LIBOUT=build_e2m2/libctis.so build_e2m2/libctis.so >> gpurun_out/back4_build.txt 2>&1
B=$PWD/build_e2/libctis.so
for nb in 12 10 8; do
  echo "C4 def nb$nb $(CTIS_BACK_NB=$nb timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-70)" >> $O
  echo "C4 e2m3 nb$nb $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 CTIS_BACK_NB=$nb timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-70)" >> $O
done
echo "C4 e2m2 nb12 $(CTIS_LIB_PATH=$PWD/build_e2m2/libctis.so timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-70)" >> $O
echo "C4 def step $(timeout 120 python tools/step_time.py C4 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
echo "C4 e2m3 step $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 timeout 120 python tools/step_time.py C4 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
echo "C5/64 def $(timeout 300 python tools/kernel_times.py C5 64 2>&1 | tail -1 | cut -c1-110)" >> $O
echo "C5/64 e2m3 $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 timeout 300 python tools/kernel_times.py C5 64 2>&1 | tail -1 | cut -c1-110)" >> $O
echo "C3 def $(timeout 120 python tools/kernel_times.py C3 2>&1 | tail -1 | cut -c1-70)" >> $O
echo "C3 e2m3 $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 timeout 120 python tools/kernel_times.py C3 2>&1 | tail -1 | cut -c1-70)" >> $O
echo "T1w75 def $(timeout 120 python tools/kernel_times.py T1w75 2>&1 | tail -1 | cut -c1-70)" >> $O
echo "T1w75 e2m3 $(CTIS_LIB_PATH=$B CTIS_BACK_PER_SM=3 timeout 120 python tools/kernel_times.py T1w75 2>&1 | tail -1 | cut -c1-70)" >> $O
cat $O
