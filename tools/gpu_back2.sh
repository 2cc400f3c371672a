# Back kernel occupancy: 32 x 16 tiles (CTIS_BACK_TC=16) at 2/3/4 resident CTAs per SM (CTIS_BACK2_MINB builds)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/back2_times.txt; : > $O
make -j8 all > gpurun_out/back2_build.txt 2>&1 || { tail -20 gpurun_out/back2_build.txt; exit 1; }
for m in 3 4; do make BUILD=build_b2m$m EXTRA="-DCTIS_BACK2_MINB=$m" LIBOUT=build_b2m$m/libctis.so build_b2m$m/libctis.so >> gpurun_out/back2_build.txt 2>&1; done
for w in C4 C3 T1w75; do
 for v in "def::" "tc16:16:" "m3:16:3" "m4:16:4"; do
  n=${v%%:*}; r=${v#*:}; tc=${r%%:*}; ps=${r#*:}
  L=""; [ -n "$ps" ] && L=$PWD/build_b2m$ps/libctis.so
  echo "$w $n $(CTIS_LIB_PATH=$L CTIS_BACK_TC=$tc CTIS_BACK_PER_SM=$ps timeout 120 python tools/kernel_times.py $w 2>&1 | tail -1 | cut -c1-70)" >> $O
  echo "$w $n $(CTIS_LIB_PATH=$L CTIS_BACK_TC=$tc CTIS_BACK_PER_SM=$ps timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
 done
done
cat $O
