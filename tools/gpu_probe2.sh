# Strip forward: always-probe dispatch (CTIS_STRIP_PROBE=2, one dispatch copy) vs the default; C5 split.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/probe2_times.txt; : > $O
make -j8 all > gpurun_out/probe2_build.txt 2>&1 || { tail -20 gpurun_out/probe2_build.txt; exit 1; }
make BUILD=build_p2 EXTRA="-DCTIS_STRIP_PROBE=2" LIBOUT=build_p2/libctis.so build_p2/libctis.so >> gpurun_out/probe2_build.txt 2>&1
for rep in 1 2; do
  for n in default p2; do
    if [ $n = default ]; then L=""; else L=$PWD/build_$n/libctis.so; fi
    echo "$n $(CTIS_LIB_PATH=$L timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)" >> $O
    echo "$n $(CTIS_LIB_PATH=$L timeout 120 python tools/step_time.py C4 2>&1 | grep ' flush ' )" >> $O
  done
done
echo "C5/64 $(timeout 300 python tools/kernel_times.py C5 64 2>&1 | tail -1 | cut -c1-120)" >> $O
echo "C3 $(timeout 300 python tools/kernel_times.py C3 2>&1 | tail -1 | cut -c1-120)" >> $O
cat $O
