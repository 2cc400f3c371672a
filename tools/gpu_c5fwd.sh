# Classic forward knobs at C3 / C5 (probe placement, refill period)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/c5fwd_times.txt; : > $O
make -j8 all > gpurun_out/c5fwd_build.txt 2>&1 || { tail -20 gpurun_out/c5fwd_build.txt; exit 1; }
for v in "p2:-DCTIS_FWD_PROBE=2" "p0:-DCTIS_FWD_PROBE=0" "k6:-DCTIS_FWD_K=6" "k2:-DCTIS_FWD_K=2"; do
  n=${v%%:*}; f=${v#*:}
  make BUILD=build_$n EXTRA="$f" LIBOUT=build_$n/libctis.so build_$n/libctis.so >> gpurun_out/c5fwd_build.txt 2>&1
done
for n in default p2 p0 k6 k2; do
  if [ $n = default ]; then L=""; else L=$PWD/build_$n/libctis.so; fi
  echo "$n C5 $(CTIS_LIB_PATH=$L timeout 300 python tools/c5_batch.py 20 256 2>&1 | tail -1)" >> $O
  echo "$n C3 $(CTIS_LIB_PATH=$L timeout 120 python tools/step_time.py C3 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
done
cat $O
