# Strip-forward loop variants (CTIS_STRIP_PIN / CTIS_STRIP_PROBE builds): kernel times at C4, C5-shaped
# batches and the MLEM step, then the strip parity subset on the fastest candidate.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/probe_times.txt; : > $O
make -j8 all > gpurun_out/probe_build.txt 2>&1 || { tail -20 gpurun_out/probe_build.txt; exit 1; }
for v in "pin:-DCTIS_STRIP_PIN=1" "probe:-DCTIS_STRIP_PROBE=1" "pp:-DCTIS_STRIP_PIN=1 -DCTIS_STRIP_PROBE=1"; do
  n=${v%%:*}; f=${v#*:}
  make BUILD=build_$n EXTRA="$f" LIBOUT=build_$n/libctis.so build_$n/libctis.so >> gpurun_out/probe_build.txt 2>&1
done
for rep in 1 2; do
  for n in default pin probe pp; do
    if [ $n = default ]; then L=""; else L=$PWD/build_$n/libctis.so; fi
    echo "$n $(CTIS_LIB_PATH=$L timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)" >> $O
    echo "$n $(CTIS_LIB_PATH=$L timeout 120 python tools/step_time.py C4 2>&1 | grep ' flush ' )" >> $O
  done
done
for n in default pp; do
  if [ $n = default ]; then L=""; else L=$PWD/build_$n/libctis.so; fi
  echo "$n $(CTIS_LIB_PATH=$L CTIS_FWD_STRIP=1 timeout 120 python tools/kernel_times.py C3 2>&1 | tail -1 | cut -c1-60)" >> $O
done
CTIS_LIB_PATH=$PWD/build_pp/libctis.so timeout 600 python -m pytest tests -m gpu -x -q -k "paper_configs or random_wrapping or stale or many_items or C4" > gpurun_out/probe_pytest.txt 2>&1
tail -2 gpurun_out/probe_pytest.txt >> $O
cat $O
