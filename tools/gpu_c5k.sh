# Ring refill periods at C5 / C4 / C3: classic forward K = 7, back K = 4 / 7
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/c5k_times.txt; : > $O
make -j8 all > gpurun_out/c5k_build.txt 2>&1 || { tail -20 gpurun_out/c5k_build.txt; exit 1; }
for v in "fk7:-DCTIS_FWD_K=7" "bk4:-DCTIS_BACK_K=4" "bk7:-DCTIS_BACK_K=7"; do
  n=${v%%:*}; f=${v#*:}
  make BUILD=build_$n EXTRA="$f" LIBOUT=build_$n/libctis.so build_$n/libctis.so >> gpurun_out/c5k_build.txt 2>&1
done
for n in default fk7 bk4 bk7; do
  if [ $n = default ]; then L=""; else L=$PWD/build_$n/libctis.so; fi
  echo "$n C5 $(CTIS_LIB_PATH=$L timeout 300 python tools/c5_batch.py 20 256 2>&1 | tail -1)" >> $O
  for w in C3 C4; do echo "$n $w $(CTIS_LIB_PATH=$L timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' | cut -c1-60)" >> $O; done
done
cat $O
