# Time experiment builds against the default: VARS="name:flags ..." (built here as build_<name>), REPS.
# Kernel times at C4 and the MLEM step (tools/kernel_times.py, tools/step_time.py); PYTEST=1 runs the
# strip parity subset on the first variant.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-vars}; O=gpurun_out/${TAG}_times.txt; : > $O
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1 || { tail -20 gpurun_out/${TAG}_build.txt; exit 1; }
names="default"
for v in $VARS; do
  n=${v%%:*}; f=${v#*:}; f=${f//,/ }
  make BUILD=build_$n EXTRA="$f" LIBOUT=build_$n/libctis.so build_$n/libctis.so >> gpurun_out/${TAG}_build.txt 2>&1 || echo "build $n failed" >> $O
  names="$names $n"
done
for rep in $(seq 1 ${REPS:-2}); do
  for n in $names; do
    if [ $n = default ]; then L=""; else L=$PWD/build_$n/libctis.so; fi
    for w in ${WLS:-C4}; do
      echo "$n $(CTIS_LIB_PATH=$L timeout 120 python tools/kernel_times.py $w 2>&1 | tail -1 | cut -c1-60)" >> $O
      echo "$n $(CTIS_LIB_PATH=$L timeout 120 python tools/step_time.py $w 2>&1 | grep ' flush ' )" >> $O
    done
  done
done
if [ "${PYTEST:-0}" = "1" ]; then
  first=$(echo $names | cut -d' ' -f2)
  CTIS_LIB_PATH=$PWD/build_$first/libctis.so timeout 900 python -m pytest tests -m gpu -x -q -k "paper_configs or random_wrapping or stale or many_items or C4 or strip" > gpurun_out/${TAG}_pytest.txt 2>&1
  echo "pytest $first: $(tail -1 gpurun_out/${TAG}_pytest.txt)" >> $O
fi
cat $O
