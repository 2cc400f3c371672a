# Build several compile-time variants of libctis (VARIANTS="name:-DFLAGS;..."), time each on one GPU.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-var}; CONFIGS=${CONFIGS:-"C4 C3"}
make -j8 all > gpurun_out/${TAG}_build_base.txt 2>&1
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name=${v%%:*}; flags=${v#*:}
  make -j8 BUILD=build_$name LIBOUT=build_$name/libctis.so EXTRA="$flags" build_$name/libctis.so > gpurun_out/${TAG}_build_$name.txt 2>&1 || { echo "BUILD FAIL $name"; tail -5 gpurun_out/${TAG}_build_$name.txt; }
done
{
for rep in 1 2; do
for c in $CONFIGS; do
  echo "base $(timeout 120 python tools/kernel_times.py $c)"
  for v in "${VS[@]}"; do name=${v%%:*}; echo "$name $(CTIS_LIB_PATH=$PWD/build_$name/libctis.so timeout 120 python tools/kernel_times.py $c)"; done
done; done
if [ "${MLEM:-0}" = "1" ]; then
for c in $CONFIGS; do
  echo "base $(timeout 120 python tools/mlem_time.py $c 100)"
  for v in "${VS[@]}"; do name=${v%%:*}; echo "$name $(CTIS_LIB_PATH=$PWD/build_$name/libctis.so timeout 120 python tools/mlem_time.py $c 100)"; done
done; fi
} > gpurun_out/${TAG}_times.txt 2>&1
cat gpurun_out/${TAG}_times.txt
if [ "${PARITY:-0}" = "1" ]; then
  for v in "${VS[@]}"; do name=${v%%:*};
    CTIS_LIB_PATH=$PWD/build_$name/libctis.so timeout 900 python -m pytest tests -m gpu -x -q -k "${PK:-paper_configs or random_wrapping or many_items or stale or large_tap or C5_launch}" > gpurun_out/${TAG}_parity_$name.txt 2>&1
    echo "parity $name: $(tail -1 gpurun_out/${TAG}_parity_$name.txt)"
  done
fi
