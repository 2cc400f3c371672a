# Strip forward ring position as a barrier address + 32-bit entry index (CTIS_STRIP_ADV=1) vs default;
# flush / TMA-wait attribution (CTIS_DEBUG=2 / 3) of both
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/adv_times.txt; : > $O
make -j8 all > gpurun_out/adv_build.txt 2>&1 || { tail -20 gpurun_out/adv_build.txt; exit 1; }
make BUILD=build_adv EXTRA="-DCTIS_STRIP_ADV=1" LIBOUT=build_adv/libctis.so build_adv/libctis.so >> gpurun_out/adv_build.txt 2>&1
for rep in 1 2; do
  for n in default adv; do
    if [ $n = default ]; then L=""; else L=$PWD/build_$n/libctis.so; fi
    echo "$n $(CTIS_LIB_PATH=$L timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)" >> $O
    echo "$n $(CTIS_LIB_PATH=$L timeout 120 python tools/step_time.py C4 2>&1 | grep ' flush ' | cut -c1-60)" >> $O
  done
done
for n in default adv; do
  if [ $n = default ]; then L=""; else L=$PWD/build_$n/libctis.so; fi
  for d in 2 3; do echo "$n dbg$d $(CTIS_DEBUG=$d CTIS_LIB_PATH=$L timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)" >> $O; done
done
CTIS_LIB_PATH=$PWD/build_adv/libctis.so timeout 900 python -m pytest tests -m gpu -x -q -k "paper_configs or random_wrapping or stale or many_items or C4 or strip" > gpurun_out/adv_pytest.txt 2>&1
echo "pytest adv: $(tail -1 gpurun_out/adv_pytest.txt)" >> $O
cat $O
