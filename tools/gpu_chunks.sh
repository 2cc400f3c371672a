# Strip forward chunking at C4: bands per chunk x mode span (CTIS_FWD_BANDS / CTIS_FWD_SPAN)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
O=gpurun_out/chunks_times.txt; : > $O
make -j8 all > gpurun_out/chunks_build.txt 2>&1 || { tail -20 gpurun_out/chunks_build.txt; exit 1; }
echo "default $(timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-300)" >> $O
for v in 20:16 20:13 17:12 34:22 34:20 25:20 50:32; do
  b=${v%%:*}; sp=${v#*:}
  echo "bands=$b span=$sp $(CTIS_FWD_BANDS=$b CTIS_FWD_SPAN=$sp timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-300)" >> $O
done
cat $O
