# Strip forward diagnosis: debug switches and one ncu full capture of the strip kernel (C4)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-strip2}
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -20 gpurun_out/${T}_build.txt; exit 1; }
{
for d in 0 2 3; do
  echo "strip dbg=$d $(CTIS_DEBUG=$d CTIS_FWD_STRIP=1 timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)"
done
} > gpurun_out/${T}_times.txt 2>&1
cat gpurun_out/${T}_times.txt
CTIS_FWD_STRIP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctis_fwd -s 2 -c 1 -o gpurun_out/${T}_prof_fwd -f python tools/prof_driver.py > gpurun_out/${T}_ncu_fwd.txt 2>&1
ncu -i gpurun_out/${T}_prof_fwd.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_src_fwd.csv 2>&1
ncu -i gpurun_out/${T}_prof_fwd.ncu-rep --page raw --csv > gpurun_out/${T}_raw_fwd.csv 2>&1
python tools/src_stalls.py gpurun_out/${T}_src_fwd.csv > gpurun_out/${T}_stalls.txt 2>&1
head -60 gpurun_out/${T}_stalls.txt
