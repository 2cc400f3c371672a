# One ncu --set full capture of the strip forward at C4 (source-level stalls), TAG names the outputs.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-fwd}
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1 || { tail -20 gpurun_out/${TAG}_build.txt; exit 1; }
timeout 120 python tools/prof_driver.py > gpurun_out/${TAG}_driver.txt 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctis_fwd -s 2 -c 1 \
   -o gpurun_out/${TAG}_prof_fwd -f python tools/prof_driver.py > gpurun_out/${TAG}_ncu_fwd.txt 2>&1
ncu -i gpurun_out/${TAG}_prof_fwd.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_fwd.csv 2>&1
ncu -i gpurun_out/${TAG}_prof_fwd.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src_fwd.csv 2>&1
python tools/src_stalls.py gpurun_out/${TAG}_src_fwd.csv > gpurun_out/${TAG}_stalls_fwd.txt 2>&1
head -60 gpurun_out/${TAG}_stalls_fwd.txt
