# ncu full captures (forward + back, C4) with source; sanitizer tool check on a plain TMA kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -j8 all > gpurun_out/r2d_build.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o build/tma_test tools/tma_test.cu -lcuda
(timeout 120 compute-sanitizer --tool synccheck ./build/tma_test; echo "exit $?"; timeout 120 compute-sanitizer --tool racecheck ./build/tma_test; echo "exit $?") > gpurun_out/r2d_san_tma_test.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctis_fwd -s 2 -c 1 -o gpurun_out/r2d_prof_fwd -f python tools/prof_driver.py > gpurun_out/r2d_ncu_fwd.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctis_back -s 2 -c 1 -o gpurun_out/r2d_prof_back -f python tools/prof_driver.py > gpurun_out/r2d_ncu_back.txt 2>&1
for k in fwd back; do
  ncu -i gpurun_out/r2d_prof_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r2d_src_$k.csv 2>&1
  ncu -i gpurun_out/r2d_prof_$k.ncu-rep --page raw --csv > gpurun_out/r2d_raw_$k.csv 2>&1
done
