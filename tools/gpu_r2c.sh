cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -j8 all > gpurun_out/r2c_build.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/flushbench tools/flushbench.cu
timeout 120 ./build/flushbench > gpurun_out/r2c_flushbench.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --num-cuda-barriers 4096 --error-exitcode 9 python tools/san_case.py bench > gpurun_out/r2c_san_synccheck_bench.txt 2>&1; echo "exit $?" >> gpurun_out/r2c_san_synccheck_bench.txt
timeout 900 compute-sanitizer --tool racecheck --num-cuda-barriers 4096 --error-exitcode 9 python tools/san_case.py bench > gpurun_out/r2c_san_racecheck_bench.txt 2>&1; echo "exit $?" >> gpurun_out/r2c_san_racecheck_bench.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/san_case.py loader > gpurun_out/r2c_san_racecheck_loader.txt 2>&1; echo "exit $?" >> gpurun_out/r2c_san_racecheck_loader.txt
