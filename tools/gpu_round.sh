#!/bin/bash
# One gpurun session: microbench, GPU tests, smoke, bench, ncu launch list and full captures.
set +e
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_nvsmi.txt 2>&1
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1
[ -x build/microbench ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu
if [ "${MICRO:-1}" = "1" ]; then timeout 300 ./build/microbench > gpurun_out/${TAG}_microbench.json 2>&1; fi
if [ "${TESTS:-1}" = "1" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.txt; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
     > gpurun_out/${TAG}_ncu_bench.txt 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctis_fwd -s 2 -c 1 \
     -o gpurun_out/${TAG}_prof_fwd -f python tools/prof_driver.py > gpurun_out/${TAG}_ncu_fwd.txt 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctis_back -s 2 -c 1 \
     -o gpurun_out/${TAG}_prof_back -f python tools/prof_driver.py > gpurun_out/${TAG}_ncu_back.txt 2>&1
fi
echo done
