#!/bin/bash
# One gpurun session: GPU tests, smoke, bench (+ latency-mode lines), ncu launch list and full captures,
# compute-sanitizer.  TAG names the outputs under gpurun_out/.
set +e
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_nvsmi.txt 2>&1
(nproc; lscpu | grep -i "model name") > gpurun_out/${TAG}_host.txt 2>&1
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.txt; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ "${BANDS:-1}" = "1" ]; then
  timeout 300 python bench.py --mode bands --steps 3 --warmup 3 --extra "" --no-cpu-baseline > gpurun_out/${TAG}_bench_bands_nccl.json 2>&1
  timeout 300 python bench.py --mode bands --exchange fused --steps 3 --warmup 3 --extra "" --no-cpu-baseline > gpurun_out/${TAG}_bench_bands_fused.json 2>&1
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --extra "" \
     > gpurun_out/${TAG}_ncu_bench.txt 2>&1
  for k in fwd back; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctis_$k -s 2 -c 1 \
       -o gpurun_out/${TAG}_prof_$k -f python tools/prof_driver.py > gpurun_out/${TAG}_ncu_$k.txt 2>&1
    ncu -i gpurun_out/${TAG}_prof_$k.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_$k.csv 2>&1
    ncu -i gpurun_out/${TAG}_prof_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src_$k.csv 2>&1
  done
fi
if [ "${SAN:-0}" = "1" ]; then
  timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/san_case.py bench > gpurun_out/${TAG}_san_memcheck_bench.txt 2>&1; echo "exit $?" >> gpurun_out/${TAG}_san_memcheck_bench.txt
  CTIS_FWD_STRIP=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/san_case.py bench > gpurun_out/${TAG}_san_memcheck_strip.txt 2>&1; echo "exit $?" >> gpurun_out/${TAG}_san_memcheck_strip.txt
  timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/san_case.py loader > gpurun_out/${TAG}_san_memcheck_loader.txt 2>&1; echo "exit $?" >> gpurun_out/${TAG}_san_memcheck_loader.txt
  timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/san_case.py loader > gpurun_out/${TAG}_san_racecheck_loader.txt 2>&1; echo "exit $?" >> gpurun_out/${TAG}_san_racecheck_loader.txt
  timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/san_case.py loader > gpurun_out/${TAG}_san_synccheck_loader.txt 2>&1; echo "exit $?" >> gpurun_out/${TAG}_san_synccheck_loader.txt
fi
echo done
