cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-c5}
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1 || exit 1
{ for F in 8 256; do timeout 300 python tools/kernel_times.py C3 $F; CTIS_NO_TPUT=1 timeout 300 python tools/kernel_times.py C3 $F; done
  for F in 8; do timeout 300 python tools/kernel_times.py C2 $F; CTIS_NO_TPUT=1 timeout 300 python tools/kernel_times.py C2 $F; done; } > gpurun_out/${TAG}_times.txt 2>&1
cat gpurun_out/${TAG}_times.txt | cut -c1-150
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or batched or C5 or smart or many_items" > gpurun_out/${TAG}_test.txt 2>&1; tail -1 gpurun_out/${TAG}_test.txt
timeout 600 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c5.json 2>&1; cut -c1-400 gpurun_out/${TAG}_bench_c5.json
