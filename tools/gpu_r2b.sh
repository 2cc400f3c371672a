cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(nproc; lscpu | grep -i "model name\|^CPU(s)\|Socket\|Thread"; free -g | head -2) > gpurun_out/r2b_host.txt 2>&1
make -j8 all > gpurun_out/r2b_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "C4_headline or C5_launch or band_shards or large_tap or pdl or paper_configs" > gpurun_out/r2b_pytest_new.txt 2>&1; echo "exit $?" >> gpurun_out/r2b_pytest_new.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/san_case.py bench > gpurun_out/r2b_san_${tool}_bench.txt 2>&1; echo "exit $?" >> gpurun_out/r2b_san_${tool}_bench.txt
done
