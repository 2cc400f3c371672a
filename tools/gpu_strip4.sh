cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -j8 all > gpurun_out/strip4_build.txt 2>&1 || { tail -20 gpurun_out/strip4_build.txt; exit 1; }
for st in 4 6 8; do echo "stages<=$st $(CTIS_STRIP_STAGES=$st timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)"; done
echo "dbg2 $(CTIS_DEBUG=2 timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)"
echo "dbg3 $(CTIS_DEBUG=3 timeout 120 python tools/kernel_times.py C4 2>&1 | tail -1 | cut -c1-60)"
timeout 600 python -m pytest tests -m gpu -x -q -k "paper_configs or random_wrapping or stale or many_items or fused_ratio or C4" 2>&1 | tail -2
