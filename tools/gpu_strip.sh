# Strip forward: kernel times (classic vs strip) and parity (auto and forced strip)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-strip1}
make -j8 all > gpurun_out/${T}_build.txt 2>&1 || { tail -20 gpurun_out/${T}_build.txt; exit 1; }
{
for c in C4 C3 C2 tiny; do
  echo "classic $(CTIS_FWD_STRIP=0 timeout 120 python tools/kernel_times.py $c 2>&1 | tail -2)"
  echo "strip   $(CTIS_FWD_STRIP=1 timeout 120 python tools/kernel_times.py $c 2>&1 | tail -2)"
done
echo "C5 classic $(CTIS_FWD_STRIP=0 timeout 120 python tools/kernel_times.py C3 64 2>&1 | tail -2)"
echo "C5 strip   $(CTIS_FWD_STRIP=1 timeout 120 python tools/kernel_times.py C3 64 2>&1 | tail -2)"
} > gpurun_out/${T}_times.txt 2>&1
cat gpurun_out/${T}_times.txt
CTIS_FWD_STRIP=1 timeout 900 python -m pytest tests -m gpu -x -q -k "${PK:-paper_configs or random_wrapping or stale or many_items or fused_ratio or unit_tap or full_wrap}" > gpurun_out/${T}_parity_forced.txt 2>&1
echo "forced strip parity: $(tail -1 gpurun_out/${T}_parity_forced.txt)"
