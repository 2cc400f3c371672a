cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -j8 all > /dev/null 2>&1 || exit 1
for c in C3 C4 C2 T1w75; do
  echo "$(timeout 200 python tools/kernel_times.py $c | cut -c1-200)"
  echo "$(timeout 200 python tools/mlem_time.py $c 100)"
done
echo "C5: $(timeout 300 python tools/kernel_times.py C3 64 | cut -c1-120)"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -20
