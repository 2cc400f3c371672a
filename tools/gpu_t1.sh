cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -j8 all > /dev/null 2>&1 || exit 1
for c in T1w75 T1w24 T1w3 C4 C3; do
  echo "$(timeout 200 python tools/kernel_times.py $c | cut -c1-80)"
  echo "$(timeout 200 python tools/mlem_time.py $c 100)"
done
echo "T1w75 loader $(CTIS_FWD_REPACK=0 timeout 200 python tools/mlem_time.py T1w75 100)"
echo "C4 fullratio $(CTIS_NO_RATIO_BOX=1 timeout 200 python tools/mlem_time.py C4 100)"
echo "C3 fullratio $(CTIS_NO_RATIO_BOX=1 timeout 200 python tools/mlem_time.py C3 100)"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
