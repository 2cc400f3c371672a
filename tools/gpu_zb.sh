cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -j8 all > /dev/null 2>&1 || exit 1
for c in C4 C3; do
echo "$c zero_in_back=1 $(timeout 200 python tools/mlem_time.py $c 100)"
echo "$c zero_in_back=0 $(CTIS_ZERO_IN_BACK=0 timeout 200 python tools/mlem_time.py $c 100)"
echo "$c fused        $(CTIS_FUSED=1 timeout 200 python tools/mlem_time.py $c 100)"
done
timeout 900 python -m pytest tests -m gpu -x -q -k "mlem or smart or monitored or fused" 2>&1 | tail -2
