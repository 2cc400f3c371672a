cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-fz}
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1 || { tail gpurun_out/${TAG}_build.txt; exit 1; }
{
for c in C4 C3 C2; do for fz in 1 0; do CTIS_FUSED=$fz timeout 120 python tools/mlem_time.py $c 100; done; done
for fz in 1 0; do CTIS_FUSED=$fz timeout 120 python tools/mlem_time.py C4 100 smart; done
} > gpurun_out/${TAG}_times.txt 2>&1
cat gpurun_out/${TAG}_times.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.txt
tail -3 gpurun_out/${TAG}_pytest.txt
