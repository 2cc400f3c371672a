cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=r02b
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/san_case.py loader > gpurun_out/${TAG}_san_synccheck_loader.txt 2>&1; echo "exit $?" >> gpurun_out/${TAG}_san_synccheck_loader.txt
tail -2 gpurun_out/${TAG}_san_synccheck_loader.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.txt 2>&1; tail -2 gpurun_out/${TAG}_pytest.txt
timeout 300 python bench.py --mode bands --steps 3 --warmup 3 --extra "" --no-cpu-baseline > gpurun_out/${TAG}_bands_nccl.json 2>&1; tail -c 600 gpurun_out/${TAG}_bands_nccl.json
timeout 300 python bench.py --mode bands --exchange fused --steps 3 --warmup 3 --extra "" --no-cpu-baseline > gpurun_out/${TAG}_bands_fused.json 2>&1; tail -c 600 gpurun_out/${TAG}_bands_fused.json
