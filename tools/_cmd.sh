cd $GRAFT_REPO_ROOT
for c in C4 C3; do python tools/kernel_times.py $c; python tools/mlem_time.py $c; done > gpurun_out/r02r.txt 2>&1
CTIS_DEBUG=8 python tests/poison_case.py >> gpurun_out/r02r.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "paper_configs or smart or wrapping or batched" >> gpurun_out/r02r.txt 2>&1
