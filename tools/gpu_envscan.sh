# Time the forward / back kernels at one config under several plan-builder env settings (SCAN="A=1 B=2;...").
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-scan}; CONFIG=${CONFIG:-C4}
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1
IFS=';' read -ra SS <<< "$SCAN"
{ echo "base $(timeout 120 python tools/kernel_times.py $CONFIG)"
for e in "${SS[@]}"; do echo "$e :: $(env $e timeout 120 python tools/kernel_times.py $CONFIG)"; done
} > gpurun_out/${TAG}_scan.txt 2>&1
cat gpurun_out/${TAG}_scan.txt
