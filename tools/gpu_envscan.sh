# Time the forward / back kernels at one config under several plan-builder env settings (SCAN="A=1 B=2;...").
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-scan}; CONFIG=${CONFIG:-C4}; FRAMES=${FRAMES:-1}
make -j8 all > gpurun_out/${TAG}_build.txt 2>&1
IFS=';' read -ra SS <<< "$SCAN"
{ for F in $FRAMES; do echo "base $(timeout 120 python tools/kernel_times.py $CONFIG $F | cut -c1-110)"
for e in "${SS[@]}"; do echo "$e :: $(env $e timeout 120 python tools/kernel_times.py $CONFIG $F | cut -c1-110)"; done; done
} > gpurun_out/${TAG}_scan.txt 2>&1
cat gpurun_out/${TAG}_scan.txt
