cd $GRAFT_REPO_ROOT
for d in 3; do CTIS_DEBUG=$d ncu --set full --clock-control none --import-source on -k regex:ctis_fwd -s 3 -c 1 -o gpurun_out/exp8_fwd_d$d -f python tools/kernel_times.py C4 > /dev/null 2>&1; done
