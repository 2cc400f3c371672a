cd $GRAFT_REPO_ROOT
for d in 0 7; do CTIS_DEBUG=$d ncu --set full --clock-control none --import-source on -k regex:ctis_back -s 3 -c 1 -o gpurun_out/exp5_back_d$d -f python tools/kernel_times.py C4 > /dev/null 2>&1; done
