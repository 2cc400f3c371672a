# The GPU parity suite under the kernel-selection switches (forced strip forward everywhere, the two-buffer
# ratio, programmatic dependent launch), each in its own process
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -j8 all > gpurun_out/envsuite_build.txt 2>&1 || { tail -20 gpurun_out/envsuite_build.txt; exit 1; }
O=gpurun_out/envsuite.txt; : > $O
for env in "CTIS_FWD_STRIP=1" "CTIS_INPLACE_RATIO=0" "CTIS_PDL=1"; do
  env $env timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/envsuite_${env%%=*}.txt 2>&1
  echo "$env: $(tail -1 gpurun_out/envsuite_${env%%=*}.txt)" >> $O
done
cat $O
