cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(timeout 300 python scripts/eig_check.py > gpurun_out/eig_pre.log 2>&1; echo rc=$? >> gpurun_out/eig_pre.log)
cat gpurun_out/eig_pre.log
(LRAMM_EIG_PRE=0 timeout 300 python scripts/eig_check.py > gpurun_out/eig_nopre.log 2>&1; echo rc=$? >> gpurun_out/eig_nopre.log)
cat gpurun_out/eig_nopre.log
