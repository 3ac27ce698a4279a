cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
EIG_REPS=1 timeout 300 python scripts/eig_check.py 272 > gpurun_out/eig_plain.log 2>&1 && \
EIG_REPS=1 ncu --set full --import-source on --clock-control none -k regex:"sytrd|backtransform|reflector|twisted|bisect" -s 5 -c 5 -o gpurun_out/eig_full -f python scripts/eig_check.py 272 > gpurun_out/eig_ncu_full.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/eig_ncu_full.log
