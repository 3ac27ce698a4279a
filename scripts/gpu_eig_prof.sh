cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/eig_check.py ${EIG_CASES:-} > gpurun_out/eig_pre.log 2>&1; echo rc=$? >> gpurun_out/eig_pre.log
cat gpurun_out/eig_pre.log
EIG_REPS=1 timeout 300 python scripts/eig_check.py ${PROF_CASE:-272} > gpurun_out/eig_plain.log 2>&1 && \
EIG_REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none -s ${PROF_SKIP:-40} -c ${PROF_COUNT:-38} --csv --log-file gpurun_out/eig_launches.csv python scripts/eig_check.py ${PROF_CASE:-272} > gpurun_out/eig_ncu.log 2>&1
echo ncu_rc=$?
python scripts/launch_table.py gpurun_out/eig_launches.csv
