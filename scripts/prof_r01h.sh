mkdir -p gpurun_out
python scripts/profile_step.py cfg1 2 > gpurun_out/ps_cfg1.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01h_cfg1.csv python scripts/profile_step.py cfg1 2 > gpurun_out/ncu_l1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01h_cfg4.csv python scripts/profile_step.py cfg4 1 > gpurun_out/ncu_l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_far_list -c 1 -o gpurun_out/farlist_r01h python scripts/profile_step.py cfg1 1 > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_feval -c 1 -o gpurun_out/feval_r01h python scripts/profile_step.py cfg1 1 > gpurun_out/ncu_fe.log 2>&1
ls -la gpurun_out
