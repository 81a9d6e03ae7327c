# ncu captures of the far-field kernels at cfg4 (8M mixture -> 8M disjoint targets)
mkdir -p gpurun_out
python scripts/profile_step.py cfg4 1 > gpurun_out/ps_cfg4.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01i_cfg4.csv python scripts/profile_step.py cfg4 1 > gpurun_out/ncu_l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_far_list -c 1 -o gpurun_out/farlist_r01i_cfg4 python scripts/profile_step.py cfg4 1 > gpurun_out/ncu_f4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_feval -c 1 -o gpurun_out/feval_r01i_cfg4 python scripts/profile_step.py cfg4 1 > gpurun_out/ncu_fe4.log 2>&1
ls -la gpurun_out
