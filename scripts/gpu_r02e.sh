#!/bin/bash
# ncu of the two-target far kernels (cfg2: P = 12, cfg1: P = 10) + the acceptance test
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_acceptance.py -m gpu -q > gpurun_out/r02e_acc.log 2>&1
python scripts/profile_step.py cfg2 1 > gpurun_out/r02e_ps2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_far_list|k_feval" -c 2 -o gpurun_out/r02e_far_cfg2 python scripts/profile_step.py cfg2 1 > gpurun_out/r02e_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_far_list|k_feval" -c 2 -o gpurun_out/r02e_far_cfg1 python scripts/profile_step.py cfg1 1 > gpurun_out/r02e_ncu1.log 2>&1
