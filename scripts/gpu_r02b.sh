#!/bin/bash
# round 2, pass b: the whole GPU suite (incl. full-size config parity), then ncu of the
# moment pass (K2) at cfg1 and cfg4 with ST_MOMENTS_INLINE=1 (nothing overlaps it)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=20 -rA > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02b_pytest.log
export ST_MOMENTS_INLINE=1
python scripts/profile_step.py cfg1 2 > gpurun_out/r02b_ps1.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_moments|k_m2m|k_fold" --launch-skip 8 -c 10 -o gpurun_out/r02b_moments_cfg1 python scripts/profile_step.py cfg1 2 > gpurun_out/r02b_ncu_m1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_moments|k_m2m|k_fold" -c 10 -o gpurun_out/r02b_moments_cfg4 python scripts/profile_step.py cfg4 1 > gpurun_out/r02b_ncu_m4.log 2>&1
ls -la gpurun_out | tail -5
