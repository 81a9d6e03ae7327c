#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "tree or config or shard" > gpurun_out/r02k_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02k_pytest.log
ST_DEBUG_TIMELINE=1 timeout 900 python scripts/shard_balance.py cfg4 8 split > gpurun_out/r02k_shard4.jsonl 2> gpurun_out/r02k_shard4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k_launches_cfg4.csv python scripts/profile_step.py cfg4 1 > gpurun_out/r02k_ncu.log 2>&1
