#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api_edges.py tests/test_acceptance.py tests/test_gpu_configs.py "tests/test_gpu_parity.py::test_shard_plan_matches_host_model" -m gpu -q -rA > gpurun_out/r02c_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02c_pytest.log
timeout 900 python scripts/sweep_cfg2_r02.py > gpurun_out/r02c_sweep.log 2>&1
cp profiles/r02_cfg2_psweep.json gpurun_out/ 2>/dev/null
bash scripts/sanitize.sh
