#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "tree or config_parity" > gpurun_out/s3c_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3c_pytest.log
for c in cfg1 cfg4; do
  ST_DEBUG_BUILD=1 timeout 300 python scripts/probe_cfg.py $c 3 >> gpurun_out/s3c_build.log 2>&1
done
