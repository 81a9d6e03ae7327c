#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02q_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02q_pytest.log
for c in cfg1 cfg4 cfg3; do
  ST_DEBUG_BUILD=1 ST_DEBUG_TIMELINE=1 timeout 600 python scripts/ab_step.py $c 4 >> gpurun_out/r02q_ab.jsonl 2>> gpurun_out/r02q_ab_$c.err
done
