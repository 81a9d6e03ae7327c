#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02p_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02p_pytest.log
for c in cfg1 cfg4 cfg3; do
  ST_DEBUG_BUILD=1 ST_DEBUG_TIMELINE=1 timeout 600 python scripts/ab_step.py $c 4 >> gpurun_out/r02p_ab.jsonl 2>> gpurun_out/r02p_ab_$c.err
done
for c in cfg1 cfg2 cfg4; do
  timeout 900 python scripts/shard_balance.py $c 8 split >> gpurun_out/r02p_shard.jsonl 2>> gpurun_out/r02p_shard.err
done
