#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "shard or ipc or split or device or multi" > gpurun_out/s3f_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3f_pytest.log
for c in cfg4 cfg2; do
  ST_DEBUG_TIMELINE=1 timeout 300 python scripts/shard_probe.py $c 8 3 3 >> gpurun_out/s3f_shard.log 2>&1
  timeout 900 python scripts/shard_balance.py $c 8 split >> gpurun_out/s3f_balance.jsonl 2>> gpurun_out/s3f_balance.err
done
