#!/bin/bash
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg4; do
  ST_DEBUG_TIMELINE=1 timeout 900 python scripts/shard_balance.py $c 8 > gpurun_out/r02h_shard_$c.log 2>&1
done
