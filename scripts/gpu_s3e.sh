#!/bin/bash
mkdir -p gpurun_out
for c in cfg4 cfg2; do
  ST_DEBUG_TIMELINE=1 timeout 300 python scripts/shard_probe.py $c 8 3 3 >> gpurun_out/s3e_shard.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/s3e_launches_$c.csv python scripts/shard_probe.py $c 8 3 2 > gpurun_out/s3e_ncu_$c.log 2>&1
done
