#!/bin/bash
# session 3: launch lists at cfg4 / cfg2 (keyed build), shard timelines, the cfg2 p-sweep
mkdir -p gpurun_out
for c in cfg4 cfg2; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s3b_launches_$c.csv python scripts/probe_cfg.py $c 2 > gpurun_out/s3b_ncu_$c.log 2>&1
done
for c in cfg4 cfg2; do
  ST_DEBUG_TIMELINE=1 ST_DEBUG_BUILD=1 timeout 900 python scripts/shard_balance.py $c 8 split >> gpurun_out/s3b_shard.jsonl 2>> gpurun_out/s3b_shard_$c.err
done
timeout 1500 python scripts/sweep_cfg2_r02.py > gpurun_out/s3b_psweep.log 2>&1
cp profiles/r02_cfg2_psweep.json gpurun_out/ 2>/dev/null
