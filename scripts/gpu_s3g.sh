#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3g_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3g_pytest.log
for c in cfg1 cfg4; do
  ST_DEBUG_BUILD=1 ST_DEBUG_TIMELINE=1 timeout 300 python scripts/probe_cfg.py $c 3 >> gpurun_out/s3g_build.log 2>&1
done
for c in cfg1 cfg4 cfg2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3g_bench_$c.json 2> gpurun_out/s3g_bench_$c.err
done
for c in cfg4 cfg2; do
  timeout 900 python scripts/shard_balance.py $c 8 split >> gpurun_out/s3g_balance.jsonl 2>> gpurun_out/s3g_balance.err
done
