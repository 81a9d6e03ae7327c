#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02r_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02r_pytest.log
for c in cfg2 cfg4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02r_bench_$c.json 2>/dev/null
  for cs in 8192 2048; do
    ST_COUNT_SAMPLES=$cs timeout 900 python scripts/shard_balance.py $c 8 split >> gpurun_out/r02r_shard_$cs.jsonl 2>> gpurun_out/r02r_shard.err
  done
done
