#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s3u_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3u_pytest.log
for c in cfg1 cfg4 cfg2; do
  ST_DEBUG_TIMELINE=1 python scripts/probe_cfg.py $c 3 2>&1 | grep timeline | tail -1 >> gpurun_out/s3u_tl.log
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3u_bench_$c.json 2> gpurun_out/s3u_bench_$c.err
done
