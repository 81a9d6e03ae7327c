#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3o_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3o_pytest.log
for c in cfg1 cfg4 cfg2; do
  ST_DEBUG_TIMELINE=1 python scripts/probe_cfg.py $c 3 2>&1 | grep timeline | tail -1 >> gpurun_out/s3o_tl.log
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3o_bench_$c.json 2> gpurun_out/s3o_bench_$c.err
  ST_WALK_RECORD=0 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3o_bench_norec_$c.json 2> gpurun_out/s3o_bench_norec_$c.err
done
