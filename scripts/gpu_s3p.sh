#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3p_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3p_pytest.log
for c in cfg1 cfg4 cfg2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3p_bench_$c.json 2> gpurun_out/s3p_bench_$c.err
done
