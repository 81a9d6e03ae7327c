#!/bin/bash
# two-target far field: full GPU suite, then the far-heavy configurations
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02d_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02d_pytest.log
for c in cfg1 cfg2 cfg4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02d_bench_$c.json 2> gpurun_out/r02d_bench_$c.err
done
