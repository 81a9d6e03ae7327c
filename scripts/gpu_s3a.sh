#!/bin/bash
# session 3: keyed tree build -- tree parity tests, build phase times (keyed vs partition), cfg1/cfg4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "tree or config_parity or treecode" > gpurun_out/s3a_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3a_pytest.log
for c in cfg1 cfg4 cfg3; do
  ST_DEBUG_BUILD=1 timeout 300 python scripts/probe_cfg.py $c 3 >> gpurun_out/s3a_build.log 2>&1
  ST_TREE_PARTITION=1 ST_DEBUG_BUILD=1 timeout 300 python scripts/probe_cfg.py $c 3 >> gpurun_out/s3a_build_part.log 2>&1
done
for c in cfg1 cfg4 cfg2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3a_bench_$c.json 2> gpurun_out/s3a_bench_$c.err
done
