#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3n_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3n_pytest.log
for c in cfg4 cfg2 cfg1; do
  ST_DEBUG_TIMELINE=1 python scripts/probe_cfg.py $c 3 2>&1 | grep timeline | tail -1 >> gpurun_out/s3n_tl.log
  ST_MOMENTS_EPT=2 ST_DEBUG_TIMELINE=1 python scripts/probe_cfg.py $c 3 2>&1 | grep timeline | tail -1 >> gpurun_out/s3n_tl.log
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3n_bench_$c.json 2> gpurun_out/s3n_bench_$c.err
done
ncu --set full --clock-control none -k regex:"k_moments" -c 1 -o gpurun_out/s3n_moments_cfg4 python scripts/probe_cfg.py cfg4 1 > /dev/null 2>&1
