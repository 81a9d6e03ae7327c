#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "treecode or config_parity or near" > gpurun_out/s3s_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s3s_pytest.log
for c in cfg1 cfg4 cfg2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3s_bench_$c.json 2> gpurun_out/s3s_bench_$c.err
  ST_LIB_PATH=$PWD/paper_1811_12498_b200/libstokestree_b200_v1.so timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3s_bench_v1_$c.json 2> gpurun_out/s3s_bench_v1_$c.err
done
