#!/bin/bash
# round-2 first GPU pass: tests, bench (N=1 and the N=2 self-launch), reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02a_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench_cfg1.json 2> gpurun_out/r02a_bench_cfg1.err
timeout 600 python bench.py --gpus 2 --config cfg0 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_n2.json 2> gpurun_out/r02a_bench_n2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02a_ref_cfg1.json 2> gpurun_out/r02a_ref_cfg1.err
