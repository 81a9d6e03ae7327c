#!/bin/bash
# run-time column loops: far-field benches, GPU suite, far flop count (ncu)
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_$c.json 2> gpurun_out/r02f_bench_$c.err
done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02f_pytest.log
ncu --set full --clock-control none --import-source on -k regex:"k_far_list|k_feval" -c 2 -o gpurun_out/r02f_far_cfg2 python scripts/profile_step.py cfg2 1 > gpurun_out/r02f_ncu2.log 2>&1
