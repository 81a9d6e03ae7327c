#!/bin/bash
# round-2 session-3 evidence: bench lines for every configuration, the reference arm, the launch
# list of the bench command, full ncu captures of the dominant kernels, N-shard projections
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02s4_cfg1.json 2> gpurun_out/bench_r02s4_cfg1.err
for c in cfg0 cfg2 cfg4 cfg3; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_r02s4_$c.json 2> gpurun_out/bench_r02s4_$c.err
done
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02s4_reference.json 2> gpurun_out/bench_r02s4_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02s4_bench_cfg1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r02s4_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_neval|k_far_list|k_feval" -c 3 -o gpurun_out/r02s4_kernels_cfg1 python scripts/profile_step.py cfg1 1 > gpurun_out/ncu_r02s4_full.log 2>&1
for c in cfg1 cfg2 cfg4 cfg3; do
  for k in 2 4 8; do
    timeout 1200 python scripts/shard_balance.py $c $k split >> gpurun_out/shard_r02s4.jsonl 2>> gpurun_out/shard_r02s4.err
  done
done
ncu --set full --clock-control none --import-source on -k regex:"k_far_list|k_feval|k_nwalk" -c 4 -o gpurun_out/r02s4_kernels_cfg4 python scripts/profile_step.py cfg4 1 > gpurun_out/ncu_r02s4_cfg4.log 2>&1
