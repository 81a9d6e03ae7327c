#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split" > gpurun_out/r02j_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r02j_pytest.log
for c in cfg1 cfg2 cfg4; do
  ST_DEBUG_TIMELINE=1 timeout 900 python scripts/shard_balance.py $c 8 split >> gpurun_out/r02j_shard.jsonl 2>> gpurun_out/r02j_shard.err
done
timeout 600 python bench.py --gpus 2 --config cfg0 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_n2.json 2> gpurun_out/r02j_bench_n2.err
