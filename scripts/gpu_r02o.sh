#!/bin/bash
mkdir -p gpurun_out
for pr in 1 0; do
for c in cfg1 cfg2 cfg4; do
  ST_AUX_PRIORITY=$pr ST_DEBUG_TIMELINE=1 timeout 600 python scripts/ab_step.py $c 5 >> gpurun_out/r02o_ab_$pr.jsonl 2>> gpurun_out/r02o_ab_$pr.err
done
done
