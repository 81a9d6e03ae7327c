#!/bin/bash
# far-field variants (scratch_libs/v*.so, built with VARIANT_FLAGS): A round-1 schedule +
# grade-outer form; B round-1 schedule + column loops; C two batches per warp + column
# loops + 64-entry packed tasks; D round-1 list + 64-entry packed tasks (two per lane)
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg4; do
  for v in vA vB vC vD; do
    ST_LIB_PATH=$PWD/scratch_libs/$v.so timeout 600 python scripts/ab_step.py $c 5 >> gpurun_out/ab_r02.jsonl 2>> gpurun_out/ab_r02.err
  done
done
