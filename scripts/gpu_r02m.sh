#!/bin/bash
mkdir -p gpurun_out
for c in cfg1 cfg4 cfg3; do
  ST_DEBUG_BUILD=1 ST_DEBUG_TIMELINE=1 timeout 600 python scripts/profile_step.py $c 3 > gpurun_out/r02m_build_$c.log 2>&1
done
