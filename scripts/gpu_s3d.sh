#!/bin/bash
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg4; do
  ST_DEBUG_TIMELINE=1 timeout 300 python scripts/probe_cfg.py $c 3 >> gpurun_out/s3d_timeline.log 2>&1
  ST_AUX_PRIORITY=1 ST_DEBUG_TIMELINE=1 timeout 300 python scripts/probe_cfg.py $c 3 >> gpurun_out/s3d_timeline_prio.log 2>&1
  ST_MOMENTS_INLINE=1 ST_DEBUG_TIMELINE=1 timeout 300 python scripts/probe_cfg.py $c 3 >> gpurun_out/s3d_timeline_inline.log 2>&1
done
