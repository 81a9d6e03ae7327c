#!/bin/bash
# compute-sanitizer on the cfg0 workload (scripts/sanitize_cfg0.py), one tool at a time;
# logs under gpurun_out/ (summaries copied to profiles/)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cfg0.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc $?" >> gpurun_out/sanitize_$tool.log
done
