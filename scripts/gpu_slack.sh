#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
for cfg in "DFX_SLACK_SPLIT_MAX=0" "DFX_SLACK_SPLIT_MAX=3" "DFX_SLACK_SPLIT_MAX=4" "DFX_SLACK_SPLIT_MAX=6" "DFX_SLACK_SPLIT_MAX=8"; do
  echo "== $cfg" >> gpurun_out/slack.log
  env $cfg timeout 300 python scripts/member_times.py --batch 1 2>&1 | grep -v Warn | grep "concurrent" >> gpurun_out/slack.log
done
done
