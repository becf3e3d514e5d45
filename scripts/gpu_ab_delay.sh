#!/bin/bash
# A/B: members with slack start after the critical chain is f of the way through (DFX_SLACK_DELAY)
export DFX_SLACK_FRAC=0.5
for rep in 1 2; do
python scripts/quick_time.py --tag "no delay"
for f in 0.3 0.5 0.7; do
DFX_SLACK_DELAY=$f python scripts/quick_time.py --tag "delay $f"
done
done
DFX_SLACK_DELAY=0.5 python scripts/quick_time.py --tag "delay 0.5 fp16" --precision fp16
python scripts/quick_time.py --tag "no delay fp16" --precision fp16
