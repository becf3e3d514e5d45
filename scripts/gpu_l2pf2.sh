#!/bin/bash
# A/B: L2 prefetch depth (DFX_L2_PREFETCH_DEPTH 1 / 2)
for rep in 1 2 3; do
for d in 1 2; do
DFX_L2_PREFETCH_DEPTH=$d python scripts/quick_time.py --tag "depth=$d"
done
done
for d in 1 2; do DFX_L2_PREFETCH_DEPTH=$d python scripts/quick_time.py --tag "depth=$d fp16" --precision fp16; done
