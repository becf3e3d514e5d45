#!/bin/bash
# 16-bit tiling knobs re-swept after the column depthwise kernel (fp16, batch 32)
Q="python scripts/quick_time.py --batch 32 --steps 20 --precision fp16"
$Q --tag base
for w in 0.75 1 1.5; do DFX_PERSIST_MIN_WAVES=$w $Q --tag "persist_min_waves $w"; done
DFX_BN_FLOOR_MANY_M=128 $Q --tag "bn_floor 128"
$Q --tag base
