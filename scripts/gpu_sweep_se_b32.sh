#!/bin/bash
# SE knobs at batch 32 in split precision (they were tuned in fp16)
Q="python scripts/quick_time.py --batch 32 --steps 20"
$Q --tag base
DFX_SE_UNSTAGED_BATCH=64 $Q --tag "se staged at b32"
DFX_SE_XTILE_BATCH=64 $Q --tag "se x tile at b32"
DFX_SE_UNSTAGED_BATCH=64 DFX_SE_XTILE_BATCH=64 $Q --tag "both"
$Q --tag base
