#!/bin/bash
# column depthwise strip target in split precision (batch 32)
Q="python scripts/quick_time.py --batch 32 --steps 20"
for w in 2 1 4 2; do DFX_DW_COL_WAVES=$w $Q --tag "dw waves $w"; done
