#!/bin/bash
# depthwise A/B: column-strip kernel strip targets (DFX_DW_COL_WAVES) vs the tile kernel
C="1056:14:32:3:1,1344:14:32:3:1,3840:7:32:3:1,768:28:32:3:2,384:56:32:3:1,64:112:32:3:1,240:28:32:3:1"
python -m pytest tests/test_gpu_parity.py -q -k depthwise 2>&1 | tail -2
for w in 1 2 3; do echo "== col waves $w"; DFX_DW_COL_WAVES=$w python scripts/dw_micro.py --cases $C; done
for w in 1 2 3; do DFX_DW_COL_WAVES=$w python scripts/quick_time.py --batch 32 --precision fp16 --steps 30 --tag "col w$w"; done
DFX_DW_COL=0 python scripts/quick_time.py --batch 32 --precision fp16 --steps 30 --tag "tile"
DFX_DW_COL_WAVES=2 python scripts/quick_time.py --batch 32 --precision fp16x2 --steps 30 --tag "col w2"
DFX_DW_COL=0 python scripts/quick_time.py --batch 32 --precision fp16x2 --steps 30 --tag "tile"
