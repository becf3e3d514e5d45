#!/bin/bash
# depthwise A/B: __launch_bounds__(128) (165 regs, 3 blocks/SM) vs (128, 4) (128 regs + spills)
C="1056:14:32:3:1,1344:14:32:3:1,3840:7:32:3:1,768:28:32:3:2,384:56:32:3:1,64:112:32:3:1,240:28:32:3:1"
for v in base lb4; do echo "== $v"; DFX_LIBRARY=build/ab/libdfx_$v.so python scripts/dw_micro.py --cases $C; done
for rep in 1 2; do for v in base lb4; do DFX_LIBRARY=build/ab/libdfx_$v.so python scripts/quick_time.py --batch 32 --precision fp16 --steps 30 --tag "$v"; done; done
