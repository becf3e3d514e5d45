#!/bin/bash
# depthwise A/B: one row (build/ab/libdfx_ahead1.so) vs two rows in flight (in-tree libdfx.so)
C="1056:14:32:3:1,1344:14:32:3:1,3840:7:32:3:1,768:28:32:3:2,384:56:32:3:1,64:112:32:3:1,240:28:32:3:1"
python -m pytest tests/test_gpu_parity.py -q -k depthwise 2>&1 | tail -1
echo "== ahead 1"; DFX_LIBRARY=build/ab/libdfx_ahead1.so python scripts/dw_micro.py --cases $C
echo "== ahead 2"; python scripts/dw_micro.py --cases $C
for rep in 1 2; do
DFX_LIBRARY=build/ab/libdfx_ahead1.so python scripts/quick_time.py --batch 32 --precision fp16 --steps 30 --tag "ahead1"
python scripts/quick_time.py --batch 32 --precision fp16 --steps 30 --tag "ahead2"
done
