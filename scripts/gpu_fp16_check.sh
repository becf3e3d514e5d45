#!/bin/bash
for rep in 1 2; do
python scripts/quick_time.py --batch 32 --steps 20 --precision fp16 --tag "fp16 b32"
DFX_PERSIST_MIN_WAVES_X2=2 DFX_BN_FLOOR_SUBWAVE_X2=64 python scripts/quick_time.py --batch 32 --steps 20 --precision fp16 --tag "fp16 b32 old-x2-knobs"
done
