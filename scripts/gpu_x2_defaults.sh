#!/bin/bash
# split-precision tiling defaults (PERSIST_MIN_WAVES_X2 0.75, BN_FLOOR_SUBWAVE_X2 128) vs the old ones
python -m pytest tests/test_gpu_split.py tests/test_gpu_north_star.py -q -x 2>&1 | tail -2
for rep in 1 2; do
python scripts/quick_time.py --tag "new b1"
DFX_PERSIST_MIN_WAVES_X2=2 DFX_BN_FLOOR_SUBWAVE_X2=64 python scripts/quick_time.py --tag "old b1"
python scripts/quick_time.py --batch 32 --steps 20 --tag "new b32"
DFX_PERSIST_MIN_WAVES_X2=2 DFX_BN_FLOOR_SUBWAVE_X2=64 python scripts/quick_time.py --batch 32 --steps 20 --tag "old b32"
done
DFX_BN_FLOOR_SUBWAVE_X2=64 python scripts/quick_time.py --tag "pmw.75 only b1"
DFX_BN_FLOOR_SUBWAVE_X2=64 python scripts/quick_time.py --batch 32 --steps 20 --tag "pmw.75 only b32"
python scripts/quick_time.py --tag "new bf16x2 b1" --precision bf16x2
python scripts/quick_time.py --tag "new fp16 b1 (unchanged)" --precision fp16
