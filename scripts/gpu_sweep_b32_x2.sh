#!/bin/bash
# host-side tiling knobs re-swept for split precision (they were tuned in fp16)
Q="python scripts/quick_time.py --batch 32 --steps 20"
$Q --tag base
for w in 0.5 0.75 1 1.5; do DFX_PERSIST_MIN_WAVES=$w $Q --tag "persist_min_waves $w"; done
DFX_PERSIST_MIN_WAVES=1 DFX_BN_FLOOR_MANY_M=128 $Q --tag "pmw 1 + bn_floor 128"
DFX_PERSIST_MIN_WAVES=0.75 DFX_BN_FLOOR_MANY_M=128 $Q --tag "pmw 0.75 + bn_floor 128"
DFX_PERSIST_MIN_WAVES=1 DFX_BN_FLOOR_MANY_M=96 $Q --tag "pmw 1 + bn_floor 96"
python scripts/quick_time.py --tag "b1 base"
DFX_PERSIST_MIN_WAVES=1 python scripts/quick_time.py --tag "b1 pmw 1"
DFX_PERSIST_MIN_WAVES=1 DFX_BN_FLOOR_MANY_M=128 python scripts/quick_time.py --tag "b1 pmw1 bnf128"
DFX_PERSIST_MIN_WAVES=1 DFX_BN_FLOOR_MANY_M=128 $Q --tag "bf16x2 pmw1 bnf128" --precision bf16x2
$Q --tag "bf16x2 base" --precision bf16x2
