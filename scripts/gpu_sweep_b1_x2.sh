#!/bin/bash
# batch-1 split-precision knobs re-swept with the new tiling defaults
Q="python scripts/quick_time.py"
for rep in 1 2; do
$Q --tag base
for v in 4 8; do DFX_SPLIT_MIN_STAGES_X2=$v $Q --tag "split_min_stages_x2 $v"; done
DFX_BN_FLOOR_SUBWAVE_X2=256 $Q --tag "bn_floor_subwave 256"
DFX_SPLITK_CLUSTER_MAX=8 $Q --tag "splitk_cluster_max 8"
done
