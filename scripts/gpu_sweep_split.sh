#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
Q="python scripts/quick_time.py --precision fp16x2"
$Q --tag base
$Q --models efficientnet_v2_l --tag effnet-alone
for v in 2 3 6; do DFX_SPLIT_MIN_STAGES=$v $Q --tag "split_min_stages=$v"; done
for v in 16 64; do DFX_GEMM_DW_BN=$v DFX_GEMM_DW_BN_PAIR=$v $Q --tag "dw_bn=$v"; done
DFX_SPLITK=kernel $Q --tag "splitk=kernel"
DFX_PRIORITY=0 $Q --tag "priority=0"
python scripts/quick_time.py --precision fp16 --tag fp16-base
