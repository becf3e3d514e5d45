#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
C="224:1344:14:32:1,256:1344:14:32:1,192:1344:14:32:1,96:384:28:32:1,128:384:28:32:1,160:960:14:32:1,64:256:56:32:3"
echo "== default"; timeout 300 python scripts/gemm_micro.py --cases $C --act silu | awk '{print $1,$2,$3,$4,$(NF-3),$(NF-1)}'
echo "== waste 0.5"; DFX_CB_WASTE=0.5 timeout 300 python scripts/gemm_micro.py --cases $C --act silu | awk '{print $1,$2,$3,$4,$(NF-3),$(NF-1)}'
echo "== b32 waste 0.5"; DFX_CB_WASTE=0.5 timeout 300 python scripts/member_times.py --batch 32
echo "== b1 waste 0.5"; DFX_CB_WASTE=0.5 timeout 300 python scripts/member_times.py --batch 1
