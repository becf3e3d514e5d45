#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
C="64:256:56:32:3,256:64:56:32:1,32:32:112:32:3,512:512:28:32:3,224:1344:14:32:1,96:384:28:32:1"
echo "== default"; timeout 300 python scripts/gemm_micro.py --cases $C
echo "== silu"; timeout 300 python scripts/gemm_micro.py --cases $C --act silu
echo "== M2=0 silu"; DFX_GEMM_M2=0 timeout 300 python scripts/gemm_micro.py --cases $C --act silu
