#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
C="64:256:56:32:3,256:64:56:32:1,32:32:112:32:3,512:512:28:32:3,224:1344:14:32:1,96:384:28:32:1"
echo "== default"; timeout 300 python scripts/gemm_micro.py --cases $C
echo "== M2=0"; DFX_GEMM_M2=0 timeout 300 python scripts/gemm_micro.py --cases $C
echo "== PERSIST=0"; DFX_GEMM_PERSIST=0 timeout 300 python scripts/gemm_micro.py --cases $C
echo "== PERSIST=0 M2=0"; DFX_GEMM_PERSIST=0 DFX_GEMM_M2=0 timeout 300 python scripts/gemm_micro.py --cases $C
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/micro_s2 python scripts/gemm_micro.py --cases 64:256:56:32:3 > /dev/null 2>&1
ls gpurun_out
