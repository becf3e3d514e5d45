#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/micro_s2_silu python scripts/gemm_micro.py --cases 64:256:56:32:3 --act silu > /dev/null 2>&1
DFX_GEMM_M2=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/micro_s2_silu_persist python scripts/gemm_micro.py --cases 64:256:56:32:3 --act silu > /dev/null 2>&1
ls gpurun_out
