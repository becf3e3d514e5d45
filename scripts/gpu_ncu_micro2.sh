#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/micro_expand_silu python scripts/gemm_micro.py --cases 224:1344:14:32:1 --act silu > /dev/null 2>&1
DFX_GEMM_PERSIST=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/micro_expand_silu_np python scripts/gemm_micro.py --cases 224:1344:14:32:1 --act silu > /dev/null 2>&1
ls gpurun_out
