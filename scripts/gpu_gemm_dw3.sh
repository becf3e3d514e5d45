#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
for cfg in "DFX_GEMM_DW=0" "DFX_GEMM_DW=1" "DFX_GEMM_DW_MODE=single"; do
  echo "== $cfg" >> gpurun_out/gdw3.log
  env $cfg timeout 300 python scripts/member_times.py --batch 1 2>&1 | grep -v Warn | grep "efficientnet\|mobilenet\|concurrent" >> gpurun_out/gdw3.log
done
done
