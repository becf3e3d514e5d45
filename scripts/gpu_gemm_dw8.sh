#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
for cfg in "DFX_GEMM_DW_BN=32" "DFX_GEMM_DW_BN=16" "DFX_GEMM_DW_BN=64" "DFX_GEMM_DW_BN_PAIR=64"; do
  echo "== $cfg" >> gpurun_out/gdw8.log
  env $cfg timeout 300 python scripts/member_times.py --batch 1 2>&1 | grep -v Warn | grep "efficientnet\|concurrent" >> gpurun_out/gdw8.log
done
done
