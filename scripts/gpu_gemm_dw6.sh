#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_zoo.py -x -q -m gpu -k "depthwise or four_model" 2>&1 | tail -15 > gpurun_out/gdw6_tests.txt
for r in 1 2; do
for cfg in "DFX_GEMM_DW_PAIR=cluster" "DFX_GEMM_DW_PAIR=m2"; do
  echo "== $cfg" >> gpurun_out/gdw6.log
  env $cfg timeout 300 python scripts/member_times.py --batch 1 2>&1 | grep -v Warn | grep "efficientnet\|mobilenet\|concurrent" >> gpurun_out/gdw6.log
done
done
