#!/bin/bash
mkdir -p gpurun_out
for cfg in "DFX_GEMM_DW=0" "DFX_GEMM_DW=1" "DFX_GEMM_DW_MODE=nosplit"; do
  echo "== $cfg" >> gpurun_out/gdw2.log
  env $cfg timeout 300 python scripts/member_times.py --batch 1 >> gpurun_out/gdw2.log 2>&1
done
for i in 1 2; do
  DFX_GEMM_DW_MODE=nosplit timeout 600 python bench.py --skip-unfused --skip-extra --steps 200 --warmup 5 > gpurun_out/gdw_ns.$i.json 2> gpurun_out/gdw_ns.$i.err
  DFX_GEMM_DW=0 timeout 600 python bench.py --skip-unfused --skip-extra --steps 200 --warmup 5 > gpurun_out/gdw_off.$i.json 2> gpurun_out/gdw_off.$i.err
done
