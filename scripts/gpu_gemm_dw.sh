#!/bin/bash
# GEMM + depthwise epilogue: parity, then bench A/B (off / bn 32 / bn 16)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_zoo.py -x -q -m gpu -k "depthwise or four_model or gather" > gpurun_out/gdw_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gdw_tests.log
for i in 1 2; do
  DFX_GEMM_DW=0 timeout 600 python bench.py --skip-unfused --skip-extra --steps 200 --warmup 5 > gpurun_out/gdw_off.$i.json 2> gpurun_out/gdw_off.$i.err
  timeout 600 python bench.py --skip-unfused --skip-extra --steps 200 --warmup 5 > gpurun_out/gdw_32.$i.json 2> gpurun_out/gdw_32.$i.err
  DFX_GEMM_DW_BN=16 timeout 600 python bench.py --skip-unfused --skip-extra --steps 200 --warmup 5 > gpurun_out/gdw_16.$i.json 2> gpurun_out/gdw_16.$i.err
done
