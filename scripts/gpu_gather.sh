#!/bin/bash
# e2e staging A/B: thread-pool gather + chunked H2D vs one-thread staging
mkdir -p gpurun_out
nproc > gpurun_out/gather_nproc.txt
timeout 900 python -m pytest tests/test_gpu_zoo.py -x -q -m gpu -k "gather or four_model" > gpurun_out/gather_tests.log 2>&1
for i in 1 2; do
  for g in 0 1; do
    DFX_E2E_GATHER=$g timeout 600 python bench.py --skip-unfused --skip-extra --steps 200 --warmup 5 > gpurun_out/gather_b$g.$i.json 2> gpurun_out/gather_b$g.$i.err
  done
done
