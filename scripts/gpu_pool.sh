#!/bin/bash
# arena pool: GPU tests, then the full bench (swap-in numbers) twice
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -4 > gpurun_out/pool_tests.txt
timeout 1200 python bench.py > gpurun_out/pool_bench1.json 2> gpurun_out/pool_bench1.err
DFX_ARENA_POOL=0 timeout 1200 python bench.py --skip-unfused > gpurun_out/pool_bench0.json 2> gpurun_out/pool_bench0.err
