#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_split.py -x -q > gpurun_out/tests_split.txt 2>&1; tail -3 gpurun_out/tests_split.txt
timeout 1200 python -m pytest tests/test_gpu_north_star.py -q -k "split" > gpurun_out/tests_ns_split.txt 2>&1; tail -3 gpurun_out/tests_ns_split.txt
PRECS="fp16x2" bash scripts/gpu_bench_prec.sh
