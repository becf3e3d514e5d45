#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_split.py -x -q > gpurun_out/tests_split.txt 2>&1; tail -3 gpurun_out/tests_split.txt
Q="python scripts/quick_time.py --precision fp16x2"
$Q --tag base
$Q --batch 32 --steps 20 --tag b32
python scripts/layer_table.py --batch 32 --top 30 --precision fp16x2 > gpurun_out/lt32_fp16x2.txt 2>&1; head -45 gpurun_out/lt32_fp16x2.txt
