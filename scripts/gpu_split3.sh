#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_grouped.py -x -q > gpurun_out/tests_split.txt 2>&1; tail -3 gpurun_out/tests_split.txt
Q="python scripts/quick_time.py --precision fp16x2"
$Q --tag base
$Q --models efficientnet_v2_l --tag effnet-alone
DFX_SPLIT_MIN_STAGES=6 $Q --tag "split_min_stages=6"
DFX_SPLIT_MIN_STAGES=8 $Q --tag "split_min_stages=8"
python scripts/quick_time.py --precision fp16x2 --batch 32 --steps 20 --tag b32
timeout 1200 python -m pytest tests/test_gpu_north_star.py -q -k "split" > gpurun_out/tests_ns_split.txt 2>&1; tail -3 gpurun_out/tests_ns_split.txt
