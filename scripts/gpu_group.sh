#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_grouped.py -x -q > gpurun_out/tests_grouped.txt 2>&1; tail -25 gpurun_out/tests_grouped.txt
timeout 900 python scripts/group_ab.py > gpurun_out/group_ab.log 2>&1; tail -8 gpurun_out/group_ab.log
