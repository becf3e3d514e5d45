#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_lifecycle.py tests/test_gpu_manager.py -x -q > gpurun_out/tests_life.txt 2>&1; tail -5 gpurun_out/tests_life.txt
timeout 1200 python scripts/table5_replay.py > gpurun_out/table5.log 2>&1; tail -45 gpurun_out/table5.log
