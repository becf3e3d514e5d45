#!/bin/bash
# full GPU suite, Table V replay, full bench line + reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/tests.txt 2>&1; tail -5 gpurun_out/tests.txt
timeout 1200 python scripts/table5_replay.py > gpurun_out/table5.log 2>&1; tail -45 gpurun_out/table5.log | head -3
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; head -c 300 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 8 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 400 gpurun_out/bench_ref.json
