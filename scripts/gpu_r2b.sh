#!/bin/bash
# Round-2 session B: racecheck re-run, Table V replay, full bench line (all blocks)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python scripts/sanitize_run.py --quick > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.txt
timeout 1200 python scripts/table5_replay.py > gpurun_out/table5.log 2>&1; tail -40 gpurun_out/table5.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; head -c 600 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 8 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 800 gpurun_out/bench_ref.json
