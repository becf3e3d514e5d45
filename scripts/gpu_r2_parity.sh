#!/bin/bash
# Round-2: GPU tests (incl. the new lifecycle + north-star parity tests) and a bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -k "north_star" > gpurun_out/tests_ns.txt 2>&1; tail -15 gpurun_out/tests_ns.txt
timeout 1500 python -m pytest tests -q -m gpu -k "not north_star" > gpurun_out/tests.txt 2>&1; tail -15 gpurun_out/tests.txt
timeout 1200 python bench.py --steps 100 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -5 gpurun_out/bench.err
head -c 1500 gpurun_out/bench.json
