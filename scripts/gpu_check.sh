#!/bin/bash
# checkpoint on the box with the in-tree libdfx.so: GPU tests, smoke, bench line
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-2000} python -m pytest tests -q -m gpu ${PYTEST_ARGS} > gpurun_out/tests.txt 2>&1; tail -5 gpurun_out/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
if [ -z "$NO_BENCH" ]; then
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
head -c 1500 gpurun_out/bench.json
fi
