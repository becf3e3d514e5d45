#!/bin/bash
# Round-2 GPU session: build check, GPU tests, bench line (N=1), reference arm.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/tests.txt 2>&1; tail -5 gpurun_out/tests.txt
if [ -z "$NO_BENCH" ]; then
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
head -c 3000 gpurun_out/bench.json
fi
