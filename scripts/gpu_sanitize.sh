#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize_run.py), summaries in gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
CS=/usr/local/cuda/bin/compute-sanitizer
python scripts/sanitize_run.py --quick > gpurun_out/san_plain.txt 2>&1; tail -3 gpurun_out/san_plain.txt
timeout 1500 $CS --tool memcheck --leak-check full --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/san_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -6 gpurun_out/san_memcheck.txt
timeout 1200 $CS --tool synccheck --error-exitcode 9 python scripts/sanitize_run.py --quick > gpurun_out/san_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/san_synccheck.txt
timeout 1500 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python scripts/sanitize_run.py --quick > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -6 gpurun_out/san_racecheck.txt
timeout 900 $CS --tool initcheck --error-exitcode 9 python scripts/sanitize_run.py --quick > gpurun_out/san_initcheck.txt 2>&1; echo "initcheck rc=$?"; tail -4 gpurun_out/san_initcheck.txt
