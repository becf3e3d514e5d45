#!/bin/bash
# Round-2 close: every GPU test, smoke, the bench line, ncu launch list + GEMM DRAM traffic
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/tests.txt 2>&1; tail -3 gpurun_out/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench_close.json 2> gpurun_out/bench_close.err; tail -2 gpurun_out/bench_close.err
head -c 300 gpurun_out/bench_close.json; echo
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_close_launches_b1_fp16x2.csv python scripts/prof_step.py --precision fp16x2 > /dev/null 2>&1
python scripts/summarize_profiles.py launches gpurun_out/r02_close_launches_b1_fp16x2.csv > gpurun_out/r02_close_launches_b1_fp16x2_summary.txt; head -12 gpurun_out/r02_close_launches_b1_fp16x2_summary.txt
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:gemm_kernel --clock-control none --csv --log-file gpurun_out/r02_close_gemm_traffic_b1_fp16x2.csv python scripts/prof_step.py --precision fp16x2 > /dev/null 2>&1
ALGO=$(python scripts/prof_step.py --precision fp16x2 --algo | tail -1)
python scripts/summarize_profiles.py traffic gpurun_out/r02_close_gemm_traffic_b1_fp16x2.csv gpurun_out/r02_gemm_traffic_b1_fp16x2.json $ALGO; cat gpurun_out/r02_gemm_traffic_b1_fp16x2.json
