#!/bin/bash
# Round-end GPU session (outputs < 64 MiB): tests, bench, reference arm, ncu launch
# list + GEMM traffic at batch 1, full captures of two depthwise-epilogue GEMMs.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/r5_tests.txt
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/launches_b1.csv python scripts/prof_step.py --batch 1 > /dev/null 2>&1
ALGO=$(python scripts/prof_step.py --batch 1 --algo | tail -1)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_kernel -c 600 --csv --log-file gpurun_out/gemm_traffic_b1.csv python scripts/prof_step.py --batch 1 > /dev/null 2>&1
python scripts/summarize_profiles.py traffic gpurun_out/gemm_traffic_b1.csv gpurun_out/gemm_traffic_b1.json $ALGO > /dev/null
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 39 -c 1 -o gpurun_out/gemm_dw_m2_b1 python scripts/prof_step.py --batch 1 --models efficientnet_v2_l > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 93 -c 1 -o gpurun_out/gemm_dw_7x7_b1 python scripts/prof_step.py --batch 1 --models efficientnet_v2_l > /dev/null 2>&1
ls -la gpurun_out
