#!/bin/bash
# Round-2 headline (fp16x2) bench line + ncu evidence: launch list, GEMM DRAM traffic, one full capture
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; head -c 400 gpurun_out/bench.json; echo
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_b1_fp16x2.csv python scripts/prof_step.py --precision fp16x2 > /dev/null 2>&1
python scripts/summarize_profiles.py launches gpurun_out/r02_launches_b1_fp16x2.csv > gpurun_out/r02_launches_b1_fp16x2_summary.txt; head -12 gpurun_out/r02_launches_b1_fp16x2_summary.txt
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:gemm_kernel --clock-control none --csv --log-file gpurun_out/r02_gemm_traffic_b1_fp16x2.csv python scripts/prof_step.py --precision fp16x2 > /dev/null 2>&1
ALGO=$(python scripts/prof_step.py --precision fp16x2 --algo | tail -1)
python scripts/summarize_profiles.py traffic gpurun_out/r02_gemm_traffic_b1_fp16x2.csv gpurun_out/r02_gemm_traffic_b1_fp16x2.json $ALGO; cat gpurun_out/r02_gemm_traffic_b1_fp16x2.json
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:gemm_kernel --launch-skip 300 -c 1 -o gpurun_out/r02_gemm_effnet_b1_fp16x2 python scripts/prof_step.py --precision fp16x2 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
python scripts/summarize_profiles.py rep gpurun_out/r02_gemm_effnet_b1_fp16x2.ncu-rep > gpurun_out/r02_ncu_summary.txt; cat gpurun_out/r02_ncu_summary.txt
