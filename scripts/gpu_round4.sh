#!/bin/bash
# Round-end style GPU session: tests, bench, ncu launch list + GEMM traffic + full captures.
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/launches_b1.csv python scripts/prof_step.py --batch 1 > /dev/null 2>&1
ALGO=$(python scripts/prof_step.py --batch 1 --algo | tail -1)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_kernel -c 600 --csv --log-file gpurun_out/gemm_traffic_b1.csv python scripts/prof_step.py --batch 1 > /dev/null 2>&1
python scripts/summarize_profiles.py traffic gpurun_out/gemm_traffic_b1.csv gpurun_out/gemm_traffic_b1.json $ALGO > /dev/null
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 40 -c 1 -o gpurun_out/gemm_effnet_b1 python scripts/prof_step.py --batch 1 --models efficientnet_v2_l > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/gemm_persist_expand_b32 python scripts/gemm_micro.py --cases 224:1344:14:32:1 --act silu > /dev/null 2>&1
ls gpurun_out


ncu --set full --clock-control none --import-source on -k regex:gemm -s 6 -c 1 -o gpurun_out/gemm_vgg_conv_b32 python scripts/prof_step.py --batch 32 --models vgg16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dwconv -c 1 -o gpurun_out/dw_s5_b32 python scripts/dw_micro.py --cases 1344:14:32:3:1 > /dev/null 2>&1
