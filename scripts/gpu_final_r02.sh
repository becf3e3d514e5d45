#!/bin/bash
# round-2 closing measurements: bench line (N=1) + ncu of the column depthwise kernel at batch 32
# (the tile kernel baseline: profiles/r01_dwconv_effnet_s5_b32.ncu-rep)
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err
head -c 400 gpurun_out/bench_final.json; echo
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:dwconv_col -c 1 -o gpurun_out/r02_dwcol_b32_1344 -f \
  python scripts/dw_micro.py --cases 1344:14:32:3:1 > gpurun_out/ncu_dwcol.log 2>&1; tail -2 gpurun_out/ncu_dwcol.log
ls -la gpurun_out/*.ncu-rep
