python scripts/gemm_micro.py 2>&1 | tail -12
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 2 -o gpurun_out/gemm_slow python scripts/gemm_micro.py --cases 96:192:28:1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 2 -o gpurun_out/gemm_fast python scripts/gemm_micro.py --cases 96:48:28:1 > /dev/null 2>&1
ls gpurun_out
