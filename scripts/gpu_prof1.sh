ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/launches_b1.csv python scripts/prof_step.py --batch 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/launches_b32.csv python scripts/prof_step.py --batch 32 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 40 -c 2 -o gpurun_out/gemm_b32 python scripts/prof_step.py --batch 32 --models vgg16 > /dev/null 2>&1
ls -la gpurun_out
