timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/launches_b1.csv python scripts/prof_step.py --batch 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 13 -c 1 -o gpurun_out/gemm_fc6_b1 python scripts/prof_step.py --batch 1 --models vgg16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 1 -o gpurun_out/gemm_conv3_b32 python scripts/prof_step.py --batch 32 --models vgg16 > /dev/null 2>&1
ls gpurun_out; cat gpurun_out/bench.json | cut -c1-1500
