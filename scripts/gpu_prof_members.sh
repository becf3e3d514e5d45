mkdir -p gpurun_out
python scripts/member_times.py --batch 1 --precision fp16x2 > gpurun_out/member_b1_x2.txt 2>&1
python scripts/member_times.py --batch 1 --precision fp16 > gpurun_out/member_b1_f16.txt 2>&1
python scripts/layer_table.py --batch 1 --precision fp16x2 --models efficientnet_v2_l --top 10 --json gpurun_out/eff_b1_x2.json > gpurun_out/eff_b1_x2.txt 2>&1
python scripts/layer_table.py --batch 32 --precision fp16x2 --top 60 --json gpurun_out/b32_x2.json > gpurun_out/b32_x2.txt 2>&1
python scripts/layer_table.py --batch 32 --precision fp16 --top 60 --json gpurun_out/b32_f16.json > gpurun_out/b32_f16.txt 2>&1
cat gpurun_out/member_b1_x2.txt gpurun_out/member_b1_f16.txt; head -12 gpurun_out/b32_x2.txt
