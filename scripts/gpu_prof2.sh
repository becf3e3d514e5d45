python scripts/layer_table.py --batch 1 --top 30 --json gpurun_out/prof_b1.json 2>&1 | tail -45
python scripts/layer_table.py --batch 32 --top 30 --json gpurun_out/prof_b32.json 2>&1 | tail -45
