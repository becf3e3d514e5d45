python scripts/gemm_micro.py 2>&1 | tail -12
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scripts/layer_table.py --batch 1 --top 25 2>&1 | tail -36
python scripts/layer_table.py --batch 32 --top 12 2>&1 | tail -22
