timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scripts/gpu_zoo_timing.py 2>&1 | grep "B="
python scripts/layer_table.py --batch 1 --top 5 2>&1 | tail -16
