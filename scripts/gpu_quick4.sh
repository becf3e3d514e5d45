timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scripts/member_times.py --batch 1
python scripts/layer_table.py --batch 1 --models efficientnet_v2_l --top 3 2>&1 | grep -A8 "sum of node"
