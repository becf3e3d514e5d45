timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
bash scripts/gpu_se_tl.sh
python scripts/member_times.py --batch 1
