timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scripts/member_times.py --batch 1
python scripts/member_times.py --batch 32 | tail -2
bash scripts/gpu_timeline.sh
