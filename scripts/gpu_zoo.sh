timeout 600 python scripts/gpu_zoo_timing.py 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_zoo.py -x -q -m gpu 2>&1 | tail -20
