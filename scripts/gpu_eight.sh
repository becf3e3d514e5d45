#!/bin/bash
# 8-model-config CNNs on the GPU: parity + per-member timings.
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_zoo.py -x -q 2>&1 | tail -5
timeout 600 python scripts/member_times.py --set eight --batch 1
timeout 600 python scripts/member_times.py --set eight --batch 8
