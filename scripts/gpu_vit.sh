#!/bin/bash
# ViT kernels + 8-model config on the GPU: parity + per-member timings.
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_vit.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_zoo.py -x -q 2>&1 | tail -5
timeout 600 python scripts/member_times.py --set eight --batch 1
