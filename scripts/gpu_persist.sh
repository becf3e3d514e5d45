#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "conv_layer" 2>&1 | tail -3
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
echo "== persist on"; python scripts/member_times.py --batch 32
echo "== persist off"; DFX_GEMM_PERSIST=0 python scripts/member_times.py --batch 32
echo "== b1"; python scripts/member_times.py --batch 1
