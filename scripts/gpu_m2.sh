#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "conv_layer" 2>&1 | tail -3
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
echo "== m2 on"; python scripts/member_times.py --batch 32
echo "== m2 off"; DFX_GEMM_M2=0 python scripts/member_times.py --batch 32
echo "== m2 on, b1"; python scripts/member_times.py --batch 1
