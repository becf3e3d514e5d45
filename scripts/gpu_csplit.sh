#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
echo "== b1 cluster"; timeout 300 python scripts/member_times.py --batch 1
echo "== b1 kernel"; DFX_SPLITK=kernel timeout 300 python scripts/member_times.py --batch 1 | tail -2
echo "== b32 cluster"; timeout 300 python scripts/member_times.py --batch 32

