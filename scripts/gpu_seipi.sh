#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
echo "== b32"; timeout 300 python scripts/member_times.py --batch 32 | tail -4
echo "== b32 IPI=1"; DFX_SE_IPI=1 timeout 300 python scripts/member_times.py --batch 32 | tail -4
echo "== b32 IPI=4 staged"; DFX_SE_UNSTAGED_BATCH=1000 timeout 300 python scripts/member_times.py --batch 32 | tail -4
echo "== b1"; timeout 300 python scripts/member_times.py --batch 1 | tail -2
