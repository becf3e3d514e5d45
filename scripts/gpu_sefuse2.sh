#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for b in 1 32; do
echo "== b$b default"; timeout 300 python scripts/member_times.py --batch $b | tail -3
echo "== b$b SE_FUSE=0"; DFX_SE_FUSE=0 timeout 300 python scripts/member_times.py --batch $b | tail -3
done
echo "== eight b1"; timeout 300 python scripts/member_times.py --batch 1 --set eight | tail -2
