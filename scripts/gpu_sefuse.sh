#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for b in 1 32; do
echo "== b$b default"; timeout 300 python scripts/member_times.py --batch $b | tail -3
echo "== b$b SE_FUSE"; DFX_SE_FUSE=1 timeout 300 python scripts/member_times.py --batch $b | tail -3
done
