#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for b in 1 32; do
echo "== b$b dwse"; timeout 300 python scripts/member_times.py --batch $b
echo "== b$b nodwse"; DFX_FUSE_DWSE=0 timeout 300 python scripts/member_times.py --batch $b | tail -4
done
