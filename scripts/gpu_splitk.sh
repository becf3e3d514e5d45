#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for m in kernel fixup cluster; do echo "== $m"; DFX_SPLITK=$m timeout 300 python scripts/member_times.py --batch 1 | grep -E "efficientnet|densenet|concurrent"; done
