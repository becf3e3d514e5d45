#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for m in 4 3 2; do echo "== min stages $m"; DFX_SPLIT_MIN_STAGES=$m timeout 300 python scripts/member_times.py --batch 1; done
