#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for v in 8 1000; do echo "== xtile batch < $v"; DFX_SE_XTILE_BATCH=$v timeout 300 python scripts/member_times.py --batch 32 | grep -E "efficient|concurrent"; DFX_SE_XTILE_BATCH=$v timeout 300 python scripts/eight_mixed.py; done
