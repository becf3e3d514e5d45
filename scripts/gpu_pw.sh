#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for w in 2 1 1.3; do echo "== waves $w"; DFX_PERSIST_MIN_WAVES=$w timeout 300 python scripts/member_times.py --batch 32 | grep -E "efficient|densenet|vgg|concurrent"; DFX_PERSIST_MIN_WAVES=$w timeout 300 python scripts/eight_mixed.py; done
