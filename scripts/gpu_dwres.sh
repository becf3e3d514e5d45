#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for r in 0 3 4 6; do echo "== resident $r"; DFX_DW_RESIDENT=$r timeout 300 python scripts/dw_micro.py; DFX_DW_RESIDENT=$r timeout 300 python scripts/member_times.py --batch 32 | grep -E "efficient|concurrent"; done
