#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for f in 64 128; do echo "== bn floor $f"; DFX_BN_FLOOR_MANY_M=$f timeout 300 python scripts/member_times.py --batch 32 | grep -E "efficient|densenet|concurrent"; DFX_BN_FLOOR_MANY_M=$f timeout 300 python scripts/member_times.py --batch 1 | grep concurrent; DFX_BN_FLOOR_MANY_M=$f timeout 300 python scripts/eight_mixed.py; done
