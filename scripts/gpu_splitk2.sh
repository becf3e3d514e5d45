#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for m in kernel auto; do
echo "== $m"; DFX_SPLITK=$m timeout 300 python scripts/member_times.py --batch 1 | grep -E "concurrent"
DFX_SPLITK=$m timeout 300 python scripts/member_times.py --batch 32 | grep -E "concurrent"
DFX_SPLITK=$m timeout 300 python scripts/member_times.py --batch 1 --set eight | grep -E "vit|resnet|inception|concurrent"
DFX_SPLITK=$m timeout 300 python scripts/eight_mixed.py
done
