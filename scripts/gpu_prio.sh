#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or corpus or concurrency" 2>&1 | tail -2
for b in 1 32; do
echo "== b$b prio"; timeout 300 python scripts/member_times.py --batch $b | tail -2
echo "== b$b noprio"; DFX_PRIORITY=0 timeout 300 python scripts/member_times.py --batch $b | tail -2
done
echo "== eight prio"; timeout 300 python scripts/member_times.py --batch 1 --set eight | tail -2
echo "== eight noprio"; DFX_PRIORITY=0 timeout 300 python scripts/member_times.py --batch 1 --set eight | tail -2
