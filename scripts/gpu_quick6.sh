#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
C="64:256:56:32:3,224:1344:14:32:1,384:2304:7:32:1,2304:384:7:32:1,192:48:56:32:3"
echo "== silu"; timeout 300 python scripts/gemm_micro.py --cases $C --act silu | awk '{print $1,$2,$3,$4,$(NF-3),$(NF-1)}'
echo "== b32"; timeout 300 python scripts/member_times.py --batch 32
echo "== b1"; timeout 300 python scripts/member_times.py --batch 1
