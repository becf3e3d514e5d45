#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
C="64:256:56:32:3,256:64:56:32:1,32:32:112:32:3,512:512:28:32:3,224:1344:14:32:1,96:384:28:32:1,192:48:56:32:3,640:3840:7:32:1,4096:4096:1:1:1"
echo "== silu"; timeout 300 python scripts/gemm_micro.py --cases $C --act silu | awk '{print $1,$2,$3,$4,$(NF-3),$(NF-1)}'
echo "== b32"; timeout 300 python scripts/member_times.py --batch 32
echo "== b1"; timeout 300 python scripts/member_times.py --batch 1
