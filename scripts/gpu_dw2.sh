#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 300 python scripts/dw_micro.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dwconv -c 1 -o gpurun_out/dw_s5_b32 python scripts/dw_micro.py --cases 1344:14:32:3:1 > /dev/null 2>&1
ls gpurun_out | grep dw
