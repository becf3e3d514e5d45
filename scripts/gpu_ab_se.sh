#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_zoo.py -x -q -k four 2>&1 | tail -2
echo "== SE fused"; python scripts/member_times.py --batch 1
echo "== SE unfused"; DFX_SE_FUSE=0 python scripts/member_times.py --batch 1
