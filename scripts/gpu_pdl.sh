#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for v in 0 1; do echo "== early $v"; DFX_GEMM_EARLY_PDL=$v timeout 300 python scripts/member_times.py --batch 1 | grep -E "efficient|densenet|concurrent"; DFX_GEMM_EARLY_PDL=$v timeout 300 python scripts/member_times.py --batch 32 | grep concurrent; done
