#!/bin/bash
# A/B sweep of every switch against the current defaults (fused 4-model, batch 1 and 32)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
run() { echo "== $1 b1 $(env $1 timeout 300 python scripts/member_times.py --batch 1 | grep concurrent)"; echo "== $1 b32 $(env $1 timeout 300 python scripts/member_times.py --batch 32 | grep concurrent)"; }
run DFX_NONE=1
run DFX_GEMM_DRAIN=staged
run DFX_SPLITK=cluster
run DFX_GEMM_M2=0
run DFX_GEMM_PERSIST=0
run DFX_SE_UNSTAGED_BATCH=4
run DFX_PDL=0
