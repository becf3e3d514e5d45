#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
echo "== b32"; timeout 300 python scripts/member_times.py --batch 32
echo "== b32 SE staged"; DFX_SE_UNSTAGED_BATCH=1000 timeout 300 python scripts/member_times.py --batch 32
echo "== b1"; timeout 300 python scripts/member_times.py --batch 1
echo "== b1 SE_CL=8"; DFX_SE_CL=8 timeout 300 python scripts/member_times.py --batch 1
timeout 300 python scripts/layer_table.py --batch 32 --models efficientnet_v2_l --top 0 --json gpurun_out/layers_efficientnet_v2_l_b32.json 
timeout 300 python scripts/layer_table.py --batch 1 --models efficientnet_v2_l --top 0 --json gpurun_out/layers_effnet_b1.json 
