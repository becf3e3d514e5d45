#!/bin/bash
# Per-layer GEMM tables (isolated node timings) at batch 32 and batch 1.
python -c "import __graft_entry__ as g; g.build()"
for m in efficientnet_v2_l densenet161 mobilenet_v3_large; do
  echo "=== $m b32"; timeout 300 python scripts/layer_table.py --batch 32 --models $m --top 45 --json gpurun_out/layers_${m}_b32.json
done
echo "=== effnet b1"; timeout 300 python scripts/layer_table.py --batch 1 --models efficientnet_v2_l --top 30 --json gpurun_out/layers_effnet_b1.json
