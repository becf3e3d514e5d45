#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for m in efficientnet_v2_l densenet161 vgg16 mobilenet_v3_large; do
  timeout 300 python scripts/layer_table.py --batch 32 --models $m --top 0 --json gpurun_out/layers_${m}_b32.json | head -9
done
