#!/bin/bash
# A/B: staged vs direct epilogue drain, persistent on/off, over representative batch-32 layers
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
C="64:256:56:32:3,256:64:56:32:1,32:32:112:32:3,512:512:28:32:3,224:1344:14:32:1,96:384:28:32:1,192:48:56:32:3,640:3840:7:32:1,4096:4096:1:1:1"
for act in silu ""; do
for drain in staged direct; do
for pers in 1 0; do
  echo "== act=$act drain=$drain persist=$pers"; DFX_GEMM_DRAIN=$drain DFX_GEMM_PERSIST=$pers timeout 300 python scripts/gemm_micro.py --cases $C --act "$act" | awk '{print $1,$2,$3,$4,$(NF-3),$(NF-1)}'
done; done; done
