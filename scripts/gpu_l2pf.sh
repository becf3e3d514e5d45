#!/bin/bash
# A/B: L2 prefetch of the member's next weight blobs from every batch-1 GEMM (DFX_L2_PREFETCH)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -q -x 2>&1 | tail -1
for rep in 1 2; do
for pf in 0 1; do
DFX_L2_PREFETCH=$pf python scripts/quick_time.py --tag "l2pf=$pf"
done
done
for pf in 0 1; do
DFX_L2_PREFETCH=$pf python scripts/quick_time.py --tag "l2pf=$pf eff" --models efficientnet_v2_l
DFX_L2_PREFETCH=$pf python scripts/quick_time.py --tag "l2pf=$pf fp16" --precision fp16
DFX_L2_PREFETCH=$pf python scripts/quick_time.py --tag "l2pf=$pf b32" --batch 32 --steps 20
done
