#!/bin/bash
# split-precision persistent GEMM (bn <= 64): 2 CTAs x 2 slots per SM vs 1 CTA with a deeper ring
python scripts/dump_outputs.py --out /tmp/o1.npz
DFX_PERSIST_ONE_CTA_X2=1 python scripts/dump_outputs.py --out /tmp/o0.npz
python -c "
import numpy as np
a=np.load('/tmp/o1.npz'); b=np.load('/tmp/o0.npz')
print([('bitwise' if np.array_equal(a[k],b[k]) else float(np.abs(a[k]-b[k]).max())) for k in a.files])"
for rep in 1 2; do
python scripts/quick_time.py --batch 32 --steps 20 --tag "2 CTAs/SM"
DFX_PERSIST_ONE_CTA_X2=1 python scripts/quick_time.py --batch 32 --steps 20 --tag "1 CTA/SM deep ring"
done
