#!/bin/bash
# split SE x tile at every batch (DFX_SE_XTILE_BATCH_X2): bitwise check + A/B
python scripts/dump_outputs.py --out /tmp/o1.npz
DFX_SE_XTILE_BATCH_X2=8 python scripts/dump_outputs.py --out /tmp/o0.npz
python -c "
import numpy as np
a=np.load('/tmp/o1.npz'); b=np.load('/tmp/o0.npz')
print([('bitwise' if np.array_equal(a[k],b[k]) else float(np.abs(a[k]-b[k]).max())) for k in a.files])"
for rep in 1 2; do
python scripts/quick_time.py --batch 32 --steps 20 --tag "xtile all batches"
DFX_SE_XTILE_BATCH_X2=8 python scripts/quick_time.py --batch 32 --steps 20 --tag "xtile < 8"
done
python scripts/quick_time.py --batch 32 --steps 20 --precision bf16x2 --tag "bf16x2 xtile all"
DFX_SE_XTILE_BATCH_X2=8 python scripts/quick_time.py --batch 32 --steps 20 --precision bf16x2 --tag "bf16x2 xtile < 8"
