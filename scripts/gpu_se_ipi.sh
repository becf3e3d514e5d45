#!/bin/bash
# A/B: split-precision SE with 4 images per cluster at batch >= 8 (DFX_SE_IPI_SPLIT=4)
python scripts/dump_outputs.py --out /tmp/o1.npz
DFX_SE_IPI_SPLIT=4 python scripts/dump_outputs.py --out /tmp/o4.npz
python -c "
import numpy as np
a=np.load('/tmp/o1.npz'); b=np.load('/tmp/o4.npz')
for k in a.files:
    x,y=a[k],b[k]; print(k, x.shape, 'bitwise' if np.array_equal(x,y) else float(np.abs(x-y).max()/np.abs(x).max()))
"
for rep in 1 2; do
python scripts/quick_time.py --batch 32 --steps 20 --tag "ipi1"
DFX_SE_IPI_SPLIT=4 python scripts/quick_time.py --batch 32 --steps 20 --tag "ipi4"
done
DFX_SE_IPI_SPLIT=4 python scripts/quick_time.py --tag "ipi4 b1"
