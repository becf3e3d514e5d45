#!/bin/bash
# GEMM CTA timeline probes for the batch-1 EfficientNet expand conv (development).
cd paper_2410_21120_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DDFX_TIMELINE -diag-suppress 20281 -o /tmp/libdfx_tl.so dfx_api.cu dfx_gemm.cu dfx_bw.cu dfx_fused.cu dfx_vit.cu > /dev/null 2>&1; cd ../..
python -c "import __graft_entry__ as g; g.build()"
for ch in 1 8; do
DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/gemm_timeline.py --chain $ch --cases 384:2304:7:1,2304:384:7:1,576:256:56:1 2>&1 | tail -21
done
python scripts/gemm_timeline.py --chain 8 --cases 384:2304:7:1,2304:384:7:1,576:256:56:1 2>&1 | grep graph
python scripts/member_times.py --batch 1
