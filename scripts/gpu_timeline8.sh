#!/bin/bash
# GEMM CTA timeline probes (debug build) for batch-1 EfficientNetV2-L shapes
cd paper_2410_21120_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DDFX_TIMELINE -diag-suppress 20281 -o /tmp/libdfx_tl.so dfx_api.cu dfx_gemm.cu dfx_gemm_persist.cu dfx_bw.cu dfx_fused.cu dfx_vit.cu > /dev/null 2>&1
cd ../..
python -c "import __graft_entry__ as g; g.build()"
for ch in 8; do
echo "== chain $ch"; DFX_LIBRARY=/tmp/libdfx_tl.so timeout 300 python scripts/gemm_timeline.py --chain $ch --cases 384:2304:7:1,2304:384:7:1,256:64:56:1,224:1344:14:1 2>&1 | tail -40
done
