#!/bin/bash
cd paper_2410_21120_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DDFX_TIMELINE -diag-suppress 20281 -o /tmp/libdfx_tl.so dfx_api.cu dfx_gemm.cu dfx_bw.cu dfx_fused.cu dfx_vit.cu > /dev/null 2>&1
cd ../..
python -c "import __graft_entry__ as g; g.build()"
echo "== param desc"; DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/gemm_timeline.py --chain 1 --cases 384:2304:7:1 2>&1 | tail -8
echo "== global desc"; DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/gemm_timeline.py --chain 1 --global-desc --cases 384:2304:7:1 2>&1 | tail -8
