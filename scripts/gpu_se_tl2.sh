#!/bin/bash
cd paper_2410_21120_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DDFX_TIMELINE -diag-suppress 20281 -o /tmp/libdfx_tl.so dfx_api.cu dfx_gemm.cu dfx_gemm_persist.cu dfx_bw.cu dfx_fused.cu dfx_vit.cu 2>&1 | grep error; cd ../..
python -c "import __graft_entry__ as g; g.build()"
DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/se_timeline.py 2>&1 | tail -6
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python scripts/member_times.py --batch 1 | tail -3
timeout 300 python scripts/member_times.py --batch 32 | tail -3
