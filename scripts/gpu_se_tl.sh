cd paper_2410_21120_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DDFX_TIMELINE -diag-suppress 20281 -o /tmp/libdfx_tl.so dfx_api.cu dfx_gemm.cu dfx_bw.cu dfx_fused.cu 2>&1 | grep error; cd ../..
DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/se_timeline.py 2>&1 | tail -5
