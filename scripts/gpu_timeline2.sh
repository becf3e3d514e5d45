cd paper_2410_21120_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DDFX_TIMELINE -diag-suppress 20281 -o /tmp/libdfx_tl.so dfx_api.cu dfx_gemm.cu dfx_bw.cu dfx_fused.cu > /dev/null 2>&1; cd ../..
echo PARAM; DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/gemm_timeline.py --cases 384:2304:7:1,192:768:14:1 2>&1 | tail -12
echo GLOBAL; DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/gemm_timeline.py --cases 384:2304:7:1,192:768:14:1 --global-desc 2>&1 | tail -12
