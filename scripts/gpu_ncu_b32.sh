#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NCU=/usr/local/cuda/bin/ncu
# VGG16 conv1_1 at batch 32 as a real 3-channel stem (im2col input), MobileNetV3 24->72 1x1 at 56x56
$NCU --set full --import-source on --clock-control none -k regex:gemm --launch-skip 1 -c 1 -o gpurun_out/r02_b32_vgg_stem python scripts/one_layer.py 3 224 224 64 3 1 1 32 > gpurun_out/ncu1.log 2>&1; tail -2 gpurun_out/ncu1.log
$NCU --set full --import-source on --clock-control none -k regex:gemm --launch-skip 1 -c 1 -o gpurun_out/r02_b32_mbv3_1x1 python scripts/one_layer.py 24 56 56 72 1 1 0 32 > gpurun_out/ncu2.log 2>&1; tail -2 gpurun_out/ncu2.log
python scripts/summarize_profiles.py rep gpurun_out/r02_b32_vgg_stem.ncu-rep gpurun_out/r02_b32_mbv3_1x1.ncu-rep
