#!/bin/bash
# which member slows EfficientNetV2-L's chain in the 4-model DAG (batch 1), and cluster sizes
python scripts/quick_time.py --tag "eff alone" --models efficientnet_v2_l
python scripts/quick_time.py --tag "eff+vgg" --models efficientnet_v2_l vgg16
python scripts/quick_time.py --tag "eff+mbv3" --models efficientnet_v2_l mobilenet_v3_large
DFX_SE_CL=8 python scripts/quick_time.py --tag "eff alone se8" --models efficientnet_v2_l
DFX_SE_CL=8 python scripts/quick_time.py --tag "eff+vgg se8" --models efficientnet_v2_l vgg16
DFX_SE_CL=8 python scripts/quick_time.py --tag "4 se8"
DFX_SPLITK_CLUSTER_MAX=8 python scripts/quick_time.py --tag "4 skcl8"
python scripts/quick_time.py --tag "4 base"
