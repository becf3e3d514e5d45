#!/bin/bash
# A/B: batch-1 weight tiles with an L2 evict_first policy (DFX_W_EVICT_FIRST)
for rep in 1 2; do
python scripts/quick_time.py --tag base
DFX_W_EVICT_FIRST=1 python scripts/quick_time.py --tag "evict_first"
DFX_W_EVICT_FIRST=1 DFX_SLACK_SMS=32 DFX_SLACK_FRAC=0.5 python scripts/quick_time.py --tag "evict_first sms32"
done
python scripts/quick_time.py --tag "eff+vgg base" --models efficientnet_v2_l vgg16
DFX_W_EVICT_FIRST=1 python scripts/quick_time.py --tag "eff+vgg evict_first" --models efficientnet_v2_l vgg16
DFX_W_EVICT_FIRST=1 python scripts/quick_time.py --tag "eff evict_first" --models efficientnet_v2_l
python scripts/quick_time.py --tag "base fp16" --precision fp16
DFX_W_EVICT_FIRST=1 python scripts/quick_time.py --tag "evict_first fp16" --precision fp16
