#!/bin/bash
# A/B: members with slack on a bounded SM budget (DFX_SLACK_SMS, persistent GEMMs) or
# with capped split-K (DFX_SLACK_SPLIT_MAX); DFX_SLACK_FRAC picks the members
export DFX_SLACK_DEBUG=1
for rep in 1 2; do
python scripts/quick_time.py --tag base
for sms in 32 64; do
for fr in 0.5 0.95; do
DFX_SLACK_SMS=$sms DFX_SLACK_FRAC=$fr python scripts/quick_time.py --tag "sms$sms frac$fr"
done
done
done
DFX_SLACK_SMS=48 DFX_SLACK_FRAC=0.5 python scripts/quick_time.py --tag "sms48 frac0.5 eff+vgg" --models efficientnet_v2_l vgg16
DFX_SLACK_SMS=48 DFX_SLACK_FRAC=0.5 python scripts/quick_time.py --tag "sms48 frac0.5 fp16" --precision fp16
python scripts/quick_time.py --tag "base fp16" --precision fp16
