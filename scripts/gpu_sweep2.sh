#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_lifecycle.py tests/test_gpu_manager.py -q -x 2>&1 | tail -1
for p in fp16x2 fp16; do
  Q="python scripts/quick_time.py --precision $p"
  $Q --tag "cmax8"
  DFX_SPLITK_CLUSTER_MAX=16 $Q --tag "cmax16"
  DFX_SPLITK_CLUSTER_MAX=16 DFX_SPLIT_MIN_STAGES_X2=4 DFX_SPLIT_MIN_STAGES=3 $Q --tag "cmax16 minst4/3"
done
