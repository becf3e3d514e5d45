#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scripts/effnet_classes.py fp16 base
python scripts/effnet_classes.py fp16x2 base
DFX_GEMM_DW=0 python scripts/effnet_classes.py fp16x2 no-dw-fusion
DFX_SPLITK=kernel python scripts/effnet_classes.py fp16x2 splitk-kernel
