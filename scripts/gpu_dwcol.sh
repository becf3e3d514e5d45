#!/bin/bash
# column-strip depthwise kernel: GPU tests, A/B at batch 32 (DFX_DW_COL), bench line
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/tests.txt 2>&1; tail -5 gpurun_out/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for prec in fp16 fp16x2; do
DFX_DW_COL=0 python scripts/quick_time.py --batch 32 --precision $prec --steps 30 --tag "tile dw"
python scripts/quick_time.py --batch 32 --precision $prec --steps 30 --tag "col dw"
done
python scripts/layer_table.py --batch 32 --precision fp16 --top 0 --json gpurun_out/b32_f16_col.json | head -9
DFX_DW_COL=0 python scripts/layer_table.py --batch 32 --precision fp16 --top 0 --json gpurun_out/b32_f16_tile.json | head -9
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
head -c 600 gpurun_out/bench.json
