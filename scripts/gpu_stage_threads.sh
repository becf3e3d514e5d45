#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
for n in 2 4 8 15; do
  DFX_STAGE_THREADS=$n timeout 600 python bench.py --skip-unfused --skip-extra --steps 300 --warmup 5 > gpurun_out/st_$n.$r.json 2>/dev/null
done
done
