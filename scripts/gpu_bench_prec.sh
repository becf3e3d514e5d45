#!/bin/bash
# bench lines per precision (batch 1 headline config + batch 32), no extras
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for p in ${PRECS:-fp16x2 bf16x2}; do
  timeout 900 python bench.py --precision $p --steps 100 --skip-extra --skip-unfused > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$p.json'))
print('$p', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'b32', round(d['sharded_batch32']['ms_per_step'],3), d['parity_rel_err'])
r=d['roofline']; print({k:(v['ms'],v['launches']) for k,v in r['classes'].items()})" || tail -5 gpurun_out/bench_$p.err
done
