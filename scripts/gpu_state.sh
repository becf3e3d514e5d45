#!/bin/bash
# Re-entry check: build, GPU tests, per-member times, bench (ours + reference arm).
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
echo "== b32"; timeout 300 python scripts/member_times.py --batch 32
echo "== b1"; timeout 300 python scripts/member_times.py --batch 1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
cat gpurun_out/bench.json gpurun_out/bench_ref.json
