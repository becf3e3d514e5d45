timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for pdl in 0 1; do echo "DFX_PDL=$pdl"; DFX_PDL=$pdl python scripts/gpu_zoo_timing.py 2>&1 | grep "B="; done
python scripts/layer_table.py --batch 1 --top 12 2>&1 | tail -22
