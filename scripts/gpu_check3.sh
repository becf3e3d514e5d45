#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scripts/member_times.py --batch 1
python scripts/member_times.py --batch 32
