#!/bin/bash
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
bash scripts/ab_step_multi.sh 1 2048 2 old new
bash scripts/ab_step_multi.sh 8 1024 2 old new
