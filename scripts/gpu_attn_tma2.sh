#!/bin/bash
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for B in 16 64 128 256; do bash scripts/ab_step.sh_multi 2>/dev/null; bash scripts/ab_step_multi.sh $B 256 2 pre new; done
