#!/bin/bash
# quick_bench with a one-line-per-config summary: bash tools/qb.sh "2 3 4"
python tools/quick_bench.py $1 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    if not line.startswith('{'): continue
    d = json.loads(line)
    print('%-12s apply %8.2f us (%.3f)  step %8.2f us (%.3f)' % (d['cfg'], d['t_apply_us'], d['frac_hbm_apply'], d['t_step_us'], d['frac_hbm_step']))"
