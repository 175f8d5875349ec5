#!/bin/bash
# Developer A/B timing on the GPU box: tools/ab.sh "<quick_bench args>" lib1.so lib2.so ...
# Each library is copied over the in-tree libsfmg.so in turn (twice, interleaved) and timed.
args="$1"; shift
LIB=paper_1402_5938_b200/libsfmg.so
cp $LIB /tmp/ab_orig.so
for rep in 1 2; do
  for l in "$@"; do
    cp "$l" $LIB
    echo "== $l (rep $rep)"
    python tools/quick_bench.py $args 2>&1 | grep cfg | python -c "
import sys, json
for line in sys.stdin:
    d = json.loads(line)
    print('%-12s apply %8.2f us (%.3f)  step %8.2f us (%.3f)' % (d['cfg'], d['t_apply_us'], d['frac_hbm_apply'], d['t_step_us'], d['frac_hbm_step']))"
  done
done
cp /tmp/ab_orig.so $LIB
