# Developer A/B over L2 flush modes: bash tools/flush_ab.sh "<quick_bench args>" "<modes>" lib1.so lib2.so ...
args="$1"; modes="$2"; shift 2
cp paper_1402_5938_b200/libsfmg.so /tmp/fab_orig.so
for lib in "$@"; do
  cp $lib paper_1402_5938_b200/libsfmg.so
  for mode in $modes; do
    echo "== $lib $mode"; QB_FLUSH=$mode python tools/quick_bench.py $args | python -c "
import sys, json
for line in sys.stdin:
    if 'cfg' not in line: continue
    d = json.loads(line)
    print('%-12s apply %8.2f us (%.3f)  step %8.2f us (%.3f)' % (d['cfg'], d['t_apply_us'], d['frac_hbm_apply'], d['t_step_us'], d['frac_hbm_step']))"
  done
done
cp /tmp/fab_orig.so paper_1402_5938_b200/libsfmg.so
