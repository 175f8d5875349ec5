#!/bin/bash
# r02 full-set captures of the collocated element kernel at p = 8 (config 2 = config 3 p 8), 4 and 16.
O=gpurun_out
for p in 8 4 16; do
  python tools/quick_bench.py 3:$p > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_apply_v4 -s 6 -c 1 -o /tmp/ap$p -f python tools/quick_bench.py 3:$p > $O/ap$p.log 2>&1
  python tools/ncu_summary.py /tmp/ap$p.ncu-rep > $O/r02_k_apply_v4_p${p}_summary.txt
  python tools/ncu_sections.py /tmp/ap$p.ncu-rep > $O/r02_k_apply_v4_p${p}_sections.txt
done
