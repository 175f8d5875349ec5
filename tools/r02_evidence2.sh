#!/bin/bash
# second part of the r02 ncu evidence (Gauss / 2-D / h-MG kernels), bounded launch count
O=gpurun_out
python tools/kernel_zoo.py gauss 2d hmg > $O/zoo_plain.log 2>&1 && ncu --set full --clock-control none -k regex:"k_apply_gauss|k_apply2d|k_prolong2d|k_restrict2d|k_prolong_hp|k_restrict_hp" -c 40 -o /tmp/zoo -f python tools/kernel_zoo.py gauss 2d hmg > $O/zoo.log 2>&1
python tools/ncu_summary.py /tmp/zoo.ncu-rep --unique > $O/r02_next_kernels_ncu_full.txt
