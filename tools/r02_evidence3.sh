#!/bin/bash
# third part of the r02 ncu evidence: the 2-D p = 16 apply, 2-D prolongation, h-MG transfers at order p
O=gpurun_out
python tools/kernel_zoo.py 2d hmg > $O/zoo3_plain.log 2>&1 && ncu --set full --clock-control none -k regex:"k_apply2d<16|k_prolong2d|k_prolong_hp|k_restrict_hp|k_restrict2d<8" -c 16 -o /tmp/zoo3 -f python tools/kernel_zoo.py 2d hmg > $O/zoo3.log 2>&1
python tools/ncu_summary.py /tmp/zoo3.ncu-rep --unique > $O/r02_next_kernels2_ncu_full.txt
