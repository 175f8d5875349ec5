#!/bin/bash
# ncu evidence for the kernels outside k_apply_v4 (round-1 verdict, missing item 2).  Run on the GPU box:
#   bash tools/r02_evidence.sh   -> gpurun_out/r02_*  (summaries are copied to profiles/ by hand)
set -x
O=gpurun_out
# (1) launch list of config-5 V-cycles: per-kernel time and DRAM bytes
python tools/vcycle_bench.py 3 nosolve && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/r02_vcycle_launches.csv python tools/vcycle_bench.py 3 nosolve > $O/vc1.log 2>&1
# (2) full-set captures of the V-cycle kernels (transfer, coarse CG, update, init, the p = 16 / 4 / 2 / 1 applies)
ncu --set full --clock-control none --import-source on -k regex:"k_prolong|k_restrict|k_coarse_cg|k_cheb_update|k_init|k_apply|k_residual|k_axpy" -c 400 -o /tmp/vc -f python tools/vcycle_bench.py 1 nosolve > $O/vc2.log 2>&1
python tools/ncu_summary.py /tmp/vc.ncu-rep --unique > $O/r02_vcycle_kernels_ncu_full.txt
# (3) Gauss apply, 2-D kernels, h-MG transfers
python tools/kernel_zoo.py gauss 2d hmg && ncu --set full --clock-control none --import-source on -k regex:"gauss|2d|_hp|k_cgc|k_dot" -c 400 -o /tmp/zoo -f python tools/kernel_zoo.py gauss 2d hmg > $O/zoo.log 2>&1
python tools/ncu_summary.py /tmp/zoo.ncu-rep --unique > $O/r02_next_kernels_ncu_full.txt
ls -la /tmp/*.ncu-rep
