#!/bin/bash
# Developer probe: time and DRAM bytes per launch of the step kernels on one config (ncu metrics pass).
# usage: tools/ncu_bytes.sh <config> <tag>   (env passes through)
cfg=${1:-4}; tag=${2:-x}
python tools/fused_probe.py $cfg 3 1 > /dev/null && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_apply_v4|k_cheb_update|k_init" --csv --log-file gpurun_out/bytes_$tag.csv python tools/fused_probe.py $cfg 3 1 > /dev/null 2>&1
python - <<P
import csv
rows=[r for r in csv.reader(open("gpurun_out/bytes_$tag.csv")) if len(r)>14 and r[0].isdigit()]
cur={}
for r in rows:
    key=(r[0],r[4][:40])
    cur.setdefault(key,{})[r[12]]=float(r[14])
for (i,k),d in cur.items():
    print("%-42s %8.3f ms  read %7.3f GB  write %6.3f GB  L2 hit %5.1f%%" % (k, d.get("gpu__time_duration.sum",0)/1e6, d.get("dram__bytes_read.sum",0)/1e9, d.get("dram__bytes_write.sum",0)/1e9, d.get("lts__t_sector_hit_rate.pct",0)))
P
