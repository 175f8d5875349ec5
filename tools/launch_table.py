"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) into a per-kernel table:
launches, mean duration and share of all GPU time.  Developer tool:
python tools/launch_table.py launches.csv "<header comment>" > profiles/...txt"""
import csv
import sys
from collections import defaultdict


def main(path, title=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    agg = defaultdict(list)
    for r in rows:
        agg[r[4][:72] + " grid" + r[8].split(",")[0].strip("(")].append(float(r[14]))
    tot = sum(sum(v) for v in agg.values())
    if title:
        print(title)
    print("# kernel | launches | mean us | share of all GPU time in the run (incl. setup)   [raw unit: ns]")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print("%-90s | %4d | %9.2f | %5.1f%%" % (k[:90], len(v), sum(v) / len(v) / 1e3, 100.0 * sum(v) / tot))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
