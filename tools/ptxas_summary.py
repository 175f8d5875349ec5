"""Registers / spills per kernel from an nvcc -Xptxas -v log (developer tool).
Usage: python tools/ptxas_summary.py paper_1402_5938_b200/build/k_operator.o.log [name-regex]"""
import re
import subprocess
import sys


def main():
    log, pat = sys.argv[1], re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
    cur = None
    rows = []
    for line in open(log):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            spill = (int(m.group(1)), int(m.group(2)))
            rows.append([cur, spill, None])
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and rows and rows[-1][2] is None:
            rows[-1][2] = int(m.group(1))
    names = [r[0] for r in rows]
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    for (n, sp, reg), d in zip(rows, dem):
        if pat.search(d):
            print("%4s regs  spill st/ld %6d/%6d  %s" % (reg, sp[0], sp[1], d[:150]))


if __name__ == "__main__":
    main()
