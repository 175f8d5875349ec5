"""Per-section split of an ncu report (source page): executed instructions and warp-stall samples
between consecutive block barriers / mbarrier waits of a kernel.  Developer tool:
python tools/ncu_sections.py report.ncu-rep"""
import csv
import subprocess
import sys

path = sys.argv[1]
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
isrc, iex, ismp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[iex] or 0) for r in body); stot = sum(int(r[ismp] or 0) for r in body)
sec, acc, sacc, start = 0, 0, 0, body[0][isrc]
cnt = 0
for r in body:
    src = r[isrc].strip()
    acc += int(r[iex] or 0); sacc += int(r[ismp] or 0); cnt += 1
    if "BAR.SYNC" in src or "SYNCS.PHASECHK" in src or "EXIT" in src:
        print("sect %2d: %5d instr static, %5.1f%% executed, %5.1f%% stall samples  (ends %s)" % (sec, cnt, 100.0*acc/tot, 100.0*sacc/stot, src[:40]))
        sec += 1; acc = 0; sacc = 0; cnt = 0
print("tail: %d static %.1f%% exec %.1f%% samples" % (cnt, 100.0*acc/tot, 100.0*sacc/stot))
