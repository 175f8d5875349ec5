"""Per-section split of an ncu report (source page): executed instructions and warp-stall samples
(total and the top stall reasons) between consecutive block barriers / mbarrier waits of a kernel.
Developer tool: python tools/ncu_sections.py report.ncu-rep"""
import csv
import subprocess
import sys

path = sys.argv[1]
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
isrc, iex, ismp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = [r for r in rows[2:] if len(r) == len(hdr)]
num = lambda x: int(float(x or 0))
tot = sum(num(r[iex]) for r in body)
stot = sum(num(r[ismp]) for r in body)


def flush(sec, cnt, acc, sacc, rs, end):
    top = sorted(rs.items(), key=lambda kv: -kv[1])[:4]
    tops = " ".join("%s %.1f" % (k, 100.0 * v / stot) for k, v in top if v > 0)
    print("sect %2d: %5d instr static, %5.1f%% executed, %5.1f%% stall samples [%s]  (ends %s)"
          % (sec, cnt, 100.0 * acc / tot, 100.0 * sacc / stot, tops, end[:40]))


sec, acc, sacc, cnt, rs = 0, 0, 0, 0, {}
for r in body:
    src = r[isrc].strip()
    acc += num(r[iex]); sacc += num(r[ismp]); cnt += 1
    for i, name in reasons:
        rs[name] = rs.get(name, 0) + num(r[i])
    if "BAR.SYNC" in src or "SYNCS.PHASECHK" in src or "EXIT" in src:
        flush(sec, cnt, acc, sacc, rs, src)
        sec += 1; acc = 0; sacc = 0; cnt = 0; rs = {}
flush(sec, cnt, acc, sacc, rs, "tail")
