"""Top SASS instructions by warp-stall samples from an ncu report (source page), with a running
window so a stalled instruction can be read in context.  Developer tool."""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ia, isrc, ismp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(int(r[ismp] or 0) for r in body)
    print("total samples", tot)
    order = sorted(range(len(body)), key=lambda i: -int(body[i][ismp] or 0))
    for i in order[:top]:
        r = body[i]
        print("%6d %5.1f%%  %5d  %s" % (int(r[ismp]), 100.0 * int(r[ismp]) / tot, i, r[isrc].strip()[:90]))
    # coarse profile: samples per 100-instruction window
    print("-- per window of 64 instructions")
    for w in range(0, len(body), 64):
        s = sum(int(r[ismp] or 0) for r in body[w:w + 64])
        if s > 0.01 * tot:
            print("%5d-%5d %5.1f%%  first: %s" % (w, w + 63, 100.0 * s / tot, body[w][isrc].strip()[:60]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
