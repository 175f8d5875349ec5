"""Summarise an ncu report (raw page) into the handful of numbers used in DESIGN.md / profiles/."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "local_load", "lts__t_sectors_op_red.sum"]
STALLS = "smsp__average_warps_issue_stalled_"


def main(path, unique=False):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    seen = set()
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if unique:   # one launch per (kernel, grid, block): the first
            key = (d.get("Kernel Name", ""), d.get("launch__grid_size", ""), d.get("launch__block_size", ""))
            if key in seen:
                continue
            seen.add(key)
        u = dict(zip(hdr, units))
        print("==", d.get("Kernel Name", "")[:100])
        for k in KEYS:
            for h in hdr:
                if h == k or (k == "local_load" and "local" in h and h.endswith(".sum") and "inst" in h):
                    print("  %-70s %s %s" % (h, d[h], u[h]))
        st = sorted(((float(d[h] or 0), h) for h in hdr if h.startswith(STALLS) and h.endswith("_per_issue_active.ratio")),
                    reverse=True)[:6]
        for v, h in st:
            print("  stall %-62s %.3f" % (h[len(STALLS):], v))


if __name__ == "__main__":
    main(sys.argv[1], len(sys.argv) > 2 and sys.argv[2] == "--unique")
