"""Summarise ncu reports (raw page) into one line per kernel: time, DRAM
bytes, DRAM %, L2 hit rate, occupancy, registers, top stall reasons."""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__t_sector_hit_rate.pct", "L2hit%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1%"),
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0]
        parts = [name[:60]]
        for key, short in WANT:
            if key in h:
                i = h.index(key)
                parts.append(f"{short}={r[i]}{units[i] if units[i] not in ('', 'none', '%') else ''}")
        stalls = [(h[i], r[i]) for i in range(len(h))
                  if h[i].startswith("smsp__average_warp_latency_issue_stalled_") and h[i].endswith(".ratio")]
        if not stalls:
            stalls = [(h[i], r[i]) for i in range(len(h))
                      if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
        try:
            top = sorted(((float(v.replace(",", "")), k) for k, v in stalls if v), reverse=True)[:4]
            parts.append("stalls=" + ",".join(f"{k.split('stalled_')[-1].split('.')[0]}:{v:.0f}" for v, k in top))
        except ValueError:
            pass
        out.append(" | ".join(parts))
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for line in summarise(p):
            print(line)
