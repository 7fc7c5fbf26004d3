"""Summarise an ncu launch list taken with
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`:
per kernel launches, average time, share of GPU time, DRAM bytes per launch
and DRAM GB/s (cold-cache, serialised launches: shares, not absolutes).

    python tools/launch_traffic.py launches.csv [OUT.txt]
"""
import collections
import csv
import re
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
         "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def short(name: str) -> str:
    name = name.split("(")[0]
    name = re.sub(r"^void ", "", name)
    return name.replace("tsd::<unnamed>::", "")


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ii, ki, mi, ui, vi = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    per, names = collections.defaultdict(dict), {}
    for r in data:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        names[r[ii]] = short(r[ki])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':58s} {'n':>5s} {'avg_us':>9s} {'share%':>7s} {'dram_MB':>9s} {'dram_GB/s':>9s}"]
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n[:58]:58s} {a[0]:5d} {a[1] / a[0] * 1e6:9.1f} {a[1] / total * 100:7.2f} "
                     f"{a[2] / a[0] / 1e6:9.1f} {a[2] / a[1] / 1e9 if a[1] else 0:9.0f}")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text, end="")


if __name__ == "__main__":
    main(*sys.argv[1:])
