"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by
kernel name: total, share, count, average."""
import collections
import csv
import sys


def main(path, skip_setup=True):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("tsd::<unnamed>::", "")[:60]
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    setup = {k for k in agg if "init_weights" in k}
    tot = sum(v[1] for k, v in agg.items() if k not in setup)
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = "  setup" if k in setup else f"{100 * v[1] / tot:6.1f}%"
        print(f"{v[1] / 1e3:9.3f} ms {share} n={v[0]:4d} avg={v[1] / v[0]:9.1f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
