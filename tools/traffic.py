"""Build profiles/ncu_traffic.json from `ncu --set full` reports: DRAM bytes
(read + write) per launch of every kernel, summed per bench phase (one step's
launches of that phase).  bench.py reports it as roofline.traffic.

    python tools/traffic.py OUT.json source-label REPORT.ncu-rep [...]
"""
import collections
import csv
import io
import json
import subprocess
import sys

PHASES = {
    "gather": ["gather_local_kernel"],
    "segment_update": ["seg_short_kernel", "long_prefix_kernel", "piece_kernel", "long_combine_kernel"],
    "dedup_sort": ["onesweep_hist_kernel", "onesweep_offsets_kernel", "onesweep_pass_kernel"],
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def kernel_bytes(report):
    raw = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    out = collections.defaultdict(list)
    for r in data:
        name = r[h.index("Kernel Name")]
        total = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(key)
            total += float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
        for phase, kernels in PHASES.items():
            for k in kernels:
                if k in name:
                    out[k].append(total)
    return out


def main():
    out_path, source, reports = sys.argv[1], sys.argv[2], sys.argv[3:]
    per_kernel = collections.defaultdict(list)
    for rep in reports:
        for k, v in kernel_bytes(rep).items():
            per_kernel[k] += v
    launches_per_step = {"onesweep_pass_kernel": 4}  # 27-bit keys at C2 U=1
    doc = {"source": source, "n1": {}}
    for phase, kernels in PHASES.items():
        got = {k: sum(per_kernel[k]) / len(per_kernel[k]) for k in kernels if per_kernel.get(k)}
        if not got:
            continue
        doc["n1"][phase] = {
            "dram_bytes_per_step": sum(v * launches_per_step.get(k, 1) for k, v in got.items()),
            "per_kernel_launch": got,
            "complete": len(got) == len(kernels),
        }
    with open(out_path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
