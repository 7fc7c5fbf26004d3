"""Summarise an ncu launch list with NVLink counters (tools/ncu_nvlink.sh)
into per-kernel averages: time, DRAM bytes, NVLink tx/rx bytes (total and
user payload), and the rates they imply.  ncu serialises launches, so rates
are per kernel running alone (cold caches); the in-step NVLink fraction is
bench.py's.

    python tools/nvlink_summary.py gpurun_out/ncu_nvlink_n2.csv OUT.json "label"
"""
import collections
import csv
import io
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def main():
    src, out, label = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = [l for l in open(src).read().splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h, data = rows[0], rows[1:]
    col = {k: h.index(k) for k in ("ID", "Kernel Name", "Device", "Metric Name", "Metric Unit", "Metric Value")}
    launches = collections.defaultdict(dict)
    names = {}
    for r in data:
        key = (r[col["ID"]], r[col["Device"]])
        name = r[col["Kernel Name"]].split("(")[0].split("::")[-1].split("<")[0]
        names[key] = name
        v = float(r[col["Metric Value"]].replace(",", "")) * SCALE.get(r[col["Metric Unit"]], 1)
        launches[key][r[col["Metric Name"]]] = v
    per = collections.defaultdict(list)
    for key, m in launches.items():
        name = names[key]
        if name == "seg_short_kernel":  # the replicated-row range pushes partials over NVLink
            name += " (replicated range)" if m.get("nvltx__bytes_data_user.sum", 0) > 0 else " (rest)"
        per[name].append(m)
    res = {}
    for name, ms in sorted(per.items()):
        avg = {k: sum(x.get(k, 0.0) for x in ms) / len(ms) for k in ms[0]}
        t = avg.get("gpu__time_duration.sum", 0.0)
        dram = avg.get("dram__bytes_read.sum", 0.0) + avg.get("dram__bytes_write.sum", 0.0)
        tx_user = avg.get("nvltx__bytes_data_user.sum", 0.0)
        res[name] = {
            "launches": len(ms), "avg_time_us": round(t * 1e6, 2),
            "dram_bytes": round(dram), "nvltx_bytes": round(avg.get("nvltx__bytes.sum", 0.0)),
            "nvltx_user_bytes": round(tx_user), "nvlrx_user_bytes": round(avg.get("nvlrx__bytes_data_user.sum", 0.0)),
            "dram_gbs": round(dram / t / 1e9, 1) if t else None,
            "nvlink_user_tx_gbs": round(tx_user / t / 1e9, 1) if t else None,
        }
    # per step and rank, from the launches each makes per step: one gather,
    # one short-segment launch per segment range (replicated, rest), and the
    # long path (prefix, pieces, combine) once per range
    per_step = {"seg_short_kernel (replicated range)": 1, "seg_short_kernel (rest)": 1, "piece_kernel": 2,
                "long_combine_kernel": 2, "long_prefix_kernel": 2}
    seg = tuple(per_step)
    seg_bytes = sum(res[k]["dram_bytes"] * per_step[k] for k in seg if k in res)
    n_steps = None
    phases = {"gather": {"dram_bytes_per_step": res["gather_local_kernel"]["dram_bytes"]} if "gather_local_kernel" in res
              else None,
              "segment_update": {"dram_bytes_per_step": seg_bytes, "launches_per_step": per_step}
              if any(k in res for k in seg) else None}
    json.dump({"source": label, "per_kernel": res, "phases": phases}, open(out, "w"), indent=1)
    for k, v in res.items():
        print(k, v)


if __name__ == "__main__":
    main()
