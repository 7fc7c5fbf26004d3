#!/usr/bin/env python
"""bench.py — FlexShard per-row tiered sequence embedding, forward + backward.

One step = one training step of the tiered sequence-embedding path on one
batch: route -> (exchange) -> unpooled L x D gather -> loss 0.5*|out|^2 ->
backward (reverse exchange, dedup sort, segment-reduce, DP/Flex all-reduce)
-> fused row-wise Adagrad, all through the C-ABI of libtiershard_b200.so.

Workload (BASELINE.json configs[1], "C2"): 8 tables x 10M rows x D=128 fp32,
seq len 128 per table (L_total = 1024), batch 4096 per GPU, Zipf 1.05,
synthesized with the reference's synthesize_zipf (seeds 1000+t) and sampled
with its Workload (seed 7) by the product's bit-exact host API (ts_driver).
Rows are sharded over N GPUs (topology 1 x N, homogeneous NVSwitch =>
2-tier plan; --virtual-nodes uses 2 x N/2 with the paper's bandwidths and a
3-tier plan).  Per-GPU batch fixed => "scaling": "weak".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank drives its own GPU; timing is CUDA events on the
table's stream, summed over the K timed steps (L2 flushed between steps
outside the events), max over ranks.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sequence samples/sec fwd+bwd (8×B200) + all-to-all GB saved vs row-wise; HBM GB/s"
HOMO = dict(a2a_global_gibs=1, a2a_intra_gibs=1, ar_global_gibs=1, ar_cross_gibs=1)
PAPER_BW = dict(a2a_global_gibs=23, a2a_intra_gibs=95, ar_global_gibs=73, ar_cross_gibs=15)


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--tables", type=int, default=8)
    p.add_argument("--rows", type=int, default=10_000_000)
    p.add_argument("--dim", type=int, default=128)
    p.add_argument("--seq-len", type=int, default=128, help="expected occurrences per table per sample")
    p.add_argument("--batch", type=int, default=4096, help="samples per GPU")
    p.add_argument("--exponent", type=float, default=1.05)
    p.add_argument("--iterations", type=int, default=4, help="distinct batches cycled by the timed loop")
    p.add_argument("--optimizer", choices=("sgd", "adagrad"), default="adagrad")
    p.add_argument("--lr", type=float, default=0.01)
    p.add_argument("--virtual-nodes", action="store_true", help="2 x N/2 virtual nodes, paper bw, 3-tier")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-routing", action="store_true", help="skip the logical-U=8 routing record (N=1)")
    p.add_argument("--sampler", choices=("host", "gpu"), default="host",
                   help="host: the reference Workload's batches (bit-exact), materialized once and "
                        "cycled; gpu: each step's batch drawn on the GPU inside the timed region "
                        "(ts_sampler, same law, for C4/C5-scale throughput runs)")
    p.add_argument("--cache", default="/tmp/tiershard_bench")
    return p.parse_args(argv)


# --------------------------------------------------------------------------
# distributed plumbing (gloo on the host: barrier, max, id broadcast)
# --------------------------------------------------------------------------

class Dist:
    def __init__(self):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as td
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            td.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.td = td

    def barrier(self):
        if self.world > 1:
            self.td.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.td.all_reduce(t, op=self.td.ReduceOp.SUM)
        return float(t.item())

    def gather(self, obj):
        """All ranks' objects, in rank order (every rank gets the list)."""
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.td.all_gather_object(out, obj)
        return out

    def bcast(self, obj):
        if self.world == 1:
            return obj
        box = [obj]
        self.td.broadcast_object_list(box, src=0)
        return box[0]

    def close(self):
        if self.world > 1:
            self.td.destroy_process_group()


# --------------------------------------------------------------------------
# workload preparation (host C++ planner via ts_driver, cached on disk)
# --------------------------------------------------------------------------

def workload_spec(args, n_gpus):
    if args.virtual_nodes and n_gpus >= 4 and n_gpus % 2 == 0:
        topo = dict(num_nodes=2, gpus_per_node=n_gpus // 2, **PAPER_BW)
        goal = "3tier"
    else:
        topo = dict(num_nodes=1, gpus_per_node=n_gpus, **HOMO)
        goal = "2tier"
    tables = [dict(table_id=t, rows=args.rows, exponent=args.exponent, target_length=args.seq_len,
                   seed=1000 + t) for t in range(args.tables)]
    return dict(tables=tables, topology=topo,
                cost_model=dict(local_batch=args.batch, embedding_dim=args.dim), goal=goal,
                frontier=False, hash_seed=2,
                workload=dict(seed=7, iterations=args.iterations if args.sampler == "host" else 1),
                export_alias=args.sampler == "gpu")


def job_config(args, u, w, goal, dp_cut, flex_cut):
    """The workload identity both arms print (identical dicts => the driver's
    same_config).  Arm-specific run details go under "run"."""
    c2 = (args.tables, args.rows, args.seq_len, args.dim, args.batch) == (8, 10_000_000, 128, 128, 4096)
    return {
        "workload": f"{'C2' if c2 else 'custom'}: {args.tables} tables x {args.rows} rows x D={args.dim} fp32, "
                    f"seq len {args.seq_len}/table, batch {args.batch}/GPU, Zipf {args.exponent}",
        "topology": f"{u // w} x {w}" + (" virtual nodes, paper bw" if args.virtual_nodes and u // w > 1
                                         else " homogeneous"),
        "plan": goal, "dp_cut": dp_cut, "flex_cut": flex_cut,
        "global_batch": u * args.batch, "seq_len": args.seq_len * args.tables,
        "parallelism": f"row-sharded over {u} GPU(s): DP/Flex/RW tiers",
        "optimizer": args.optimizer,
        "l2": "GPU arm: 256 MiB written between timed steps (outside the events); tables 41 GB >> L2",
    }


def prepare(args, dist, n_gpus):
    from paper_2301_02959_b200 import DRIVER_PATH
    spec = workload_spec(args, n_gpus)
    key = hashlib.sha1(json.dumps(spec, sort_keys=True).encode()).hexdigest()[:16]
    out_dir = Path(args.cache) / key
    meta_path = out_dir / "meta.json"
    rank0 = dist is None or dist.rank == 0
    if rank0 and not meta_path.exists():
        out_dir.mkdir(parents=True, exist_ok=True)
        spec_run = dict(spec, export_dir=str(out_dir))
        (out_dir / "spec.json").write_text(json.dumps(spec_run))
        t0 = time.time()
        subprocess.run([str(DRIVER_PATH), str(out_dir / "spec.json"), str(out_dir / "doc.json")],
                       check=True)
        doc = json.loads((out_dir / "doc.json").read_text())
        if "error" in doc:
            raise RuntimeError(doc)
        doc["prep_wall_s"] = time.time() - t0
        meta_path.write_text(json.dumps(doc))
    if dist is not None:
        dist.barrier()
    doc = json.loads(meta_path.read_text())
    return spec, out_dir, doc


# --------------------------------------------------------------------------
# clocks sampling during the timed region
# --------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    # One sampler per job (rank 0) over every GPU of the job: per-rank
    # nvidia-smi pollers at 50 ms added driver-query stalls to the timed steps.
    def __init__(self, devices):
        self.devices = ",".join(str(d) for d in devices)
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.devices, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(name)
        under_load = [s for s in sm if s > 0.5 * max(smax or [1])] or sm
        return {"sm_mhz": float(np.median(under_load)) if under_load else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

PHASE_BYTES_DOC = {
    "gather": "occ_local x (2*row_bytes + 4): index read, row read, row write",
    "segment_update": "entries x (row_bytes + 8) + unique x (2*row_bytes + 8): grad + sorted pair read, "
                      "weight read+write, Adagrad state read+write",
    "dedup_sort": "passes x entries x 20: key read (histogram) + pair read + pair write",
}


PHASE_KERNELS = {
    "gather": ["gather_bulk_kernel (U=1)", "gather_local_kernel (U>1)"],
    "segment_update": ["seg_short_kernel", "long_prefix_kernel", "piece_kernel", "long_combine_kernel"],
    "dedup_sort": ["onesweep_hist_kernel", "onesweep_offsets_kernel", "onesweep_pass_kernel"],
}


def ncu_traffic(phase, u):
    """DRAM bytes (read + write) per launch of the phase's kernels, from the
    committed ncu --set full capture summarised in profiles/ncu_traffic.json
    (tools/traffic.py).  None when that capture does not cover the phase."""
    try:
        doc = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
    except Exception:
        return None, None
    entry = doc.get("n1" if u == 1 else f"n{u}", {}).get(phase)
    if not entry:
        return None, None
    return entry["dram_bytes_per_step"], entry.get("source", doc.get("source"))


def ncu_nvlink(u):
    """Per-kernel NVLink payload rates of the exchange kernels running alone
    (profiles/r02_ncu_nvlink_n<U>.json, tools/ncu_nvlink.sh), or None."""
    try:
        doc = json.loads((ROOT / "profiles" / f"r02_ncu_nvlink_n{u}.json").read_text())
    except Exception:
        return None
    keep = ("serve_rows_kernel", "void push_grads_kernel", "replica_update_kernel", "seg_short_kernel (replicated range)")
    return {"source": doc["source"],
            "kernels": {k.replace("void ", ""): {"nvlink_user_tx_gbs": v["nvlink_user_tx_gbs"],
                                                 "nvltx_user_bytes": v["nvltx_user_bytes"], "avg_time_us": v["avg_time_us"]}
                        for k, v in doc["per_kernel"].items() if k in keep}}


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def measure_p2p_ceiling(u):
    """tools/p2p_bw --json on the job's GPUs (every GPU storing 512 B rows
    into random slots of every peer at once): the NVLink ceiling for the
    exchange kernels' access pattern, measured on this box in this run."""
    tool = ROOT / "tools" / "p2p_bw"
    if not tool.exists():
        return None
    try:
        out = subprocess.run([str(tool), str(u), "--json"], capture_output=True, text=True, timeout=300)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 - reported, the fallback peak is labelled
        return {"error": repr(e)}


def nvlink_peak(ceiling):
    if ceiling and ceiling.get("gather_store_gbs"):
        return float(ceiling["gather_store_gbs"]), ("tools/p2p_bw gather_store (all-to-all 512 B row stores, "
                                                     "every GPU at once), measured in this run")
    return 770.0, "fallback: B200_PROFILING.md peer copy per direction (p2p_bw unavailable)"


def run_routing(args, dist):
    """The reference's routing loop (simulator.cpp:223-257) on the GPU for a
    whole LOGICAL iteration of the C2 job at U = 8 -- 1 x 8 (2-tier) and
    2 x 4 virtual nodes (3-tier) -- device-resident: ts_router_iteration_device,
    event-timed.  Bytes model: 4 B index + 1 B placement byte per occurrence
    (the bitmap clears, U x n bits, are timed separately)."""
    import torch
    import paper_2301_02959_b200 as ts
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    res = {}
    for label, vn in (("1x8", False), ("2x4", True)):
        a = argparse.Namespace(**vars(args))
        a.iterations, a.sampler, a.virtual_nodes = 1, "host", vn
        _, ddir, doc = prepare(a, None, 8)
        exp, plan = doc["export"], doc["plan"]
        u, w, B = exp["num_gpus"], exp["gpus_per_node"], exp["local_batch"]
        dest = np.fromfile(ddir / "dest.u8", np.uint8)
        rows = np.fromfile(ddir / "batch_0.rows.u32", np.uint32)
        off = np.fromfile(ddir / "batch_0.offsets.u64", np.uint64)
        bounds = np.ascontiguousarray(off[np.arange(u + 1) * B])
        router = ts.Router(exp["n_rows"], plan["dp_cut"], plan["flex_cut"], dest, u // w, w)
        d_rows = torch.from_numpy(rows.view(np.int32)).cuda()
        d_b = torch.from_numpy(bounds.view(np.int64)).cuda()
        torch.cuda.synchronize()
        kms, tms = [], []
        for k in range(12):
            counters = router.iteration_device(d_b.data_ptr(), d_rows.data_ptr(), rows.size)
            if k >= 2:
                km, tm = router.last_timing()
                kms.append(km)
                tms.append(tm)
        router.close()
        km, tm = float(np.median(kms)), float(np.median(tms))
        algo = rows.size * 5
        res[label] = {
            "topology": f"{u // w} x {w}", "plan": plan["goal"], "dp_cut": plan["dp_cut"],
            "flex_cut": plan["flex_cut"], "occurrences": int(rows.size),
            "kernel_ms": round(km, 4), "iteration_ms": round(tm, 4),
            "occurrences_per_s": round(rows.size / (km / 1e3), 1),
            "algorithmic_bytes": algo, "hbm_gbs": round(algo / (km / 1e3) / 1e9, 1),
            "hbm_frac": round(algo / (km / 1e3) / 1e9 / hbm, 4),
            "bitmap_clear_bytes": int(u * ((exp["n_rows"] + 31) // 32) * 4),
            "counters": counters.tolist(),
            "_inputs": dict(dest=dest, rows=rows, bounds=bounds, u=u, w=w, plan=plan),
        }
        del d_rows, d_b
    return res


def run_ours(args, dist: Dist):
    import torch
    import paper_2301_02959_b200 as ts

    n_gpus = dist.world if dist.world > 1 else args.gpus
    if dist.world == 1 and n_gpus > 1:
        raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    if ts.device_count() == 0:  # the product path has no CPU fallback: fail before preparing anything
        raise SystemExit("tiershard-b200: NoDevice: no CUDA device available (no CPU fallback)")
    spec, data_dir, doc = prepare(args, dist, n_gpus)
    exp = doc["export"]
    u, w = exp["num_gpus"], exp["gpus_per_node"]
    B, D = exp["local_batch"], exp["embedding_dim"]
    g = dist.rank
    device = dist.local_rank
    torch.cuda.set_device(device)
    plan = doc["plan"]
    dest = np.fromfile(data_dir / "dest.u8", np.uint8)
    batches = []
    for it in range(exp["iterations"]):
        rows = np.fromfile(data_dir / f"batch_{it}.rows.u32", np.uint32)
        off = np.fromfile(data_dir / f"batch_{it}.offsets.u64", np.uint64)
        lo, hi = int(off[g * B]), int(off[(g + 1) * B])
        batches.append(np.ascontiguousarray(rows[lo:hi]))
    max_occ = max(b.size for b in batches)
    sampler = None
    if args.sampler == "gpu":
        # capacity: the Poisson(L) batch total stays far below L*B + 8 sqrt(L*B)
        L = float(doc["expected_length"])
        max_occ = max(max_occ, int(L * B + 8 * np.sqrt(L * B)) + 1024)
        sampler = ts.Sampler(np.fromfile(data_dir / "alias.prob.f64", np.float64),
                             np.fromfile(data_dir / "alias.idx.u32", np.uint32), L, seed=7, device=device)

    # NVLink ceiling of this box, measured in this run before any table
    # exists: tools/p2p_bw's all-to-all row-store pattern (the serve /
    # gradient-push access pattern), every GPU of the job at once
    p2p_ceiling = dist.bcast(measure_p2p_ceiling(u) if (u > 1 and g == 0) else None) if u > 1 else None
    nccl_id = None
    if u > 1:
        nccl_id = dist.bcast(ts.nccl_unique_id() if g == 0 else None)
    opt = ts.OPT_ROWWISE_ADAGRAD if args.optimizer == "adagrad" else ts.OPT_SGD
    # gradient receive buffer from the plan: the most loaded server's
    # off-device requests over the prepared iterations, +25 % (+50 % with
    # GPU-sampled batches); a step that needs more grows it collectively
    recv_hint = 0
    if u > 1:
        most = max(t["max_send_off_device_bytes"]["plan"] for t in exp["traffic"]) / (D * 4)
        recv_hint = int(most * (1.5 if sampler is not None else 1.25)) + 4096
    table = ts.Table(n_rows=exp["n_rows"], dim=D, dp_cut=plan["dp_cut"], flex_cut=plan["flex_cut"],
                     tier_dest=dest if u > 1 else None, num_nodes=u // w, gpus_per_node=w, rank=g,
                     device=device, weight_seed=1234, optimizer=opt, lr=args.lr,
                     max_occurrences=max_occ, nccl_unique_id=nccl_id, recv_rows_hint=recv_hint)
    stream = torch.cuda.ExternalStream(table.stream(), device=device)
    d_rows = [torch.from_numpy(b.view(np.int32)).to(f"cuda:{device}") for b in batches]
    d_out = torch.empty((max_occ, D), dtype=torch.float32, device=f"cuda:{device}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")  # 2x L2
    torch.cuda.synchronize()

    if sampler is not None:
        d_sampled = torch.empty(max_occ, dtype=torch.int32, device=f"cuda:{device}")
        sampled_occ = []

    def step(k):
        if sampler is not None:  # this rank's samples [g B, (g+1) B) of iteration k, on the GPU
            occ = sampler.iteration(k, g * B, B, d_sampled.data_ptr(), max_occ, 0, table.stream())
            sampled_occ.append(occ)
            table.train_step(d_sampled.data_ptr(), occ, d_out.data_ptr())
            return
        b = d_rows[k % len(d_rows)]
        table.train_step(b.data_ptr(), b.numel(), d_out.data_ptr())

    # clocks are sampled from the warm-up through the e2e pass (the timed
    # region is inside that window; only samples under load are reported)
    clocks = ClockSampler(range(int(os.environ.get("LOCAL_WORLD_SIZE", u)))) if g == 0 else None
    if clocks:
        clocks.start()
    for k in range(args.warmup):
        step(k)
    table.synchronize()
    dist.barrier()

    # ---- timed region: device-side, CUDA events on the table stream --------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = ts.kernel_launches()
    table.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    wall0 = time.perf_counter()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            if not os.environ.get("TS_BENCH_NOFLUSH"):
                flush.zero_()  # evict L2 (outside the timed events)
            starts[k].record(stream)
        step(args.warmup + k)
        with torch.cuda.stream(stream):
            ends[k].record(stream)
    table.synchronize()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    launches = ts.kernel_launches() - launches0
    per_step = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    step_ms_pct = [round(float(np.percentile(per_step, q)), 4) for q in (0, 50, 100)]
    dev_ms = dist.max(sum(per_step))
    samples = u * B * args.steps
    value = samples / (dev_ms / 1e3)
    loss = table.loss()
    counters = table.counters()

    # ---- lookup + exchange alone (forward only) -----------
    # the same batches, forward passes back to back (the dedup the forward
    # prefetches for the backward is drained between passes, outside events)
    fwd_ms = []
    for k in range(min(args.steps, 20)):
        b = d_rows[k % len(d_rows)] if sampler is None else None
        if b is None:
            occ_k = sampler.iteration(k, g * B, B, d_sampled.data_ptr(), max_occ, 0, table.stream())
            ptr, n_occ = d_sampled.data_ptr(), occ_k
        else:
            ptr, n_occ = b.data_ptr(), b.numel()
        table.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
        table.forward(ptr, n_occ, d_out.data_ptr())
        with torch.cuda.stream(stream):
            e1.record(stream)
        table.synchronize()
        fwd_ms.append(e0.elapsed_time(e1))
    lookup_ms = dist.max(float(np.median(fwd_ms)))

    # ---- per-phase device times (roofline numerator) ------------------------
    table.enable_timing(True)
    prof_steps = min(args.steps, 20)
    for k in range(prof_steps):
        step(k)
    phases = table.phase_times()
    # the same window's timeline: at U = 1 the long-segment path runs on the
    # aux stream beside the short-segment kernel, so the segment update's
    # device time is the union of both phases' intervals, not their sum
    seg_iv = sorted((a, b) for n, _, a, b in table.phase_trace() if n in ("segment_update", "segment_long"))
    seg_union_ms = 0.0
    if seg_iv:
        lo, hi = seg_iv[0]
        for a, b in seg_iv[1:]:
            if a > hi:
                seg_union_ms += hi - lo
                lo, hi = a, b
            else:
                hi = max(hi, b)
        seg_union_ms += hi - lo
    step(prof_steps)  # one more step: its timeline (both streams)
    trace = [(n, sid, round(a, 4), round(b, 4)) for n, sid, a, b in table.phase_trace()]
    all_traces = dist.gather(trace) if os.environ.get("TS_BENCH_DIAG") else None
    rank_phases = dist.gather({k: round(v[0] / prof_steps, 4) for k, v in phases.items() if v[1]}) \
        if os.environ.get("TS_BENCH_DIAG") else None
    table.enable_timing(False)

    # ---- end to end through the host-buffer public entry point -------------
    e2e = None
    if not args.no_e2e:
        pinned = [torch.from_numpy(b.view(np.int32)).pin_memory().numpy().view(np.uint32) for b in batches]
        for k in range(min(args.warmup, 3)):
            table.train_step_host(pinned[k % len(pinned)])
        dist.barrier()
        # one call per step (ts_table_train_step_host) ...
        t0 = time.perf_counter()
        marks = []
        for k in range(args.steps):
            table.train_step_host(pinned[k % len(pinned)])
            marks.append(time.perf_counter())
        e2e_call_s = dist.max(time.perf_counter() - t0)
        step_wall = np.diff(np.array([t0] + marks)) * 1e3
        # ... and the pipelined entry point (ts_table_train_steps_host): the
        # same K steps, each H2D overlapping the previous step's compute
        steps_in = [pinned[k % len(pinned)] for k in range(args.steps)]
        table.train_steps_host(steps_in[:min(3, len(steps_in))])
        dist.barrier()
        ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev_a.record(stream)
        t0 = time.perf_counter()
        table.train_steps_host(steps_in)
        e2e_s = dist.max(time.perf_counter() - t0)
        with torch.cuda.stream(stream):
            ev_b.record(stream)
        torch.cuda.synchronize()
        pipelined_dev_ms = ev_a.elapsed_time(ev_b)  # device span of the call (table stream)
        h2d = float(np.mean([pinned[k % len(pinned)].nbytes for k in range(args.steps)]))
        e2e = {"value": samples / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8,
               "api": "ts_table_train_steps_host (pinned host batches in, per-step loss out)",
               "per_call_value": samples / e2e_call_s,
               "pipelined_device_ms_per_step": round(pipelined_dev_ms / args.steps, 4),
               "pipelined_wall_ms_per_step": round(e2e_s * 1e3 / args.steps, 4),
               "per_call_step_wall_ms": [round(float(np.percentile(step_wall, q)), 3) for q in (0, 50, 100)]}
        if os.environ.get("TS_BENCH_DIAG"):
            # diagnostic: the device-resident steps timed by wall clock, no L2
            # flush (the apples-to-apples partner of the e2e wall time)
            torch.cuda.synchronize()
            dist.barrier()
            t1 = time.perf_counter()
            for k in range(args.steps):
                step(k)
            table.synchronize()
            e2e["diag_device_wall_value"] = samples / dist.max(time.perf_counter() - t1)
            # diagnostic variant: same host copies, torch-owned device buffers
            pin_t = [torch.from_numpy(b.view(np.int32)).pin_memory() for b in batches]
            dist.barrier()
            t1 = time.perf_counter()
            for k in range(args.steps):
                b = d_rows[k % len(d_rows)]
                with torch.cuda.stream(stream):
                    b.copy_(pin_t[k % len(pin_t)], non_blocking=True)
                table.train_step(b.data_ptr(), b.numel(), d_out.data_ptr())
                table.loss()
            e2e["diag_torch_buffers_value"] = samples / dist.max(time.perf_counter() - t1)
            views = [t.numpy().view(np.uint32) for t in pin_t]  # tensors stay referenced by pin_t
            dist.barrier()
            t1 = time.perf_counter()
            for k in range(args.steps):
                table.train_step_host(views[k % len(views)])
            e2e["diag_host_api_pinned_value"] = samples / dist.max(time.perf_counter() - t1)
            import ctypes
            hostmem = []
            for k in range(min(2, len(batches))):
                flags = ctypes.c_uint(0)
                rc = torch.cuda.cudart().cudaHostGetFlags(ctypes.byref(flags), pinned[k].ctypes.data) \
                    if hasattr(torch.cuda.cudart(), "cudaHostGetFlags") else None
                hostmem.append(str(rc))
            e2e["diag_pinned_check"] = hostmem
            torch.cuda.synchronize()
            del views
            torch.cuda.synchronize()
            del pin_t  # pinned blocks carry events on the table's stream: free before it goes
        # one more host-buffer step with the phase timeline (diagnostics)
        table.enable_timing(True)
        table.train_step_host(pinned[0])
        table.phase_times()
        e2e["step_trace_ms"] = [(n, sid, round(a, 4), round(b, 4)) for n, sid, a, b in table.phase_trace()]
        table.enable_timing(False)
    clk = clocks.stop() if clocks else None

    # ---- roofline of the dominant kernel -----------------------------------
    row_bytes = D * 4
    occ_mean = float(np.mean([b.size for b in batches]))
    distinct = float(counters[6, g])
    entries = float(counters[5, g])
    if u == 1:
        n_local_occ = occ_mean
    else:  # DP rows, RW rows this rank owns, Flex rows of its slot
        dp_c, fx_c = plan["dp_cut"], plan["flex_cut"]
        loc = []
        for b in batches:
            d_b = dest[b]
            loc.append(int(((b < dp_c) | ((b < fx_c) & (d_b == g % w)) | ((b >= fx_c) & (d_b == g))).sum()))
        n_local_occ = float(np.mean(loc))
    key_bits = int(np.ceil(np.log2(max(2, exp["n_rows"] if u == 1 else exp["n_rows"] // u))))
    passes = (key_bits + 7) // 8
    algo = {
        "gather": n_local_occ * (2 * row_bytes + 4),
        "segment_update": entries * (row_bytes + 8) + distinct * (2 * row_bytes + (8 if opt else 0)),
        "dedup_sort": passes * entries * 20,
    }
    # phase device time per step (a phase may span several launches per step:
    # the segment update is split into short / long-segment kernels, and at
    # U > 1 runs once for the replicated rows and once for the rest)
    step_ms = {k: v[0] / prof_steps for k, v in phases.items() if v[1]}
    if seg_union_ms > 0:
        step_ms["segment_update"] = seg_union_ms / prof_steps
    per_launch_ms = step_ms
    # the dedup sort's phase spans the gather it runs beside (its own kernels
    # are ~0.2 ms in the ncu launch list), so the dominant kernel is the
    # gather or the segment update, whichever takes longer
    dominant = max((k for k in ("gather", "segment_update") if k in per_launch_ms), key=lambda k: per_launch_ms[k])
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    achieved = algo[dominant] / (per_launch_ms[dominant] / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(dominant, u)
    roofline = {"bound": "hbm", "kernel": dominant, "kernels": PHASE_KERNELS.get(dominant),
                "achieved": round(achieved, 1),
                "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                "traffic": traffic, "traffic_source": traffic_src,
                # DRAM bytes the kernels really moved per step (ncu) over the
                # same in-step time: below `frac` where L2 hits serve reads
                "traffic_frac": (round(traffic / (per_launch_ms[dominant] / 1e3) / 1e9 / hbm_peak, 4)
                                 if traffic else None),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
                "algorithmic_bytes_per_step": algo[dominant], "avg_step_ms": per_launch_ms[dominant],
                "bytes_model": PHASE_BYTES_DOC[dominant],
                "all_phases_ms_per_step": {k: round(v[0] / prof_steps, 4) for k, v in phases.items() if v[1]}}
    for k in ("gather", "segment_update"):
        if k in per_launch_ms:
            roofline[f"{k}_gbs"] = round(algo[k] / (per_launch_ms[k] / 1e3) / 1e9, 1)

    # ---- all-to-all bytes saved (plan vs RW vs TW, per iteration, whole job) --
    tr = exp["traffic"]
    ref_conv = {k: float(np.mean([t["reference_convention"][k] for t in tr]))
                for k in tr[0]["reference_convention"]}
    off_dev = {k: float(np.mean([t["off_device"][k] for t in tr])) for k in tr[0]["off_device"]}
    max_send = {k: float(np.mean([t["max_send_bytes"][k] for t in tr])) / 1e9 for k in tr[0]["max_send_bytes"]}
    max_send_off = {k: float(np.mean([t["max_send_off_device_bytes"][k] for t in tr])) / 1e9
                    for k in tr[0]["max_send_off_device_bytes"]}
    a2a = {
        "unit": "GB per iteration (one direction, one pass, whole job)",
        "saved_vs_rw_reference_convention": (ref_conv["rw_global_bytes"] - ref_conv["plan_global_bytes"]) / 1e9,
        # table-wise moves the same total as row-wise under the reference's
        # self-inclusive convention; where it differs is the most loaded
        # server (one table = one GPU): the all-to-all's critical path
        "max_send_per_gpu_GB": {"plan": max_send["plan"], "rw": max_send["rw"], "tw": max_send["tw"],
                                "convention": "reference (self-inclusive)"},
        "max_send_per_gpu_off_device_GB": max_send_off,
        "global_a2a_reduction": 1 - ref_conv["plan_global_bytes"] / ref_conv["rw_global_bytes"],
        "predicted_reduction": plan["predicted"]["global_a2a_reduction"],
        "saved_vs_rw_off_device": (off_dev["rw_bytes"] - off_dev["plan_global_bytes"] - off_dev["plan_intra_bytes"]) / 1e9,
        "saved_vs_tw_off_device": (off_dev["tw_bytes"] - off_dev["plan_global_bytes"] - off_dev["plan_intra_bytes"]) / 1e9,
        "plan_off_device_GB": (off_dev["plan_global_bytes"] + off_dev["plan_intra_bytes"]) / 1e9,
    }

    # ---- NVLink roofline (U > 1): bytes each GPU must move per step, one
    # direction: its share of the off-device row traffic for the forward rows
    # and the backward gradients (2 passes), plus the replicated tiers'
    # reduce + broadcast, 2 (G-1)/G x replicated rows x row_bytes per group
    # of G (the all-reduce volume); over the measured step
    # time, against the measured peer-copy bandwidth (B200_PROFILING.md).
    nvlink = None
    if u > 1:
        n_nodes = u // w
        flex_slot_rows = (plan["flex_cut"] - plan["dp_cut"]) / w
        per_gpu = {
            "rows_fwd_bwd": 2 * (off_dev["plan_global_bytes"] + off_dev["plan_intra_bytes"]) / u,
            "replicated_dp": 2 * (u - 1) / u * plan["dp_cut"] * row_bytes,
            "replicated_flex": 2 * (n_nodes - 1) / n_nodes * flex_slot_rows * row_bytes if n_nodes > 1 else 0.0,
        }
        total = sum(per_gpu.values())
        step_s = dev_ms / args.steps / 1e3
        peer_peak, peak_src = nvlink_peak(p2p_ceiling)
        nvlink = {"bytes_per_gpu_per_step": total, "breakdown": per_gpu,
                  "achieved_gbs": round(total / step_s / 1e9, 1), "peak_gbs": peer_peak,
                  "peak_source": peak_src, "p2p_ceiling": p2p_ceiling, "ncu_alone": ncu_nvlink(u),
                  "frac": round(total / step_s / 1e9 / peer_peak, 4),
                  "bound_ms": round(total / (peer_peak * 1e9) * 1e3, 4)}

    # lookup + exchange throughput: forward only, whole job; HBM fraction of
    # the gather's algorithmic bytes, NVLink fraction of the forward rows
    occ_job = dist.sum(occ_mean)
    lookup = {"occurrences_per_s": round(occ_job / (lookup_ms / 1e3), 1),
              "samples_per_s": round(u * B / (lookup_ms / 1e3), 1),
              "ms_per_forward": round(lookup_ms, 4),
              "hbm_gbs_per_gpu": round(algo["gather"] / (lookup_ms / 1e3) / 1e9, 1),
              "hbm_frac": round(algo["gather"] / (lookup_ms / 1e3) / 1e9 / hbm_peak, 4)}
    if u > 1:
        fwd_rows = (off_dev["plan_global_bytes"] + off_dev["plan_intra_bytes"]) / u
        lookup["nvlink_gbs_per_gpu"] = round(fwd_rows / (lookup_ms / 1e3) / 1e9, 1)
        lookup["nvlink_frac"] = round(fwd_rows / (lookup_ms / 1e3) / 1e9 / nvlink_peak(p2p_ceiling)[0], 4)

    # ---- routing at logical U = 8 (the reference loop's scale), N = 1 -------
    routing = None
    if u == 1 and not args.no_routing and g == 0:
        routing = run_routing(args, dist)

    # ---- parity of this run's path on one C2 batch (N = 1): a fresh table,
    # one step on batch 0, every touched row read back for the oracle check
    parity_dev = None
    if u == 1 and not args.no_cpu_baseline and g == 0:
        table.close()
        table = ts.Table(n_rows=exp["n_rows"], dim=D, dp_cut=plan["dp_cut"], flex_cut=plan["flex_cut"],
                         num_nodes=1, gpus_per_node=1, rank=0, device=device, weight_seed=1234, optimizer=opt,
                         lr=args.lr, max_occurrences=max_occ)
        b0 = d_rows[0]
        table.train_step(b0.data_ptr(), b0.numel(), d_out.data_ptr())
        table.synchronize()
        probe = np.random.default_rng(5).choice(batches[0].size, size=min(100_000, batches[0].size), replace=False)
        probe.sort()
        out_probe = d_out[torch.from_numpy(probe).to(d_out.device)].cpu().numpy()
        touched = np.unique(batches[0])
        w_dev, st_dev = table.read_rows(touched, with_state=True)
        parity_dev = dict(probe=probe, out_probe=out_probe, touched=touched, w=w_dev, state=st_dev,
                          loss=table.loss())

    cpu = None
    parity = None
    if dist.rank == 0 and u == 1 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline_port(batches[0], dest, plan, exp, B, D, args, parity_dev, routing)
    for r in (routing or {}).values():
        r.pop("_inputs", None)

    result = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "samples/s",
        "n_gpus": u,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dev_ms / args.steps, 4),
        "step_ms_min_median_max_rank0": step_ms_pct,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": ("synthetic: reference synthesize_zipf (seeds 1000+t) + Workload (seed 7), materialized "
                 "bit-exactly by the product host API; weights seeded-hash init") if sampler is None else
                ("synthetic: reference synthesize_zipf (seeds 1000+t); every step's batch drawn on the GPU "
                 "inside the timed region (ts_sampler: the Workload's per-sample law over its alias table); "
                 "weights seeded-hash init"),
        "config": job_config(args, u, w, plan["goal"], plan["dp_cut"], plan["flex_cut"]),
        "run": {"batches_cycled": len(batches) if sampler is None else "gpu-sampled per step",
                "occurrences_per_gpu_step": occ_mean if sampler is None else float(np.mean(sampled_occ))},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
        "roofline": roofline,
        "a2a": a2a,
        "nvlink": nvlink,
        "lookup_exchange": lookup,
        "routing": routing,
        "parity": parity,
        "loss_last_step": loss,
        "step_trace_ms": trace,
        **({"step_trace_ms_all_ranks": all_traces} if all_traces else {}),
        **({"phases_ms_all_ranks": rank_phases} if rank_phases else {}),
        "wall_s_timed": round(wall, 4),
        "prep_wall_s": doc.get("prep_wall_s"),
    }
    if cpu is not None:
        result["cpu_baseline"] = cpu
    table.close()
    return result


def cpu_baseline_port(rows, dest, plan, exp, B, D, args, dev=None, routing=None):
    """Oracle port (oracle/restate.c) of one step on the host cores: the
    reference's routing loop restated (single thread, as the reference runs
    one iteration) + gather + dedup/segment-sum + row-wise Adagrad (threaded).
    Bounded sample: the first batch of the workload, weights compacted to the
    rows it touches (same values: seeded by canonical index).

    The same oracle results are then the checker of this run's device path
    (after every timed region): `dev` = a fresh table's forward + update on
    that batch (probe of the output, every touched row and its Adagrad state)
    must equal them bit for bit; `routing` = the logical-U=8 router counters,
    checked against the restated reference loop over the same 33.6M
    occurrences.  Returns (cpu_baseline, parity)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_bind as orc
    n = exp["n_rows"]
    threads = len(os.sched_getaffinity(0))
    dp, fx = plan["dp_cut"], plan["flex_cut"]
    idx = np.arange(n, dtype=np.uint64)
    tier = np.where(idx < dp, 0, np.where(idx < fx, 1, 2)).astype(np.uint8)
    owner = np.where(tier == 2, dest, 0).astype(np.uint32)
    slot = np.where(tier == 1, dest, 0).astype(np.uint32)
    del idx
    off = np.array([0, rows.size], np.uint64)
    t0 = time.perf_counter()
    orc.route_counts(1, 1, 1, off, rows, tier, owner, slot)
    t_route = time.perf_counter() - t0
    uniq, compact = np.unique(rows, return_inverse=True)
    w = orc.init_rows(1234, uniq.astype(np.uint32), D, threads)
    w0_probe = None
    if dev is not None:
        w0_probe = orc.gather(w, compact.astype(np.uint32)[dev["probe"]], threads)
    state = np.zeros(uniq.size, np.float32)
    compact = compact.astype(np.uint32)
    t0 = time.perf_counter()
    out = orc.gather(w, compact, threads)
    orc.backward_update(w, state, compact, out, orc.OPT_ROWWISE_ADAGRAD, args.lr, 1e-8, threads)
    t_value = time.perf_counter() - t0
    total = t_route + t_value
    cpu = {"value": round(B / total, 2), "unit": "samples/s", "cores": threads, "kind": "port",
           "sample": f"one C2 batch ({B} samples, {rows.size} occurrences): restated reference routing "
                     f"loop {t_route:.3f}s (1 thread) + gather/dedup/Adagrad {t_value:.3f}s "
                     f"({threads} threads); weights compacted to the {uniq.size} touched rows"}
    parity = {}
    if dev is not None and args.optimizer == "adagrad":
        assert np.array_equal(dev["touched"], uniq)
        parity["value_path"] = {
            "what": "fresh table, one train step on C2 batch 0, vs oracle/restate.c (parity unpinned: the "
                    "reference has no value path)",
            "occurrences": int(rows.size), "touched_rows": int(uniq.size),
            "forward_probe_occurrences": int(dev["probe"].size),
            "forward_bit_exact": bool(np.array_equal(dev["out_probe"].view(np.uint32), w0_probe.view(np.uint32))),
            "weights_bit_exact": bool(np.array_equal(dev["w"].view(np.uint32), w.view(np.uint32))),
            "state_bit_exact": bool(np.array_equal(dev["state"].view(np.uint32), state.view(np.uint32))),
            "weights_max_abs_diff": float(np.abs(dev["w"] - w).max()),
        }
    for label, r in (routing or {}).items():
        inp = r.pop("_inputs")
        n_r = inp["dest"].size
        dp_r, fx_r = inp["plan"]["dp_cut"], inp["plan"]["flex_cut"]
        idx = np.arange(n_r, dtype=np.uint64)
        tier_r = np.where(idx < dp_r, 0, np.where(idx < fx_r, 1, 2)).astype(np.uint8)
        del idx
        owner_r = np.where(tier_r == 2, inp["dest"], 0).astype(np.uint32)
        slot_r = np.where(tier_r == 1, inp["dest"], 0).astype(np.uint32)
        t0 = time.perf_counter()
        ref_c = orc.route_counts(inp["u"], inp["w"], 1, inp["bounds"], inp["rows"], tier_r, owner_r, slot_r)
        t_r = time.perf_counter() - t0
        r["cpu_port_occurrences_per_s_1thread"] = round(inp["rows"].size / t_r, 1)
        parity[f"routing_{label}"] = {
            "what": "GPU router counters (7 x U) vs the restated reference loop (oracle/restate.c, pinned to "
                    "the reference's SimReport), one logical C2 iteration",
            "occurrences": int(inp["rows"].size),
            "bit_exact": bool(np.array_equal(np.array(r["counters"], np.uint64), ref_c))}
    return cpu, (parity or None)


# --------------------------------------------------------------------------
# reference arm: the reference's own CPU path (oracle/_ref, unmodified)
# --------------------------------------------------------------------------

def run_reference(args, dist: Dist):
    n_gpus = dist.world if dist.world > 1 else args.gpus
    if dist.rank != 0:
        return None
    ref = ROOT / "oracle" / "_ref" / "ref_driver"
    if not ref.exists():
        return {"impl": "reference", "unavailable": "oracle/_ref/ref_driver was not built (needs /root/reference)"}
    spec = workload_spec(args, n_gpus)
    threads = max(1, min(len(os.sched_getaffinity(0)), args.steps, 32))
    # the reference's simulate() samples every iteration inside its timed
    # pool; the same pool materializing alone (materialize_parallel) is
    # subtracted so `value` is routing + accounting, like for like with the
    # GPU arm, whose batches are materialized before its timed region
    spec["workload"] = dict(seed=7, iterations=args.steps, materialize_pass=False, materialize_parallel=True)
    spec["threads"] = threads
    spec["simulate"] = True
    spec["frontier"] = False
    tmp = Path(args.cache) / "reference"
    tmp.mkdir(parents=True, exist_ok=True)
    (tmp / "spec.json").write_text(json.dumps(spec))
    t0 = time.time()
    subprocess.run([str(ref), str(tmp / "spec.json"), str(tmp / "out.json")], check=True)
    doc = json.loads((tmp / "out.json").read_text())
    wall = time.time() - t0
    sim_s = doc["timing"]["simulate_s"]
    sample_s = doc["timing"]["materialize_parallel_s"]
    route_s = max(sim_s - sample_s, 1e-9)
    u = spec["topology"]["num_nodes"] * spec["topology"]["gpus_per_node"]
    w = spec["topology"]["gpus_per_node"]
    samples = args.steps * u * args.batch
    value = samples / route_s
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "samples/s",
        "n_gpus": n_gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * route_s / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 (integer routing + fp64 accounting)",
        "data": "synthetic (same workload as --impl ours)",
        "config": job_config(args, u, w, doc["plan"]["goal"], doc["plan"]["dp_cut"], doc["plan"]["flex_cut"]),
        "cpu_baseline": {"value": round(value, 2), "unit": "samples/s", "cores": threads, "kind": "reference",
                         "sample": f"tiershard::simulate (unmodified reference, oracle/_ref) over {args.steps} "
                                   f"iterations of the workload, threads={threads}, minus the same pool's "
                                   f"Workload::materialize_iteration time ({sample_s:.2f} of {sim_s:.2f} s): "
                                   "routing + traffic accounting of every occurrence; the reference has no "
                                   "gather/exchange/update to time"},
        "value_including_sampling": round(samples / sim_s, 2),
        "e2e": {"value": round(value, 2), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_timing": doc["timing"],
        "wall_s": round(wall, 1),
        "global_a2a_reduction": doc.get("comparison", {}).get("global_a2a_reduction"),
    }


def main():
    args = parse_args()
    # stdout carries exactly one JSON line: with NCCL_DEBUG set (even WARN)
    # NCCL prints its version banner there, so it stays unset here
    if not os.environ.get("TS_BENCH_KEEP_NCCL_DEBUG"):
        os.environ.pop("NCCL_DEBUG", None)
    dist = Dist()
    try:
        if args.impl == "reference":
            res = run_reference(args, dist)
        else:
            res = run_ours(args, dist)
        if dist.rank == 0 and res is not None:
            print(json.dumps(res), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
