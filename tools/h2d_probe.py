"""Host-to-device path probe (diagnostic): C2 at N=1 -- device-resident
steps vs ts_table_train_steps_host with torch-pinned and with pageable host
batches, and the raw H2D bandwidth of one batch."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import bench
    import paper_2301_02959_b200 as ts
    args = bench.parse_args([])
    _, ddir, doc = bench.prepare(args, None, 1)
    exp, plan = doc["export"], doc["plan"]
    batches = [np.fromfile(ddir / f"batch_{it}.rows.u32", np.uint32) for it in range(exp["iterations"])]
    t = ts.Table(n_rows=exp["n_rows"], dim=exp["embedding_dim"], dp_cut=plan["dp_cut"], flex_cut=plan["flex_cut"],
                 weight_seed=1234, optimizer=ts.OPT_ROWWISE_ADAGRAD, lr=0.01,
                 max_occurrences=max(b.size for b in batches))
    K = 40
    d_rows = [torch.from_numpy(b.view(np.int32)).cuda() for b in batches]
    out = torch.empty((max(b.size for b in batches), exp["embedding_dim"]), dtype=torch.float32, device="cuda")
    for k in range(3):
        t.train_step(d_rows[k % 4].data_ptr(), d_rows[k % 4].numel(), out.data_ptr())
    t.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        t.train_step(d_rows[k % 4].data_ptr(), d_rows[k % 4].numel(), out.data_ptr())
    t.synchronize()
    print(f"device-resident: {(time.perf_counter() - t0) * 1e3 / K:.4f} ms/step")
    pinned_t = [torch.from_numpy(b.view(np.int32)).pin_memory() for b in batches]
    pinned = [p.numpy().view(np.uint32) for p in pinned_t]
    print("pinned:", [p.is_pinned() for p in pinned_t])
    # the device-resident loop with a 16.8 MB pinned H2D per step on a side
    # stream (no dependency): pure copy-engine interference
    side = torch.cuda.Stream()
    dst_side = torch.empty(min(b.size for b in batches), dtype=torch.int32, device="cuda")
    t.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        with torch.cuda.stream(side):
            dst_side.copy_(pinned_t[k % 4][:dst_side.numel()], non_blocking=True)
        t.train_step(d_rows[k % 4].data_ptr(), d_rows[k % 4].numel(), out.data_ptr())
    t.synchronize()
    torch.cuda.synchronize()
    print(f"device-resident + side H2D: {(time.perf_counter() - t0) * 1e3 / K:.4f} ms/step")
    for name, arrs in (("torch-pinned", pinned), ("pageable", batches)):
        steps = [arrs[k % 4] for k in range(K)]
        t.train_steps_host(steps[:3])
        t0 = time.perf_counter()
        t.train_steps_host(steps)
        print(f"train_steps_host {name}: {(time.perf_counter() - t0) * 1e3 / K:.4f} ms/step")
    dst = torch.empty(batches[0].size, dtype=torch.int32, device="cuda")
    for name, src in (("pinned", pinned_t[0]), ("pageable", torch.from_numpy(batches[0].view(np.int32)))):
        for _ in range(3):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 10
        print(f"H2D {name}: {batches[0].nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.3f} ms per batch)")
    t.close()


if __name__ == "__main__":
    main()
