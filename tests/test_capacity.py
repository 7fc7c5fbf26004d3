"""Capacity (SURVEY.md §7 "Capacity", BASELINE configs C4 / C5): the host-side
footprint calculator (ts_table_plan_footprint, the same sum ts_table_create
checks against free HBM before allocating) shows each rank of the
production-scale configs fits in one B200's HBM once the gradient receive
buffer is sized from the plan (recv_rows_hint) instead of the worst case."""
import paper_2301_02959_b200 as ts

HBM = 180e9  # B200 HBM3e per GPU (usable is a little below the 192 GB part)
D = 128


def rank_bytes(n_rows, u, n_nodes, occ, dp_rows, flex_rows, rw_share, hint_margin=1.25, host_api=False):
    """One rank of a U-GPU job: shard = all DP rows + its Flex slot + its RW
    share; receive hint = the expected remote RW/Flex occurrences with a
    margin (rw_share = the fraction of occurrences outside DP)."""
    w = u // n_nodes
    rw_rows = (n_rows - dp_rows - flex_rows + u - 1) // u
    hint = int(rw_share * occ * (u - 1) / u * hint_margin)
    f = ts.plan_footprint(n_rows=n_rows, dim=D, dp_rows=dp_rows, flex_rows=(flex_rows + w - 1) // w,
                          rw_rows=rw_rows, num_nodes=n_nodes, gpus_per_node=w, max_occurrences=occ,
                          recv_rows_hint=hint, host_api=host_api)
    worst = ts.plan_footprint(n_rows=n_rows, dim=D, dp_rows=dp_rows, flex_rows=(flex_rows + w - 1) // w,
                              rw_rows=rw_rows, num_nodes=n_nodes, gpus_per_node=w, max_occurrences=occ)
    user_out = occ * D * 4  # the caller's [occ x D] output / gradient buffer
    return f, worst, user_out


def test_c5_fits_per_gpu_at_u8():
    # C5: 16 tables x 100M rows, D=128, L = 512/table (8192 per sample),
    # batch 8192/GPU -> 67.1M occurrences per GPU (+ Poisson headroom).
    # Plan: C4's 2-tier covers 77 % with 2.2M DP rows; C5 is
    # taken with twice the DP rows and a 25 % RW share (conservative).
    n, occ = 1_600_000_000, 8192 * 8192 + 65_536
    f, worst, user_out = rank_bytes(n, 8, 1, occ, dp_rows=4_400_000, flex_rows=0, rw_share=0.25)
    assert f["weights"] > 100e9  # 200M rows of 512 B on every rank
    assert f["total"] + user_out < HBM, (f, user_out)
    # the round-1 sizing (receive buffer for every peer's whole batch) does not
    assert worst["total"] + user_out > HBM
    assert worst["exchange"] > 200e9


def test_c4_fits_per_gpu_at_u4_virtual_nodes():
    # C4: 16 x 50M rows, L = 256/table, batch 4096/GPU (16.8M occurrences),
    # 2 x 2 virtual nodes, 3-tier (BASELINE.md 2x4 plan: 147K DP + 2.8M Flex)
    n, occ = 800_000_000, 4096 * 4096 + 32_768
    f, worst, user_out = rank_bytes(n, 4, 2, occ, dp_rows=146_672, flex_rows=2_786_768, rw_share=0.25,
                                    host_api=True)
    assert f["total"] + user_out < HBM, (f, user_out)


def test_footprint_counts_each_part():
    f = ts.plan_footprint(n_rows=1000, dim=64, dp_rows=10, flex_rows=0, rw_rows=990, max_occurrences=5000)
    assert f["remap"] == 0 and f["exchange"] == 0 and f["host_api"] == 0
    assert f["total"] == sum(v for k, v in f.items() if k != "total")
    g = ts.plan_footprint(n_rows=1000, dim=64, dp_rows=10, flex_rows=0, rw_rows=495, gpus_per_node=2,
                          max_occurrences=5000, host_api=True)
    assert g["remap"] > 0 and g["exchange"] > 0 and g["host_api"] > 0
