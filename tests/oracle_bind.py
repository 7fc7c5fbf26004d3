"""ctypes binding of oracle/_build/liboracle.so — the CHECKER (test-only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module (oracle/restate.h explains the contract).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_LIB = ROOT / "oracle" / "_build" / "liboracle.so"
REF_DRIVER = ROOT / "oracle" / "_ref" / "ref_driver"

OPT_SGD = 0
OPT_ROWWISE_ADAGRAD = 1
PIECE = 256

_lib = None
vp = C.c_void_p


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_LIB.exists():
            raise FileNotFoundError(f"{ORACLE_LIB} missing: run `make -C oracle restate`")
        L = C.CDLL(str(ORACLE_LIB))
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_row_key_hash.restype = C.c_uint64
        L.orc_row_key_hash.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_assign_rows.restype = None
        L.orc_assign_rows.argtypes = [C.c_uint64, vp, vp, C.c_uint64, C.c_uint64, C.c_uint32,
                                      C.c_uint32, C.c_uint64, vp, vp, vp]
        L.orc_route_counts.restype = C.c_int
        L.orc_route_counts.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, vp, vp, C.c_uint64,
                                       vp, vp, vp, vp]
        L.orc_iteration_metrics.restype = C.c_int
        L.orc_iteration_metrics.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.c_int, C.c_double, C.c_double,
                                            C.c_double, C.c_double, C.c_double, C.c_double,
                                            C.c_double, C.c_double, vp, vp]
        L.orc_init_weight.restype = C.c_float
        L.orc_init_weight.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_init_table.restype = None
        L.orc_init_table.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, vp, C.c_int]
        L.orc_init_rows.restype = None
        L.orc_init_rows.argtypes = [C.c_uint64, vp, C.c_uint64, C.c_uint32, vp, C.c_int]
        L.orc_gather.restype = None
        L.orc_gather.argtypes = [vp, C.c_uint32, vp, C.c_uint64, vp, C.c_int]
        L.orc_half_sq_sum.restype = C.c_double
        L.orc_half_sq_sum.argtypes = [vp, C.c_uint64]
        L.orc_backward_update.restype = C.c_uint64
        L.orc_backward_update.argtypes = [vp, vp, C.c_uint64, C.c_uint32, vp, C.c_uint64, vp,
                                          C.c_int, C.c_float, C.c_float, C.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


METRIC_FIELDS = (
    "global_a2a_send_max", "global_a2a_recv_max", "global_a2a_bytes_mean", "global_a2a_total",
    "intra_a2a_send_max", "intra_a2a_recv_max", "intra_a2a_bytes_mean", "intra_a2a_total",
    "ar_global_bytes", "ar_cross_bytes_max", "ar_cross_bytes_mean", "global_a2a_seconds",
    "intra_a2a_seconds", "ar_global_seconds", "ar_cross_seconds", "total_seconds",
    "total_seconds_critical", "peak_dynamic_memory_bytes", "rows_accessed_scalars_min",
    "rows_accessed_scalars_max", "rows_accessed_scalars_mean", "load_imbalance",
    "distinct_rows_min", "distinct_rows_max", "distinct_rows_mean", "distinct_row_imbalance",
)


def assign_rows(table_id, row_id, dp_cut, flex_cut, u, w, hash_seed=2):
    n = len(table_id)
    t = np.ascontiguousarray(table_id, dtype=np.uint32)
    r = np.ascontiguousarray(row_id, dtype=np.uint64)
    tier = np.zeros(n, np.uint8)
    owner = np.zeros(n, np.uint32)
    slot = np.zeros(n, np.uint32)
    lib().orc_assign_rows(n, _p(t), _p(r), dp_cut, flex_cut, u, w, hash_seed, _p(tier), _p(owner), _p(slot))
    return tier, owner, slot


def route_counts(u, w, local_batch, offsets, rows, tier, owner, slot):
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    rw = np.ascontiguousarray(rows, dtype=np.uint32)
    tr = np.ascontiguousarray(tier, dtype=np.uint8)
    ow = np.ascontiguousarray(owner, dtype=np.uint32)
    sl = np.ascontiguousarray(slot, dtype=np.uint32)
    out = np.zeros(7 * u, np.uint64)
    rc = lib().orc_route_counts(u, w, local_batch, _p(off), _p(rw), len(tr), _p(tr), _p(ow), _p(sl), _p(out))
    if rc != 0:
        raise ValueError(f"orc_route_counts failed: {rc}")
    return out.reshape(7, u)


def iteration_metrics(counters, *, dim, scalar_bytes=4, dyn=2, stat=1, include_id=False,
                      bytes_per_id=8.0, bw=(1.0, 1.0, 1.0, 1.0), ar_global_bytes=0.0,
                      ar_cross_max=0.0, ar_cross_mean=0.0):
    c = np.ascontiguousarray(counters, dtype=np.uint64).reshape(-1)
    u = c.size // 7
    m = np.zeros(26, np.float64)
    rc = lib().orc_iteration_metrics(u, dim, scalar_bytes, dyn, stat, int(include_id), bytes_per_id,
                                      *bw, ar_global_bytes, ar_cross_max, ar_cross_mean, _p(c), _p(m))
    if rc != 0:
        raise ValueError("conservation violated")
    return dict(zip(METRIC_FIELDS, m.tolist()))


def init_table(seed, n, dim, threads=8):
    w = np.zeros((n, dim), np.float32)
    lib().orc_init_table(seed, n, dim, _p(w), threads)
    return w


def init_rows(seed, canon, dim, threads=8):
    canon = np.ascontiguousarray(canon, dtype=np.uint32)
    w = np.zeros((canon.size, dim), np.float32)
    lib().orc_init_rows(seed, _p(canon), canon.size, dim, _p(w), threads)
    return w


def gather(w, rows, threads=8):
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    out = np.zeros((rows.size, w.shape[1]), np.float32)
    lib().orc_gather(_p(w), w.shape[1], _p(rows), rows.size, _p(out), threads)
    return out


def half_sq_sum(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    return lib().orc_half_sq_sum(_p(x), x.size)


def backward_update(w, state, rows, grads, optimizer, lr, eps=1e-8, threads=8):
    """In-place update of w (and state) following the contract in restate.h."""
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    grads = np.ascontiguousarray(grads, dtype=np.float32)
    assert w.flags.c_contiguous and w.dtype == np.float32
    st = state if state is not None else np.zeros(1, np.float32)
    return lib().orc_backward_update(_p(w), _p(st), w.shape[0], w.shape[1], _p(rows), rows.size,
                                     _p(grads), optimizer, lr, eps, threads)
