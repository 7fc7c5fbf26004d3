"""ctypes binding of include/tiershard_b200.h (the drop-in C-ABI).

Mirrors the C entry points one to one; every non-zero ts_status raises
TSError carrying the status code and ts_last_error()'s message, mapped the
same way the C++ shim maps them (TS_ERR_CONFIG -> ConfigError, ...).
Device pointers are passed as plain integers (e.g. torch.Tensor.data_ptr()).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "lib" / "libtiershard_b200.so"
DRIVER_PATH = PKG_DIR / "bin" / "ts_driver"

TS_OK = 0
STATUS_NAMES = {
    1: "ConfigError",
    2: "ValidationError",
    3: "Error",
    4: "CudaError",
    5: "NcclError",
    6: "NoDevice",
}
COUNTER_NAMES = (
    "send_global",
    "recv_global",
    "send_intra",
    "recv_intra",
    "dp_local",
    "served",
    "distinct",
)
OPT_SGD = 0
OPT_ROWWISE_ADAGRAD = 1

# symbols declared by include/tiershard_b200.h (tests check the export list)
EXPORTS = (
    "ts_last_error",
    "ts_build_info",
    "ts_abi_version",
    "ts_device_count",
    "ts_nccl_unique_id",
    "ts_kernel_launches",
    "ts_router_create",
    "ts_router_iteration",
    "ts_router_iteration_device",
    "ts_router_destroy",
    "ts_router_last_timing",
    "ts_shard_layout",
    "ts_exchange_plan",
    "ts_table_create",
    "ts_table_destroy",
    "ts_table_shard_rows",
    "ts_table_stream",
    "ts_table_forward",
    "ts_table_backward",
    "ts_table_train_step",
    "ts_table_train_step_host",
    "ts_table_loss",
    "ts_table_counters",
    "ts_table_read_rows",
    "ts_table_synchronize",
    "ts_table_enable_timing",
    "ts_table_phase_times",
    "ts_table_phase_name",
    "ts_table_phase_trace",
    "ts_keymap_create",
    "ts_keymap_lookup",
    "ts_keymap_destroy",
    "ts_table_forward_keys",
    "ts_sampler_create",
    "ts_sampler_iteration",
    "ts_sampler_destroy",
    "ts_table_train_steps_host",
    "ts_frontier_preview",
    "ts_group_create",
    "ts_group_destroy",
    "ts_group_abort",
    "ts_table_plan_footprint",
    "ts_table_recv_capacity",
)


class TSError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status{status}")
        super().__init__(f"{self.kind}: {message}")
        self.message = message


class TableConfig(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_uint32),
        ("gpus_per_node", C.c_uint32),
        ("rank", C.c_uint32),
        ("device", C.c_int32),
        ("dim", C.c_uint32),
        ("n_rows", C.c_uint64),
        ("dp_cut", C.c_uint64),
        ("flex_cut", C.c_uint64),
        ("weight_seed", C.c_uint64),
        ("optimizer", C.c_int32),
        ("lr", C.c_float),
        ("eps", C.c_float),
        ("max_occurrences", C.c_uint64),
        ("nccl_unique_id", C.c_void_p),
        ("group", C.c_void_p),
        ("recv_rows_hint", C.c_uint64),
    ]


class Footprint(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("weights", "optimizer_state", "remap", "step_buffers", "exchange",
                                          "replicated", "host_api", "total")]


_lib = None

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


def load() -> C.CDLL:
    """Loads the in-tree libtiershard_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise FileNotFoundError(
            f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(str(LIB_PATH))
    sig = {
        "ts_last_error": (C.c_char_p, []),
        "ts_build_info": (C.c_char_p, []),
        "ts_abi_version": (C.c_int, []),
        "ts_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "ts_nccl_unique_id": (C.c_int, [vp]),
        "ts_kernel_launches": (C.c_uint64, []),
        "ts_router_create": (C.c_int, [C.POINTER(vp), C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                       vp, C.c_uint32, C.c_uint32]),
        "ts_router_iteration": (C.c_int, [vp, C.c_uint32, vp, vp, C.c_uint64, vp]),
        "ts_router_iteration_device": (C.c_int, [vp, vp, vp, C.c_uint64, vp]),
        "ts_router_destroy": (C.c_int, [vp]),
        "ts_router_last_timing": (C.c_int, [vp, f64p, f64p]),
        "ts_shard_layout": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, vp, C.c_uint32, C.c_uint32,
                                      C.c_uint32, vp, u64p, u64p, u64p]),
        "ts_exchange_plan": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, vp, vp, vp, vp, vp, u64p,
                                       u64p]),
        "ts_table_create": (C.c_int, [C.POINTER(vp), C.POINTER(TableConfig), vp]),
        "ts_table_destroy": (C.c_int, [vp]),
        "ts_table_shard_rows": (C.c_int, [vp, u64p, u64p, u64p]),
        "ts_table_stream": (C.c_int, [vp, C.POINTER(vp)]),
        "ts_table_forward": (C.c_int, [vp, vp, C.c_uint64, vp]),
        "ts_table_backward": (C.c_int, [vp, vp]),
        "ts_table_train_step": (C.c_int, [vp, vp, C.c_uint64, vp]),
        "ts_table_train_step_host": (C.c_int, [vp, vp, C.c_uint64, f64p]),
        "ts_table_loss": (C.c_int, [vp, f64p]),
        "ts_table_counters": (C.c_int, [vp, vp]),
        "ts_table_read_rows": (C.c_int, [vp, vp, C.c_uint64, vp, vp]),
        "ts_table_synchronize": (C.c_int, [vp]),
        "ts_table_enable_timing": (C.c_int, [vp, C.c_int]),
        "ts_table_phase_times": (C.c_int, [vp, f64p, u64p, C.c_int, C.POINTER(C.c_int)]),
        "ts_table_phase_name": (C.c_char_p, [C.c_int]),
        "ts_table_phase_trace": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.POINTER(C.c_int)]),
        "ts_keymap_create": (C.c_int, [C.POINTER(vp), C.c_int, C.c_uint64, vp, vp]),
        "ts_keymap_lookup": (C.c_int, [vp, vp, vp, C.c_uint64, vp, vp, u64p]),
        "ts_keymap_destroy": (C.c_int, [vp]),
        "ts_table_forward_keys": (C.c_int, [vp, vp, vp, vp, C.c_uint64, vp]),
        "ts_sampler_create": (C.c_int, [C.POINTER(vp), C.c_int, C.c_uint64, vp, vp, C.c_double, C.c_uint64]),
        "ts_sampler_iteration": (C.c_int, [vp, C.c_uint32, C.c_uint64, C.c_uint32, vp, C.c_uint64, vp, u64p, vp]),
        "ts_sampler_destroy": (C.c_int, [vp]),
        "ts_table_train_steps_host": (C.c_int, [vp, vp, vp, C.c_uint32, vp]),
        "ts_frontier_preview": (C.c_int, [C.c_int, C.c_uint64, vp, C.c_uint32, vp, vp]),
        "ts_group_create": (C.c_int, [C.POINTER(vp), C.c_uint32]),
        "ts_group_destroy": (C.c_int, [vp]),
        "ts_group_abort": (C.c_int, [vp]),
        "ts_table_recv_capacity": (C.c_int, [vp, u64p, u64p]),
        "ts_table_plan_footprint": (C.c_int, [C.POINTER(TableConfig), C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                              C.POINTER(Footprint)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status != TS_OK:
        msg = load().ts_last_error().decode()
        raise TSError(status, msg)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def build_info() -> str:
    return load().ts_build_info().decode()


def device_count() -> int:
    n = C.c_int(0)
    _check(load().ts_device_count(C.byref(n)))
    return n.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load().ts_nccl_unique_id(buf))
    return buf.raw


def kernel_launches() -> int:
    return int(load().ts_kernel_launches())


def shard_layout(n_rows, dp_cut, flex_cut, tier_dest, num_nodes, gpus_per_node, rank,
                 with_ids=True):
    """Host-only: (local_id[n] or None, (dp_rows, flex_rows, rw_rows)) of `rank`."""
    dest = np.ascontiguousarray(tier_dest, dtype=np.uint8)
    ids = np.zeros(n_rows, np.uint32) if with_ids else None
    a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _check(load().ts_shard_layout(n_rows, dp_cut, flex_cut, _ptr(dest) if dest.size else None,
                                  num_nodes, gpus_per_node, rank,
                                  _ptr(ids) if ids is not None and ids.size else None,
                                  C.byref(a), C.byref(b), C.byref(c)))
    return ids, (a.value, b.value, c.value)


def exchange_plan(num_nodes, gpus_per_node, rank, all_starts):
    """Host-only all-to-allv plan of `rank` from [U][U+W+2] bucket starts."""
    u = num_nodes * gpus_per_node
    st = np.ascontiguousarray(all_starts, dtype=np.uint32)
    assert st.shape == (u, u + gpus_per_node + 2)
    so, sc, ro, rc = (np.zeros(2 * u, np.uint64) for _ in range(4))
    before, total = C.c_uint64(), C.c_uint64()
    _check(load().ts_exchange_plan(num_nodes, gpus_per_node, rank, _ptr(st), _ptr(so), _ptr(sc),
                                   _ptr(ro), _ptr(rc), C.byref(before), C.byref(total)))
    return dict(send_off=so, send_cnt=sc, recv_off=ro, recv_cnt=rc, recv_before=before.value,
                recv_total=total.value)


def plan_footprint(*, n_rows, dim, dp_rows, flex_rows, rw_rows, num_nodes=1, gpus_per_node=1,
                   optimizer=OPT_ROWWISE_ADAGRAD, max_occurrences, recv_rows_hint=0, host_api=False) -> dict:
    """Host-only ts_table_plan_footprint: device bytes one rank allocates."""
    cfg = TableConfig(num_nodes, gpus_per_node, 0, 0, dim, n_rows, 0, 0, 0, optimizer, 0.0, 0.0,
                      max_occurrences, None, None, recv_rows_hint)
    out = Footprint()
    _check(load().ts_table_plan_footprint(C.byref(cfg), dp_rows, flex_rows, rw_rows, 1 if host_api else 0,
                                          C.byref(out)))
    return {k: getattr(out, k) for k, _ in Footprint._fields_}


class Router:
    """ts_router_*: GPU routing + traffic accounting of one logical U-GPU iteration."""

    def __init__(self, n_rows: int, dp_cut: int, flex_cut: int, tier_dest: np.ndarray,
                 num_nodes: int, gpus_per_node: int, device: int = 0):
        self._lib = load()
        self.u = num_nodes * gpus_per_node
        dest = np.ascontiguousarray(tier_dest, dtype=np.uint8)
        h = vp()
        _check(self._lib.ts_router_create(C.byref(h), device, n_rows, dp_cut, flex_cut,
                                          _ptr(dest), num_nodes, gpus_per_node))
        self._h = h

    def iteration(self, local_batch: int, sample_offsets: np.ndarray, rows: np.ndarray) -> np.ndarray:
        off = np.ascontiguousarray(sample_offsets, dtype=np.uint64)
        r = np.ascontiguousarray(rows, dtype=np.uint32)
        out = np.zeros(7 * self.u, dtype=np.uint64)
        _check(self._lib.ts_router_iteration(self._h, local_batch, _ptr(off),
                                             _ptr(r) if r.size else None, r.size, _ptr(out)))
        return out.reshape(7, self.u)

    def iteration_device(self, d_requester_begin: int, d_rows: int, occurrences: int) -> np.ndarray:
        """Device-resident iteration: U+1 u64 requester bounds and the rows
        (device pointers); counters to host."""
        out = np.zeros(7 * self.u, dtype=np.uint64)
        _check(self._lib.ts_router_iteration_device(self._h, d_requester_begin, d_rows or None, occurrences,
                                                    _ptr(out)))
        return out.reshape(7, self.u)

    def last_timing(self) -> tuple[float, float]:
        """(kernel ms, whole-iteration ms incl. clears) of the last iteration."""
        k, t = C.c_double(), C.c_double()
        _check(self._lib.ts_router_last_timing(self._h, C.byref(k), C.byref(t)))
        return k.value, t.value

    def close(self):
        if getattr(self, "_h", None):
            _check(self._lib.ts_router_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class KeyMap:
    """ts_keymap_*: raw (table_id, row_id) -> canonical row index on the device."""

    ABSENT = 0xFFFFFFFF

    def __init__(self, table_ids: np.ndarray, row_ids: np.ndarray, device: int = 0):
        self._lib = load()
        t = np.ascontiguousarray(table_ids, dtype=np.uint32)
        r = np.ascontiguousarray(row_ids, dtype=np.uint64)
        assert t.shape == r.shape
        h = vp()
        _check(self._lib.ts_keymap_create(C.byref(h), device, t.size, _ptr(t) if t.size else None,
                                          _ptr(r) if r.size else None))
        self._h = h

    def lookup_device(self, d_table_ids: int, d_row_ids: int, n: int, d_canon: int,
                      stream: int = 0, count_misses: bool = True):
        """Device pointers in and out; returns the miss count (synchronises) or None."""
        m = C.c_uint64(0)
        _check(self._lib.ts_keymap_lookup(self._h, d_table_ids or None, d_row_ids or None, n,
                                          d_canon or None, stream or None,
                                          C.byref(m) if count_misses else None))
        return m.value if count_misses else None

    def close(self):
        if getattr(self, "_h", None):
            _check(self._lib.ts_keymap_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Sampler:
    """ts_sampler_*: GPU workload sampler over an alias table (throughput runs)."""

    def __init__(self, alias_prob: np.ndarray, alias_index: np.ndarray, expected_length: float,
                 seed: int, device: int = 0):
        self._lib = load()
        p = np.ascontiguousarray(alias_prob, dtype=np.float64)
        a = np.ascontiguousarray(alias_index, dtype=np.uint32)
        h = vp()
        _check(self._lib.ts_sampler_create(C.byref(h), device, p.size, _ptr(p) if p.size else None,
                                           _ptr(a) if a.size else None, expected_length, seed))
        self._h = h

    def iteration(self, iteration: int, sample_begin: int, samples: int, d_rows: int, capacity: int,
                  d_offsets: int = 0, stream: int = 0) -> int:
        occ = C.c_uint64(0)
        _check(self._lib.ts_sampler_iteration(self._h, iteration, sample_begin, samples, d_rows or None,
                                              capacity, d_offsets or None, C.byref(occ), stream or None))
        return occ.value

    def close(self):
        if getattr(self, "_h", None):
            _check(self._lib.ts_sampler_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Group:
    """ts_group_*: the in-process rank group.  Every rank of a U-rank job is a
    host thread of this process (any GPUs, several ranks per GPU allowed);
    pass the group to each rank's Table instead of an NCCL id, and create,
    step and close each Table from its own thread (ctypes releases the GIL
    during the calls, so the ranks' collectives meet)."""

    def __init__(self, ranks: int):
        self._lib = load()
        h = vp()
        _check(self._lib.ts_group_create(C.byref(h), ranks))
        self._h = h
        self.ranks = ranks

    @property
    def handle(self) -> int:
        return self._h.value

    def abort(self) -> None:
        """A rank's thread failed: every pending collective fails at once."""
        _check(self._lib.ts_group_abort(self._h))

    def close(self):
        if getattr(self, "_h", None):
            _check(self._lib.ts_group_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Table:
    """ts_table_*: one rank's shard with lookup (forward) and update (backward)."""

    def __init__(self, *, n_rows: int, dim: int, dp_cut: int, flex_cut: int,
                 tier_dest: np.ndarray | None = None, num_nodes: int = 1,
                 gpus_per_node: int = 1, rank: int = 0, device: int = 0,
                 weight_seed: int = 1234, optimizer: int = OPT_SGD, lr: float = 0.01,
                 eps: float = 1e-8, max_occurrences: int = 1 << 20,
                 nccl_unique_id: bytes | None = None, group: Group | None = None,
                 recv_rows_hint: int = 0):
        self._lib = load()
        self.u = num_nodes * gpus_per_node
        self.dim = dim
        cfg = TableConfig(num_nodes, gpus_per_node, rank, device, dim, n_rows, dp_cut, flex_cut,
                          weight_seed, optimizer, lr, eps, max_occurrences, None, None, recv_rows_hint)
        if group is not None:
            cfg.group = group.handle
            self._group = group  # outlives the table
        self._id_buf = None
        if nccl_unique_id is not None:
            self._id_buf = C.create_string_buffer(nccl_unique_id, len(nccl_unique_id))
            cfg.nccl_unique_id = C.cast(self._id_buf, vp)
        dest_ptr = None
        if tier_dest is not None:
            self._dest = np.ascontiguousarray(tier_dest, dtype=np.uint8)
            dest_ptr = _ptr(self._dest)
        h = vp()
        _check(self._lib.ts_table_create(C.byref(h), C.byref(cfg), dest_ptr))
        self._h = h

    # --- device-pointer entry points -------------------------------------
    def forward(self, d_rows: int, occ: int, d_out: int) -> None:
        _check(self._lib.ts_table_forward(self._h, d_rows, occ, d_out))

    def forward_keys(self, keymap: "KeyMap", d_table_ids: int, d_row_ids: int, occ: int,
                     d_out: int) -> None:
        _check(self._lib.ts_table_forward_keys(self._h, keymap._h, d_table_ids, d_row_ids, occ, d_out))

    def backward(self, d_grad: int) -> None:
        _check(self._lib.ts_table_backward(self._h, d_grad))

    def train_step(self, d_rows: int, occ: int, d_out: int) -> None:
        _check(self._lib.ts_table_train_step(self._h, d_rows, occ, d_out))

    def train_step_host(self, rows: np.ndarray) -> float:
        r = np.ascontiguousarray(rows, dtype=np.uint32)
        loss = C.c_double(0.0)
        _check(self._lib.ts_table_train_step_host(self._h, _ptr(r) if r.size else None, r.size,
                                                  C.byref(loss)))
        return loss.value

    def train_steps_host(self, batches) -> np.ndarray:
        """Pipelined host-buffer steps (ts_table_train_steps_host): one loss per batch."""
        arrs = [np.ascontiguousarray(b, dtype=np.uint32) for b in batches]
        ptrs = (vp * len(arrs))(*[(_ptr(a) if a.size else None) for a in arrs])
        occ = np.array([a.size for a in arrs], dtype=np.uint64)
        losses = np.zeros(len(arrs), dtype=np.float64)
        _check(self._lib.ts_table_train_steps_host(self._h, ptrs, _ptr(occ) if occ.size else None, len(arrs),
                                                   _ptr(losses) if losses.size else None))
        return losses

    def loss(self) -> float:
        v = C.c_double(0.0)
        _check(self._lib.ts_table_loss(self._h, C.byref(v)))
        return v.value

    def stream(self) -> int:
        s = vp()
        _check(self._lib.ts_table_stream(self._h, C.byref(s)))
        return s.value or 0

    def synchronize(self) -> None:
        _check(self._lib.ts_table_synchronize(self._h))

    def recv_capacity(self) -> tuple[int, int]:
        """(receive-buffer rows, times grown) -- U > 1."""
        a, b = C.c_uint64(), C.c_uint64()
        _check(self._lib.ts_table_recv_capacity(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def shard_rows(self) -> tuple[int, int, int]:
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(self._lib.ts_table_shard_rows(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def counters(self) -> np.ndarray:
        out = np.zeros(7 * self.u, dtype=np.uint64)
        _check(self._lib.ts_table_counters(self._h, _ptr(out)))
        return out.reshape(7, self.u)

    def read_rows(self, rows: np.ndarray, with_state: bool = False):
        r = np.ascontiguousarray(rows, dtype=np.uint32)
        w = np.zeros((r.size, self.dim), dtype=np.float32)
        st = np.zeros(r.size, dtype=np.float32) if with_state else None
        _check(self._lib.ts_table_read_rows(self._h, _ptr(r), r.size, _ptr(w),
                                            _ptr(st) if st is not None else None))
        return (w, st) if with_state else w

    def enable_timing(self, on: bool = True) -> None:
        _check(self._lib.ts_table_enable_timing(self._h, 1 if on else 0))

    def phase_times(self) -> dict:
        cap = 32
        ms = (C.c_double * cap)()
        n_launch = (C.c_uint64 * cap)()
        count = C.c_int(0)
        _check(self._lib.ts_table_phase_times(self._h, ms, n_launch, cap, C.byref(count)))
        return {
            self._lib.ts_table_phase_name(i).decode(): (ms[i], n_launch[i]) for i in range(count.value)
        }

    def phase_trace(self) -> list:
        """[(phase name, stream id, t0 ms, t1 ms)] of the last collected window."""
        cap = 4096
        ph = np.zeros(cap, np.int32)
        sid = np.zeros(cap, np.int32)
        t0 = np.zeros(cap, np.float64)
        t1 = np.zeros(cap, np.float64)
        count = C.c_int(0)
        _check(self._lib.ts_table_phase_trace(self._h, _ptr(ph), _ptr(sid), _ptr(t0), _ptr(t1), cap,
                                              C.byref(count)))
        n = min(cap, count.value)
        return [(self._lib.ts_table_phase_name(int(ph[i])).decode(), int(sid[i]), float(t0[i]), float(t1[i]))
                for i in range(n)]

    def close(self):
        if getattr(self, "_h", None):
            _check(self._lib.ts_table_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
