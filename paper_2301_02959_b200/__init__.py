"""tiershard-b200: B200-native per-row tiered sequence-embedding path.

The product is native: ``lib/libtiershard_b200.so`` (host C++ planner API of
include/tiershard/*.hpp + sm_100a kernels + the C-ABI of
include/tiershard_b200.h) and ``bin/ts_driver``.  This Python package is only
the ctypes binding used by the tests and ``bench.py`` (see capi.py); there is
no Python or CPU implementation of any device entry point.
"""
from .capi import (  # noqa: F401
    LIB_PATH,
    DRIVER_PATH,
    TSError,
    Router,
    KeyMap,
    Sampler,
    Table,
    Group,
    plan_footprint,
    load,
    build_info,
    device_count,
    nccl_unique_id,
    kernel_launches,
    COUNTER_NAMES,
    OPT_SGD,
    OPT_ROWWISE_ADAGRAD,
)

__version__ = "0.1.0"
