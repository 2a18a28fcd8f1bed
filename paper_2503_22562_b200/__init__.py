"""B200-native hybrid-batch paged attention for Niyama (arXiv 2503.22562).

The hot path lives in libniyama.so (C ABI: include/niyama.h;
CUDA kernels for sm_100a in csrc/).  This package is a thin ctypes binding
with the same names; PyTorch is used by callers only for device memory,
streams and process groups.
"""
from ._binding import (BF16, DEFAULT_THETA, DEVICE_NONE, NUM_PARAMS, F32, Batch, DecodeQoS, GatherWindow, KVCache, NiyamaError, Plan, PlanInfo, Predictor, QoSArray,
                       SchedBatch, Scheduler, debug_gather_group, get_unique_id, lib, min_slack)

__all__ = ["BF16", "DEFAULT_THETA", "DEVICE_NONE", "NUM_PARAMS", "F32", "Batch", "DecodeQoS", "GatherWindow", "KVCache", "NiyamaError", "Plan", "PlanInfo", "Predictor",
           "QoSArray", "SchedBatch", "Scheduler", "debug_gather_group", "get_unique_id", "lib", "min_slack"]
