"""ctypes binding of ``lib/libcace_gpu.so`` — the C ABI declared in include/cace_gpu.h.

The shared library is built in-tree by ``paper_2506_18796_b200.build`` (nvcc,
sm_100a).  There is no fallback: if the library is missing this module raises
on first use, and every replay entry point fails with ``CACE_E_NO_DEVICE`` when no
CUDA device is visible.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CACE_GPU_LIB") or os.path.join(_HERE, "lib", "libcace_gpu.so")

# Status codes (include/cace_gpu.h).
CACE_OK = 0
CACE_E_WINDOW = 1
CACE_E_ACCELERATORS = 2
CACE_E_LOOKUP = 3
CACE_E_RATES = 4
CACE_E_CLOCK = 5
CACE_E_DEADLOCK = 6
CACE_E_RESIDENCY = 7
CACE_E_DEDUP_LENGTH = 8
CACE_E_METRICS_EMPTY = 9
CACE_E_METRICS_NO_TTFT = 10
CACE_E_METRICS_NO_E2E = 11
CACE_E_PARSE = 12
CACE_E_IO = 13
CACE_E_INVALID = 20
CACE_E_CUDA = 21
CACE_E_NO_DEVICE = 22

LOG_FMA, LOG_SSE2 = 0, 1


class CatalogABI(C.Structure):
    _fields_ = [
        ("n_models", C.c_int32),
        ("load_time_s", C.c_void_p),
        ("prefill_rate_tps", C.c_void_p),
        ("decode_rate_tps", C.c_void_p),
        ("expected_output_tokens", C.c_void_p),
        ("lex_rank", C.c_void_p),
        ("task_class", C.c_void_p),
        ("model_id", C.c_void_p),
    ]


class TraceABI(C.Structure):
    _fields_ = [
        ("n_requests", C.c_int64),
        ("arrival_time_s", C.c_void_p),
        ("model", C.c_void_p),
        ("prompt_tokens", C.c_void_p),
        ("output_tokens", C.c_void_p),
    ]


SCENARIO_DTYPE = np.dtype(
    [
        ("trace", "<i4"), ("variant", "<i4"), ("p1_mode", "<i4"), ("window_length", "<i4"),
        ("output_token_normalizer", "<i4"), ("num_accelerators", "<i4"),
        ("models_per_accelerator", "<i4"), ("reserved", "<i4"), ("w1", "<f8"),
        ("unload_time_s", "<f8"),
    ]
)
assert SCENARIO_DTYPE.itemsize == 48

SUMMARY_DTYPE = np.dtype(
    [
        ("hits", "<u8"), ("misses", "<u8"), ("evictions", "<u8"), ("loads", "<u8"),
        ("load_overhead_s", "<f8"), ("max_resident", "<i4"), ("status", "<i4"),
        ("n_completion", "<u8"), ("n_reasoning", "<u8"),
        ("sum_ttft_completion", "<f8"), ("sum_e2e_reasoning", "<f8"),
        ("max_ttft_completion", "<f8"), ("max_e2e_reasoning", "<f8"),
        ("eviction_hash", "<u8"), ("outcome_hash", "<u8"),
    ]
)
assert SUMMARY_DTYPE.itemsize == 112

# LatencySummary / RunMetrics (metrics.hpp:11-29) as cace_run_metrics_t.
LATENCY_DTYPE = np.dtype([("count", "<u8"), ("mean_s", "<f8"), ("p50_s", "<f8"), ("p95_s", "<f8"),
                          ("p99_s", "<f8"), ("max_s", "<f8")])
METRICS_DTYPE = np.dtype(
    [
        ("cache_hit_rate", "<f8"), ("load_overhead_s", "<f8"), ("evictions", "<f8"),
        ("ttft_completion", LATENCY_DTYPE), ("e2e_reasoning", LATENCY_DTYPE),
        ("status", "<i4"), ("reserved", "<i4"),
    ]
)
assert METRICS_DTYPE.itemsize == 128


class DumpABI(C.Structure):
    _fields_ = [
        ("n_dump", C.c_int32),
        ("scenario_index", C.c_void_p),
        ("cold_start", C.c_void_p),
        ("queue_wait_s", C.c_void_p),
        ("load_wait_s", C.c_void_p),
        ("prefill_s", C.c_void_p),
        ("decode_s", C.c_void_p),
        ("ttft_s", C.c_void_p),
        ("e2e_s", C.c_void_p),
        ("evict_cap", C.c_int64),
        ("evict_model", C.c_void_p),
        ("evict_clock", C.c_void_p),
        ("n_evict", C.c_void_p),
    ]


class OptsABI(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("kernel", C.c_int32),
        ("log_variant", C.c_int32),
        ("reserved", C.c_int32),
        ("stream", C.c_void_p),
    ]


EXPORTED = [
    "cace_version", "cace_abi_version", "cace_device_count", "cace_replay_batch",
    "cace_engine_create", "cace_engine_destroy", "cace_engine_plan", "cace_engine_replay_device",
    "cace_engine_status_message", "cace_engine_last_launches", "cace_select_victim_batch",
    "cace_eviction_score_batch", "cace_dedup_window_batch", "cace_service_times_batch",
    "cace_log_selftest", "cace_log_host", "cace_probe_log_variant", "cace_run_metrics_batch", "cace_metrics_select",
    "cace_trace_parse_jsonl", "cace_trace_load_jsonl", "cace_trace_jsonl_size", "cace_trace_jsonl_header",
    "cace_trace_jsonl_copy", "cace_trace_jsonl_free", "cace_replay_batch_multi", "cace_shard_scenarios",
    "cace_nccl_version",
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"CUDA engine library not built: {LIB_PATH}. Run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)."
        )
    L = C.CDLL(LIB_PATH)
    vp, sz = C.c_void_p, C.c_size_t
    i32, i64 = C.c_int32, C.c_int64
    P = C.POINTER
    L.cace_version.restype = C.c_char_p
    L.cace_abi_version.restype = i32
    L.cace_device_count.restype = i32
    L.cace_replay_batch.restype = i32
    L.cace_replay_batch.argtypes = [P(CatalogABI), vp, i32, vp, i64, vp, P(DumpABI), P(OptsABI), C.c_char_p, sz]
    L.cace_replay_batch_multi.restype = i32
    L.cace_replay_batch_multi.argtypes = [P(CatalogABI), vp, i32, vp, i64, vp, vp, i32, P(OptsABI), vp,
                                          C.c_char_p, sz]
    L.cace_shard_scenarios.restype = i32
    L.cace_shard_scenarios.argtypes = [vp, i64, i32, i32, vp]
    L.cace_nccl_version.restype = i32
    L.cace_run_metrics_batch.restype = i32
    L.cace_run_metrics_batch.argtypes = [P(CatalogABI), vp, i32, vp, i64, vp, vp, P(OptsABI), C.c_char_p, sz]
    L.cace_metrics_select.restype = i32
    L.cace_metrics_select.argtypes = [vp, vp, vp, vp, i64, vp, i32, P(OptsABI), C.c_char_p, sz]
    L.cace_trace_parse_jsonl.restype = i32
    L.cace_trace_parse_jsonl.argtypes = [C.c_char_p, sz, P(vp), C.c_char_p, sz]
    L.cace_trace_load_jsonl.restype = i32
    L.cace_trace_load_jsonl.argtypes = [C.c_char_p, P(vp), C.c_char_p, sz]
    L.cace_trace_jsonl_size.restype = i64
    L.cace_trace_jsonl_size.argtypes = [vp]
    L.cace_trace_jsonl_header.restype = None
    L.cace_trace_jsonl_header.argtypes = [vp, vp, vp, vp, vp, vp]
    L.cace_trace_jsonl_copy.restype = None
    L.cace_trace_jsonl_copy.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.cace_trace_jsonl_free.restype = None
    L.cace_trace_jsonl_free.argtypes = [vp]
    L.cace_engine_create.restype = i32
    L.cace_engine_create.argtypes = [P(CatalogABI), vp, i32, P(OptsABI), P(vp), C.c_char_p, sz]
    L.cace_engine_destroy.argtypes = [vp]
    L.cace_engine_plan.restype = i32
    L.cace_engine_plan.argtypes = [vp, vp, i64, C.c_char_p, sz]
    L.cace_engine_replay_device.restype = i32
    L.cace_engine_replay_device.argtypes = [vp, vp, i64, vp, vp, C.c_char_p, sz]
    L.cace_engine_status_message.restype = i32
    L.cace_engine_status_message.argtypes = [vp, i32, C.c_char_p, sz]
    L.cace_engine_last_launches.restype = i32
    L.cace_engine_last_launches.argtypes = [vp]
    L.cace_select_victim_batch.restype = i32
    L.cace_select_victim_batch.argtypes = [P(CatalogABI), i64, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp,
                                           P(OptsABI), C.c_char_p, sz]
    L.cace_eviction_score_batch.restype = i32
    L.cace_eviction_score_batch.argtypes = [P(CatalogABI), i64, vp, vp, i32, vp, vp, vp, vp, vp, P(OptsABI),
                                            C.c_char_p, sz]
    L.cace_dedup_window_batch.restype = i32
    L.cace_dedup_window_batch.argtypes = [i64, i32, vp, vp, vp, vp, vp, P(OptsABI), C.c_char_p, sz]
    L.cace_service_times_batch.restype = i32
    L.cace_service_times_batch.argtypes = [P(CatalogABI), i64, vp, vp, vp, vp, vp, P(OptsABI), C.c_char_p, sz]
    L.cace_log_selftest.restype = i32
    L.cace_log_selftest.argtypes = [vp, i64, i32, vp, P(OptsABI), C.c_char_p, sz]
    L.cace_log_host.restype = None
    L.cace_log_host.argtypes = [vp, i64, i32, vp]
    L.cace_probe_log_variant.restype = i32
    return L


_lib = None


def __getattr__(name):
    """`lib` loads the CUDA engine on first use (importing the package, e.g.
    for the synthetic-workload generators, does not map the library)."""
    global _lib
    if name == "lib":
        if _lib is None:
            _lib = _load()
        return _lib
    raise AttributeError(name)


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
