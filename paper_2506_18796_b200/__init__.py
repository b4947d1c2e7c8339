"""B200-native trace-replay engine for CACE (Context-Aware CodeLLM Eviction, arXiv 2506.18796).

The hot path — replaying request traces under the CACE / LRU / ablation
eviction policies for many independent scenarios — runs as hand-written
sm_100a CUDA kernels behind the C ABI in ``include/cace_gpu.h``
(``lib/libcace_gpu.so``).  This package is the Python mirror of the reference
simulator's API over that ABI (``api``), the synthetic workload builders of
BASELINE.json's configs (``synth``) and the multi-GPU scenario sharding
(``shard``).  Importing it does not map the CUDA library; the first engine
call loads it and fails loudly if it is missing -- there is no CPU fallback.
"""
from .api import (  # noqa: F401
    ClusterConfig,
    Engine,
    Language,
    ModelCatalog,
    ModelDescriptor,
    P1Mode,
    PolicyConfig,
    SimError,
    SimulationReport,
    TaskClass,
    Trace,
    Variant,
    average_metrics,
    metrics_select,
    dedup_window,
    device_count,
    eviction_score,
    load_trace,
    make_scenarios,
    parse_trace,
    run,
    run_batch,
    run_metrics,
    select_victim,
    service_times,
    shard_scenarios,
    version,
)
from ._native import METRICS_DTYPE, SCENARIO_DTYPE, SUMMARY_DTYPE  # noqa: F401
