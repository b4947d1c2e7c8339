"""Python mirror of the reference simulator's hot-path API, backed by the CUDA engine.

Names, argument meaning and error behaviour follow the reference
(``/root/reference/proj/include/cacesim/*.hpp``):

* ``ModelDescriptor`` / ``ModelCatalog``   catalog.hpp:13-71, catalog.cpp:76-132
* ``Request`` fields as a structure-of-arrays ``Trace``   workload.hpp:15-55
* ``PolicyConfig`` / ``Variant`` / ``P1Mode``   policy.hpp:29-45, types.hpp:63-70
* ``ClusterConfig``   engine.hpp:13-17
* ``run()`` -> ``SimulationReport``   engine.hpp:60-61 (one scenario, full outcomes)
* ``run_batch()``   the scenario fan-out of ``run_grid`` (experiment.cpp:87-122),
  one fixed-size summary per scenario
* ``select_victim`` / ``eviction_score`` / ``dedup_window`` / ``service_times``
  policy.hpp:56-71, engine.hpp:54-55 (batched)

Every call executes on the GPU through ``lib/libcace_gpu.so``; errors the
reference raises as ``cacesim::SimError`` surface as :class:`SimError` with the
reference's message text.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import SCENARIO_DTYPE, SUMMARY_DTYPE, ptr


class SimError(RuntimeError):
    """Mirror of ``cacesim::SimError`` (types.hpp:13-16)."""

    def __init__(self, msg: str, code: int = N.CACE_E_INVALID):
        super().__init__(msg)
        self.code = code


class Language(enum.IntEnum):  # types.hpp:23-32
    JAVA = 0
    PYTHON = 1
    CPP = 2
    C = 3
    GO = 4
    RUST = 5
    CSHARP = 6
    JAVASCRIPT = 7


LANGUAGE_NAMES = ["java", "python", "cpp", "c", "go", "rust", "csharp", "javascript"]


class TaskClass(enum.IntEnum):  # types.hpp:41-44
    COMPLETION = 0
    REASONING = 1


TASK_NAMES = ["completion", "reasoning"]


class Variant(enum.IntEnum):  # types.hpp:63-70
    LRU = 0
    CACE_FULL = 1
    CACE_MINUS_P1 = 2
    CACE_MINUS_P2 = 3
    CACE_MINUS_P3 = 4
    CACE_MINUS_P4 = 5


VARIANT_NAMES = ["lru", "cace", "cace-p1", "cace-p2", "cace-p3", "cace-p4"]


def variant_from_string(s: str) -> Variant:  # types.cpp:69-77
    if s not in VARIANT_NAMES:
        raise SimError("unknown policy variant: " + s)
    return Variant(VARIANT_NAMES.index(s))


class P1Mode(enum.IntEnum):  # policy.hpp:29-34
    PROSE_CONSISTENT = 0
    VERBATIM = 1


@dataclass
class ModelDescriptor:  # catalog.hpp:13-25
    model_id: str
    language: int = 0
    task_class: int = 0
    param_count: int = 0
    weight_bytes: int = 0
    load_time_s: float = 0.0
    prefill_rate_tps: float = 1.0
    decode_rate_tps: float = 1.0
    expected_output_tokens: int = 1


@dataclass
class ProfileParams:  # catalog.hpp:29-34
    staging_bandwidth_Bps: float = 2e9
    load_fixed_overhead_s: float = 1.0


def profile_model(d: ModelDescriptor, p: ProfileParams = ProfileParams()) -> ModelDescriptor:
    """load_time_s = weight_bytes / bandwidth + fixed overhead (catalog.cpp:13-30)."""
    if d.weight_bytes <= 0:
        raise SimError("profile_model: weight_bytes must be positive for " + d.model_id)
    if p.staging_bandwidth_Bps <= 0:
        raise SimError("profile_model: staging bandwidth must be positive")
    if p.load_fixed_overhead_s < 0:
        raise SimError("profile_model: fixed overhead must be non-negative")
    d.load_time_s = float(d.weight_bytes) / p.staging_bandwidth_Bps + p.load_fixed_overhead_s
    return d


class ModelCatalog:
    """Model registry (catalog.hpp:40-71).  Index order = construction order."""

    def __init__(self, models: list[ModelDescriptor], params: ProfileParams | None = None,
                 keyed: bool = True):
        self.models = list(models)
        self.params = params or ProfileParams()
        self._by_id: dict[str, int] = {}
        self._by_key: dict[tuple[int, int], int] = {}
        for i, m in enumerate(self.models):  # catalog.cpp:38-74
            if m.load_time_s <= 0:
                raise SimError("catalog: load_time_s must be positive for " + m.model_id)
            if m.model_id in self._by_id:
                raise SimError("catalog: duplicate model_id " + m.model_id)
            self._by_id[m.model_id] = i
            if keyed:
                key = (int(m.language), int(m.task_class))
                if key in self._by_key:
                    raise SimError("catalog: duplicate (language, task_class) entry for " + m.model_id)
                self._by_key[key] = i
        comp = [m.param_count for m in self.models if m.task_class == TaskClass.COMPLETION]
        reas = [m.param_count for m in self.models if m.task_class == TaskClass.REASONING]
        if keyed and comp and reas and max(comp) >= min(reas):
            raise SimError("catalog: completion models must be smaller than reasoning models")
        self._abi_cache = None

    # catalog.cpp:76-99 (RateDefaults catalog.hpp:75-80)
    @classmethod
    def build_default(cls, languages=None, params: ProfileParams | None = None) -> "ModelCatalog":
        params = params or ProfileParams()
        langs = list(range(8)) if languages is None else [int(l) for l in languages]
        models = []
        for lang in langs:
            for tc in (TaskClass.COMPLETION, TaskClass.REASONING):
                small = tc == TaskClass.COMPLETION
                pc = 500_000_000 if small else 7_000_000_000
                d = ModelDescriptor(
                    model_id=f"{LANGUAGE_NAMES[lang]}-{TASK_NAMES[tc]}", language=lang, task_class=int(tc),
                    param_count=pc, weight_bytes=pc * 2,
                    prefill_rate_tps=8192.0 if small else 2048.0,
                    decode_rate_tps=256.0 if small else 600.0,
                    expected_output_tokens=50 if small else 600)
                models.append(profile_model(d, params))
        return cls(models, params)

    @classmethod
    def synthetic_pool(cls, n_models: int, seed: int = 0) -> "ModelCatalog":
        """A generalised pool of ``n_models`` CodeLLMs (beyond the reference's
        16-model (language x task) key space; BASELINE config 5)."""
        rng = np.random.default_rng(seed)
        models = []
        for i in range(n_models):
            tc = i % 2
            small = tc == 0
            pc = int(rng.integers(3, 15)) * 100_000_000 if small else int(rng.integers(20, 140)) * 1_000_000_000 // 3
            d = ModelDescriptor(model_id=f"codellm-{i:04d}-{TASK_NAMES[tc]}", language=i % 8, task_class=tc,
                                param_count=pc, weight_bytes=pc * 2,
                                prefill_rate_tps=8192.0 if small else 2048.0,
                                decode_rate_tps=256.0 if small else 600.0,
                                expected_output_tokens=50 if small else 600)
            models.append(profile_model(d))
        return cls(models, keyed=False)

    def __len__(self):
        return len(self.models)

    def lookup(self, language: int, task_class: int) -> int:
        """Catalog index for (language, task_class) (catalog.cpp:106-116)."""
        k = self._by_key.get((int(language), int(task_class)))
        if k is None:
            raise SimError(
                f"catalog: no model registered for ({LANGUAGE_NAMES[int(language)]}, {TASK_NAMES[int(task_class)]})",
                N.CACE_E_LOOKUP)
        return k

    def index_of(self, model_id: str) -> int:
        k = self._by_id.get(model_id)
        if k is None:
            raise SimError("catalog: unknown model_id " + model_id)
        return k

    def by_id(self, model_id: str) -> ModelDescriptor:  # catalog.cpp:118-124
        return self.models[self.index_of(model_id)]

    def max_expected_output_tokens(self) -> int:  # catalog.cpp:126-132
        return max([1] + [m.expected_output_tokens for m in self.models])

    def lex_rank(self) -> np.ndarray:
        """Rank of each model_id under std::string operator< (byte order)."""
        ids = [m.model_id.encode() for m in self.models]
        order = sorted(range(len(ids)), key=lambda i: ids[i])
        r = np.empty(len(ids), np.int32)
        r[order] = np.arange(len(ids), dtype=np.int32)
        return r

    def abi(self) -> N.CatalogABI:
        if self._abi_cache is None:
            cols = dict(
                lt=np.array([m.load_time_s for m in self.models], np.float64),
                pr=np.array([m.prefill_rate_tps for m in self.models], np.float64),
                dr=np.array([m.decode_rate_tps for m in self.models], np.float64),
                tok=np.array([m.expected_output_tokens for m in self.models], np.int32),
                lex=self.lex_rank(),
                cls=np.array([m.task_class for m in self.models], np.int32),
            )
            ids = (C.c_char_p * len(self.models))(*[m.model_id.encode() for m in self.models])
            a = N.CatalogABI(len(self.models), ptr(cols["lt"]), ptr(cols["pr"]), ptr(cols["dr"]),
                             ptr(cols["tok"]), ptr(cols["lex"]), ptr(cols["cls"]),
                             C.cast(ids, C.c_void_p))
            self._abi_cache = (a, cols, ids)
        return self._abi_cache[0]


@dataclass
class Trace:
    """Request trace as structure-of-arrays (workload.hpp:15-55).

    ``model[i]`` is the catalog index ``catalog.lookup(language, task_class)``
    of request i; request_id is the position."""

    arrival_time_s: np.ndarray
    model: np.ndarray
    prompt_tokens: np.ndarray
    output_tokens: np.ndarray
    seed: int = 0

    def __post_init__(self):
        self.arrival_time_s = np.ascontiguousarray(self.arrival_time_s, np.float64)
        self.model = np.ascontiguousarray(self.model, np.int32)
        self.prompt_tokens = np.ascontiguousarray(self.prompt_tokens, np.int32)
        self.output_tokens = np.ascontiguousarray(self.output_tokens, np.int32)

    def __len__(self):
        return len(self.arrival_time_s)

    @classmethod
    def from_requests(cls, catalog: ModelCatalog, requests) -> "Trace":
        """requests: iterable of (arrival_time_s, language, task_class, prompt, output)."""
        rows = list(requests)
        return cls(np.array([r[0] for r in rows], np.float64),
                   np.array([catalog.lookup(r[1], r[2]) for r in rows], np.int32),
                   np.array([r[3] for r in rows], np.int32), np.array([r[4] for r in rows], np.int32))

    def abi(self) -> N.TraceABI:
        return N.TraceABI(len(self), ptr(self.arrival_time_s), ptr(self.model), ptr(self.prompt_tokens),
                          ptr(self.output_tokens))

    @property
    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.arrival_time_s, self.model, self.prompt_tokens, self.output_tokens))


@dataclass
class PolicyConfig:  # policy.hpp:39-45
    variant: int = Variant.CACE_FULL
    w1: float = 1.0
    window_length: int = 10
    output_token_normalizer: int = 600
    p1_mode: int = P1Mode.PROSE_CONSISTENT


@dataclass
class ClusterConfig:  # engine.hpp:13-17
    num_accelerators: int = 4
    models_per_accelerator: int = 1
    unload_time_s: float = 0.0


def make_scenarios(rows) -> np.ndarray:
    """rows: iterable of (trace, PolicyConfig, ClusterConfig) -> SCENARIO_DTYPE array."""
    rows = list(rows)
    a = np.zeros(len(rows), SCENARIO_DTYPE)
    for i, (t, p, c) in enumerate(rows):
        a[i] = (t, int(p.variant), int(p.p1_mode), p.window_length, p.output_token_normalizer,
                c.num_accelerators, c.models_per_accelerator, 0, p.w1, c.unload_time_s)
    return a


@dataclass
class SimCounters:  # engine.hpp:32-37
    hits: int = 0
    misses: int = 0
    evictions: int = 0
    load_overhead_s: float = 0.0


@dataclass
class SimulationReport:  # engine.hpp:46-52 (outcomes as structure-of-arrays)
    counters: SimCounters
    max_resident: int
    loads: int
    cold_start: np.ndarray
    queue_wait_s: np.ndarray
    load_wait_s: np.ndarray
    prefill_s: np.ndarray
    decode_s: np.ndarray
    ttft_s: np.ndarray
    e2e_s: np.ndarray
    evicted_model: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    eviction_clock: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    summary: np.ndarray | None = None


KERNEL_AUTO, KERNEL_LANE, KERNEL_WARP = 0, 1, 2


def _opts(device: int = 0, log_variant: int = -1, kernel: int = KERNEL_AUTO) -> N.OptsABI:
    return N.OptsABI(device, kernel, log_variant, 0, None)


def _raise(rc: int, msg) -> None:
    if rc != N.CACE_OK:
        raise SimError(msg.value.decode(errors="replace"), rc)


def _trace_array(traces):
    arr = (N.TraceABI * max(1, len(traces)))(*[t.abi() for t in traces])
    return arr


def shard_scenarios(scenarios: np.ndarray, n_models: int, n_shards: int) -> np.ndarray:
    """Shard of every scenario (cace_shard_scenarios): each (capacity, trace)
    group is cut into warps of 32 spread evenly over the shards.  No GPU."""
    scenarios = np.ascontiguousarray(scenarios, SCENARIO_DTYPE)
    out = np.zeros(len(scenarios), np.int32)
    rc = N.lib.cace_shard_scenarios(ptr(scenarios), len(scenarios), n_models, n_shards, ptr(out))
    if rc != N.CACE_OK:
        raise SimError("cace_shard_scenarios: invalid arguments", rc)
    return out


def run_batch(traces: list[Trace], catalog: ModelCatalog, scenarios: np.ndarray, device: int = 0,
              dump_scenarios=None, evict_cap: int | None = None, raise_on_error: bool = True,
              kernel: int = KERNEL_AUTO, devices=None, return_gather_kind: bool = False):
    """Replay every scenario on the GPU (host buffers in and out).

    Returns the summary array (SUMMARY_DTYPE); with ``dump_scenarios`` also a
    list of per-scenario full reports.  ``devices`` (a list of ordinals):
    the sweep is sharded over those devices of this process
    (cace_replay_batch_multi, summaries gathered over NCCL); summaries only."""
    scenarios = np.ascontiguousarray(scenarios, SCENARIO_DTYPE)
    summ = np.zeros(len(scenarios), SUMMARY_DTYPE)
    tarr = _trace_array(traces)
    if devices is not None:
        if dump_scenarios is not None:
            raise ValueError("run_batch: full dumps replay on one device")
        devs = np.ascontiguousarray(devices, np.int32)
        msg = C.create_string_buffer(1024)
        gk = C.c_int32(-1)
        rc = N.lib.cace_replay_batch_multi(C.byref(catalog.abi()), C.cast(tarr, C.c_void_p), len(traces),
                                           ptr(scenarios), len(scenarios), ptr(summ), ptr(devs), len(devs),
                                           C.byref(_opts(int(devs[0]), kernel=kernel)), C.byref(gk), msg, 1024)
        if rc != N.CACE_OK and (raise_on_error or rc >= N.CACE_E_INVALID):
            _raise(rc, msg)
        return (summ, int(gk.value)) if return_gather_kind else summ
    dump = None
    dump_abi = None
    if dump_scenarios is not None and len(dump_scenarios):
        idx = np.ascontiguousarray(dump_scenarios, np.int64)
        sizes = [len(traces[int(scenarios[i]["trace"])]) for i in idx]
        total = int(sum(sizes))
        cap = int(evict_cap if evict_cap is not None else max(sizes) + 1)
        dump = dict(idx=idx, sizes=sizes, cold=np.zeros(total, np.uint8),
                    **{k: np.zeros(total, np.float64) for k in ("qw", "lw", "pf", "dc", "tt", "ee")},
                    em=np.zeros(len(idx) * cap, np.int32), ec=np.zeros(len(idx) * cap, np.float64),
                    ne=np.zeros(len(idx), np.int64), cap=cap)
        dump_abi = N.DumpABI(len(idx), ptr(idx), ptr(dump["cold"]), ptr(dump["qw"]), ptr(dump["lw"]),
                             ptr(dump["pf"]), ptr(dump["dc"]), ptr(dump["tt"]), ptr(dump["ee"]), cap,
                             ptr(dump["em"]), ptr(dump["ec"]), ptr(dump["ne"]))
    msg = C.create_string_buffer(1024)
    opts = _opts(device, kernel=kernel)
    rc = N.lib.cace_replay_batch(C.byref(catalog.abi()), C.cast(tarr, C.c_void_p), len(traces), ptr(scenarios),
                                 len(scenarios), ptr(summ), C.byref(dump_abi) if dump_abi else None,
                                 C.byref(opts), msg, 1024)
    if rc != N.CACE_OK and (raise_on_error or rc >= N.CACE_E_INVALID):
        _raise(rc, msg)
    if dump is None:
        return summ
    reports = []
    off = 0
    for k, i in enumerate(dump["idx"]):
        n = dump["sizes"][k]
        sl = slice(off, off + n)
        off += n
        s = summ[i]
        ne = int(dump["ne"][k])
        cap = dump["cap"]
        reports.append(SimulationReport(
            SimCounters(int(s["hits"]), int(s["misses"]), int(s["evictions"]), float(s["load_overhead_s"])),
            int(s["max_resident"]), int(s["loads"]), dump["cold"][sl].astype(bool), dump["qw"][sl].copy(),
            dump["lw"][sl].copy(), dump["pf"][sl].copy(), dump["dc"][sl].copy(), dump["tt"][sl].copy(),
            dump["ee"][sl].copy(), dump["em"][k * cap:k * cap + min(ne, cap)].copy(),
            dump["ec"][k * cap:k * cap + min(ne, cap)].copy(), s.copy()))
    return summ, reports


PATTERN_NAMES = ("uniform", "ide-heavy", "popularity-skewed")  # types.cpp:39-46


@dataclass
class TraceHeader:
    """Trace metadata of the JSONL header (workload.hpp:46-55)."""

    pattern: int
    seed: int
    arrival_rate_per_s: float
    window_duration_s: float
    windows: int


def _trace_from_handle(h, catalog: ModelCatalog):
    n = int(N.lib.cace_trace_jsonl_size(h))
    pat, win = C.c_int32(0), C.c_int32(0)
    seed = C.c_uint64(0)
    rate, dur = C.c_double(0.0), C.c_double(0.0)
    N.lib.cace_trace_jsonl_header(h, C.byref(pat), C.byref(seed), C.byref(rate), C.byref(dur), C.byref(win))
    rid = np.zeros(n, np.uint64)
    arr = np.zeros(n, np.float64)
    lang = np.zeros(n, np.int32)
    cls = np.zeros(n, np.int32)
    pr = np.zeros(n, np.int32)
    out = np.zeros(n, np.int32)
    N.lib.cace_trace_jsonl_copy(h, ptr(rid), ptr(arr), ptr(lang), ptr(cls), ptr(pr), ptr(out))
    # catalog.lookup(language, task_class) per distinct pair (catalog.cpp:106-116)
    key = lang.astype(np.int64) * 2 + cls
    model = np.zeros(n, np.int32)
    for k in np.unique(key):
        model[key == k] = catalog.lookup(int(k) // 2, int(k) % 2)
    hdr = TraceHeader(pat.value, seed.value, rate.value, dur.value, win.value)
    return Trace(arr, model, pr, out, seed=seed.value), hdr, rid


def parse_trace(text, catalog: ModelCatalog):
    """``parse_trace`` (workload.cpp:204-266) of JSONL text (str or bytes),
    parsed in native code on all host threads; returns (Trace with catalog
    indices, TraceHeader, request_id array).  Raises SimError with the
    reference's ParseError text."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    msg = C.create_string_buffer(4096)
    rc = N.lib.cace_trace_parse_jsonl(data, len(data), C.byref(h), msg, 4096)
    if rc != N.CACE_OK:
        _raise(rc, msg)
    try:
        return _trace_from_handle(h, catalog)
    finally:
        N.lib.cace_trace_jsonl_free(h)


def load_trace(path: str, catalog: ModelCatalog):
    """``load_trace`` (workload.cpp:274-280): parse_trace of a JSONL file."""
    h = C.c_void_p()
    msg = C.create_string_buffer(4096)
    rc = N.lib.cace_trace_load_jsonl(str(path).encode(), C.byref(h), msg, 4096)
    if rc != N.CACE_OK:
        _raise(rc, msg)
    try:
        return _trace_from_handle(h, catalog)
    finally:
        N.lib.cace_trace_jsonl_free(h)


def run_metrics(traces: list[Trace], catalog: ModelCatalog, scenarios: np.ndarray, device: int = 0,
                raise_on_error: bool = True, kernel: int = KERNEL_AUTO, with_summaries: bool = False):
    """``compute_run_metrics`` (metrics.cpp:35-62) of every scenario's replay,
    computed on the GPU (``cace_run_metrics_batch``): a METRICS_DTYPE array
    (cache hit rate, load overhead, evictions, nearest-rank TTFT/E2E
    summaries).  Scenarios whose metrics the reference could not compute
    carry a non-zero ``status`` (raised as SimError when ``raise_on_error``)."""
    scenarios = np.ascontiguousarray(scenarios, SCENARIO_DTYPE)
    out = np.zeros(len(scenarios), N.METRICS_DTYPE)
    summ = np.zeros(len(scenarios), SUMMARY_DTYPE) if with_summaries else None
    tarr = _trace_array(traces)
    msg = C.create_string_buffer(1024)
    opts = _opts(device, kernel=kernel)
    rc = N.lib.cace_run_metrics_batch(C.byref(catalog.abi()), C.cast(tarr, C.c_void_p), len(traces),
                                      ptr(scenarios), len(scenarios), ptr(out), ptr(summ), C.byref(opts), msg,
                                      1024)
    if rc != N.CACE_OK and (raise_on_error or rc >= N.CACE_E_INVALID):
        _raise(rc, msg)
    return (out, summ) if with_summaries else out


def average_metrics(runs: np.ndarray) -> np.ndarray:
    """``average_metrics`` (metrics.cpp:89-104): elementwise mean over the
    per-seed RunMetrics of one grid cell, summed in the given order."""
    runs = np.asarray(runs, N.METRICS_DTYPE)
    if len(runs) == 0:
        raise SimError("average_metrics: no runs")
    k = float(len(runs))
    avg = np.zeros((), N.METRICS_DTYPE)
    for f in ("cache_hit_rate", "load_overhead_s", "evictions"):
        acc = 0.0
        for r in runs:
            acc += float(r[f])
        avg[f] = acc / k
    for lf in ("ttft_completion", "e2e_reasoning"):
        cnt = 0
        sums = {q: 0.0 for q in ("mean_s", "p50_s", "p95_s", "p99_s", "max_s")}
        for r in runs:
            cnt += int(r[lf]["count"])
            for q in sums:
                sums[q] += float(r[lf][q])
        avg[lf]["count"] = cnt
        for q, v in sums.items():
            avg[lf][q] = v / k
    return avg


def metrics_select(segments, spec: int = 1, device: int = 0) -> np.ndarray:
    """The nearest-rank order statistics of summarize (metrics.cpp:14-33) on
    the device: segments = [(ttft_samples, e2e_samples), ...] (latencies >= 0)
    -> float64 array [n, 2, 4] of {p50, p95, p99, max} per class (zeros for an
    empty class).  Runs the select kernel of run_metrics (spec: 1 speculative
    first digit, 0 off, 2 speculation forced to miss)."""
    segs = [(np.ascontiguousarray(a, np.float64).ravel(), np.ascontiguousarray(b, np.float64).ravel())
            for a, b in segments]
    n = len(segs)
    out = np.zeros((n, 2, 4), np.float64)
    if n == 0:
        return out
    flat = np.concatenate([np.concatenate([a, b]) for a, b in segs]) if n else np.zeros(0)
    ncomp = np.array([len(a) for a, _ in segs], np.uint32)
    nreq = np.array([len(a) + len(b) for a, b in segs], np.uint32)
    off = np.zeros(n, np.int64)
    off[1:] = np.cumsum(nreq.astype(np.int64))[:-1]
    flat = np.ascontiguousarray(flat if len(flat) else np.zeros(1), np.float64)
    msg = C.create_string_buffer(1024)
    opts = _opts(device)
    rc = N.lib.cace_metrics_select(ptr(flat), ptr(off), ptr(ncomp), ptr(nreq), n, ptr(out), int(spec),
                                   C.byref(opts), msg, len(msg))
    if rc != N.CACE_OK:
        _raise(rc, msg)
    return out


def run(trace: Trace, catalog: ModelCatalog, cluster: ClusterConfig = ClusterConfig(),
        policy: PolicyConfig = PolicyConfig(), device: int = 0, kernel: int = KERNEL_AUTO) -> SimulationReport:
    """``cacesim::run`` (engine.cpp:76-239) on the GPU: one scenario, full report."""
    sc = make_scenarios([(0, policy, cluster)])
    _, reps = run_batch([trace], catalog, sc, device=device, dump_scenarios=[0], kernel=kernel)
    return reps[0]


class Engine:
    """Device-resident engine (cace_engine_*): traces uploaded once, sweeps
    replayed from device arrays.  Used by bench.py and the multi-GPU shards."""

    def __init__(self, catalog: ModelCatalog, traces: list[Trace], device: int = 0, stream: int | None = None,
                 kernel: int = KERNEL_AUTO):
        self._h = C.c_void_p()
        self.catalog = catalog
        self.traces = traces
        tarr = _trace_array(traces)
        msg = C.create_string_buffer(1024)
        opts = N.OptsABI(device, kernel, -1, 0, stream)
        rc = N.lib.cace_engine_create(C.byref(catalog.abi()), C.cast(tarr, C.c_void_p), len(traces),
                                      C.byref(opts), C.byref(self._h), msg, 1024)
        _raise(rc, msg)

    def plan(self, scenarios: np.ndarray) -> None:
        scenarios = np.ascontiguousarray(scenarios, SCENARIO_DTYPE)
        msg = C.create_string_buffer(1024)
        _raise(N.lib.cace_engine_plan(self._h, ptr(scenarios), len(scenarios), msg, 1024), msg)

    def replay_device(self, d_scenarios_ptr: int, n: int, d_summaries_ptr: int, stream: int | None = None) -> int:
        msg = C.create_string_buffer(1024)
        rc = N.lib.cace_engine_replay_device(self._h, C.c_void_p(d_scenarios_ptr), n, C.c_void_p(d_summaries_ptr),
                                             C.c_void_p(stream) if stream else None, msg, 1024)
        _raise(rc, msg)
        return N.lib.cace_engine_last_launches(self._h)

    def status_message(self, status: int) -> str:
        msg = C.create_string_buffer(1024)
        N.lib.cace_engine_status_message(self._h, int(status), msg, 1024)
        return msg.value.decode(errors="replace")

    def close(self):
        if self._h:
            N.lib.cace_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------
# Policy-level batch entry points (policy.hpp:56-71, engine.hpp:54-55)

def _policy_rows(policies) -> np.ndarray:
    return make_scenarios([(0, p, ClusterConfig()) for p in policies])


def select_victim(catalog: ModelCatalog, instances, device: int = 0) -> np.ndarray:
    """instances: list of (entries=[(model_idx, last_used, busy)], window_models(deduped), clock, PolicyConfig).
    Returns victim catalog index per instance (-1 = every resident busy)."""
    B = len(instances)
    me = max(1, max(len(x[0]) for x in instances))
    mw = max(1, max(len(x[1]) for x in instances))
    ne = np.array([len(x[0]) for x in instances], np.int32)
    em = np.zeros((B, me), np.int32)
    lu = np.zeros((B, me), np.float64)
    bz = np.zeros((B, me), np.uint8)
    nw = np.array([len(x[1]) for x in instances], np.int32)
    wm = np.zeros((B, mw), np.int32)
    clk = np.array([x[2] for x in instances], np.float64)
    for b, (ents, win, _, _) in enumerate(instances):
        for k, (m, l, busy) in enumerate(ents):
            em[b, k], lu[b, k], bz[b, k] = m, l, 1 if busy else 0
        wm[b, :len(win)] = win
    pol = _policy_rows([x[3] for x in instances])
    out = np.zeros(B, np.int32)
    msg = C.create_string_buffer(1024)
    opts = _opts(device)
    rc = N.lib.cace_select_victim_batch(C.byref(catalog.abi()), B, me, ptr(ne), ptr(em), ptr(lu), ptr(bz), mw,
                                        ptr(nw), ptr(wm), ptr(clk), ptr(pol), ptr(out), C.byref(opts), msg, 1024)
    _raise(rc, msg)
    return out


def eviction_score(catalog: ModelCatalog, instances, device: int = 0) -> np.ndarray:
    """instances: list of (model_idx, last_used, window_models(deduped), clock, PolicyConfig).
    Returns [B,5] = p1, p2, p3, p4, total."""
    B = len(instances)
    mw = max(1, max(len(x[2]) for x in instances))
    m = np.array([x[0] for x in instances], np.int32)
    lu = np.array([x[1] for x in instances], np.float64)
    nw = np.array([len(x[2]) for x in instances], np.int32)
    wm = np.zeros((B, mw), np.int32)
    for b, x in enumerate(instances):
        wm[b, :len(x[2])] = x[2]
    clk = np.array([x[3] for x in instances], np.float64)
    pol = _policy_rows([x[4] for x in instances])
    out = np.zeros((B, 5), np.float64)
    msg = C.create_string_buffer(1024)
    opts = _opts(device)
    rc = N.lib.cace_eviction_score_batch(C.byref(catalog.abi()), B, ptr(m), ptr(lu), mw, ptr(nw), ptr(wm),
                                         ptr(clk), ptr(pol), ptr(out), C.byref(opts), msg, 1024)
    _raise(rc, msg)
    return out


def dedup_window(pending_lists, lengths, device: int = 0) -> list[np.ndarray]:
    B = len(pending_lists)
    mp = max(1, max(len(p) for p in pending_lists))
    npd = np.array([len(p) for p in pending_lists], np.int32)
    pm = np.zeros((B, mp), np.int32)
    for b, p in enumerate(pending_lists):
        pm[b, :len(p)] = p
    ln = np.ascontiguousarray(lengths, np.int32)
    out = np.zeros((B, mp), np.int32)
    no = np.zeros(B, np.int32)
    msg = C.create_string_buffer(1024)
    opts = _opts(device)
    rc = N.lib.cace_dedup_window_batch(B, mp, ptr(npd), ptr(pm), ptr(ln), ptr(out), ptr(no), C.byref(opts), msg, 1024)
    _raise(rc, msg)
    return [out[b, :no[b]].copy() for b in range(B)]


def service_times(catalog: ModelCatalog, model, prompt, output, device: int = 0):
    model = np.ascontiguousarray(model, np.int32)
    prompt = np.ascontiguousarray(prompt, np.int32)
    output = np.ascontiguousarray(output, np.int32)
    pf = np.zeros(len(model))
    dc = np.zeros(len(model))
    msg = C.create_string_buffer(1024)
    opts = _opts(device)
    rc = N.lib.cace_service_times_batch(C.byref(catalog.abi()), len(model), ptr(model), ptr(prompt), ptr(output),
                                        ptr(pf), ptr(dc), C.byref(opts), msg, 1024)
    _raise(rc, msg)
    return pf, dc


def device_log(x, log_variant: int = -1, device: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros_like(x)
    msg = C.create_string_buffer(1024)
    opts = _opts(device)
    _raise(N.lib.cace_log_selftest(ptr(x), len(x), log_variant, ptr(out), C.byref(opts), msg, 1024), msg)
    return out


def host_log(x, log_variant: int = -1) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros_like(x)
    N.lib.cace_log_host(ptr(x), len(x), log_variant, ptr(out))
    return out


def probe_log_variant() -> int:
    return N.lib.cace_probe_log_variant()


def device_count() -> int:
    return N.lib.cace_device_count()


def version() -> str:
    return N.lib.cace_version().decode()
