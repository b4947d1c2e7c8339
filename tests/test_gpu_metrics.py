"""GPU parity of the on-device RunMetrics (cace_run_metrics_batch) against the
reference's compute_run_metrics(run(...)) (metrics.cpp:14-62).

Counts, nearest-rank p50/p95/p99, max, hit rate, load overhead and evictions
must be bit-identical; the mean divides the replay-order sum while the
reference sums the sorted samples (metrics.cpp:26), so it is checked to
1e-12 relative (north_star's latency bar is 1e-9 relative)."""
import numpy as np
import pytest

from tests.helpers import bits, ref_catalog, ref_scenario, ref_trace

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2506_18796_b200")
from paper_2506_18796_b200 import _native as N  # noqa: E402
from paper_2506_18796_b200 import api, synth  # noqa: E402
from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig  # noqa: E402

MEAN_RTOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if P.device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU tests must run on a B200 (no CPU fallback)")


def _check(ref, catalog, traces, sc, got, ctx=""):
    rcat = ref_catalog(ref, catalog)
    for k in range(len(sc)):
        want = ref.run_metrics(rcat, ref_trace(traces[int(sc[k]["trace"])]), ref_scenario(ref, sc[k]))
        g = got[k]
        c = f"{ctx} scenario {k} {sc[k]}"
        assert g["status"] == 0, c
        for f in ("cache_hit_rate", "load_overhead_s", "evictions"):
            assert bits([g[f]])[0] == bits([want[f]])[0], f"{c} {f}: {g[f]} vs {want[f]}"
        for lf in ("ttft_completion", "e2e_reasoning"):
            assert int(g[lf]["count"]) == want[lf]["count"], c
            for q in ("p50_s", "p95_s", "p99_s", "max_s"):
                assert bits([g[lf][q]])[0] == bits([want[lf][q]])[0], f"{c} {lf}.{q}: {g[lf][q]!r} vs {want[lf][q]!r}"
            m, wm = float(g[lf]["mean_s"]), want[lf]["mean_s"]
            assert abs(m - wm) <= MEAN_RTOL * abs(wm), f"{c} {lf}.mean {m!r} vs {wm!r}"


@pytest.mark.parametrize("seed", range(4))
def test_run_metrics_random_scenarios(ref, seed):
    rng = np.random.default_rng(900 + seed)
    catalog = synth.eight_model_catalog() if seed % 2 == 0 else api.ModelCatalog.build_default()
    traces = [synth.mixed_trace(catalog, int(n), seed=50 * seed + k, rate=float(r), bursty=bool(k % 2))
              for k, (n, r) in enumerate([(1, 1.0), (37, 3.0), (2500, 10.0), (6000, 0.5)])]
    rows = []
    for _ in range(24):
        pol = PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.choice([0.0, 0.5, 1.0, 1.7])),
                           window_length=int(rng.choice([1, 2, 10, 64])),
                           output_token_normalizer=600, p1_mode=int(rng.integers(0, 2)))
        cl = ClusterConfig(num_accelerators=int(rng.integers(1, 9)),
                           unload_time_s=float(rng.choice([0.0, 0.5])))
        rows.append((int(rng.integers(1, 4)), pol, cl))
    sc = api.make_scenarios(rows)
    got, summ = P.run_metrics(traces, catalog, sc, with_summaries=True)
    _check(ref, catalog, traces, sc, got, f"seed {seed}")
    # the summaries are the replay's own (bit-identical to run_batch)
    from tests.helpers import assert_summaries_equal

    assert_summaries_equal(summ, P.run_batch(traces, catalog, sc), "run_metrics summaries")


def test_run_metrics_config4_slice(ref):
    """A slice of the config-4 grid (every variant / window / P1 mode, C 1..8)."""
    catalog = synth.eight_model_catalog()
    traces = [synth.mixed_trace(catalog, 20_000, seed=1 + s) for s in range(2)]
    sc = synth.scenario_grid(synth.weight_vectors_cfg3()[::97], range(1, 9), 2,
                             catalog.max_expected_output_tokens())
    got = P.run_metrics(traces, catalog, sc)
    pick = np.random.default_rng(3).choice(len(sc), 40, replace=False)
    _check(ref, catalog, traces, sc[pick], got[pick], "cfg4 slice")


def test_run_metrics_chunked_pipeline(ref, monkeypatch):
    """A tiny sample budget cuts the sweep into one-warp chunks (cace_run_metrics_batch's
    pipeline); a one-warp chunk (5 MB) exceeds the 1 MB budget, so the pipeline
    falls back to a single ring instead of allocating all 8 (advisor round 1):
    same records as one chunk per segment, and bit-exact against the reference."""
    catalog = synth.eight_model_catalog()
    traces = [synth.mixed_trace(catalog, 20_000, seed=7 + s) for s in range(2)]
    sc = synth.scenario_grid(synth.weight_vectors_cfg3()[::211], range(1, 9), 2,
                             catalog.max_expected_output_tokens())
    whole = P.run_metrics(traces, catalog, sc)
    monkeypatch.setenv("CACE_METRICS_BUDGET_MB", "1")
    chunked = P.run_metrics(traces, catalog, sc)
    assert whole.tobytes() == chunked.tobytes()
    pick = np.random.default_rng(5).choice(len(sc), 16, replace=False)
    _check(ref, catalog, traces, sc[pick], chunked[pick], "chunked")


def test_run_metrics_long_trace_heavy_bins(ref):
    """100k requests: the select's working set is compacted in place in global
    memory (more than METRICS_LIST keys under the targets' prefixes), including
    bins of identical samples (no-eviction capacities: warm-hit TTFT = prefill)."""
    catalog = synth.eight_model_catalog()
    traces = [synth.mixed_trace(catalog, 100_000, seed=21)]
    rows = [(0, PolicyConfig(variant=v, output_token_normalizer=600), ClusterConfig(num_accelerators=c))
            for v in (api.Variant.LRU, api.Variant.CACE_FULL) for c in (1, 2, 3, 8)]
    sc = api.make_scenarios(rows)
    got = P.run_metrics(traces, catalog, sc)
    _check(ref, catalog, traces, sc, got, "long trace")


def test_run_metrics_speculative_digit_paths(ref, monkeypatch):
    """The select's speculative first digit (segments >= 16384 samples): on,
    off, and with every guess forced wrong (CACE_METRICS_SPEC=2, the fallback
    path) give identical records, bit-exact against the reference."""
    catalog = synth.eight_model_catalog()
    traces = [synth.mixed_trace(catalog, 60_000, seed=33, bursty=True)]
    rows = [(0, PolicyConfig(variant=v, output_token_normalizer=600, window_length=w), ClusterConfig(num_accelerators=c))
            for v in (api.Variant.LRU, api.Variant.CACE_FULL) for c in (1, 3, 8) for w in (2, 10)]
    sc = api.make_scenarios(rows)
    res = {}
    for mode in ("1", "0", "2"):
        monkeypatch.setenv("CACE_METRICS_SPEC", mode)
        res[mode] = P.run_metrics(traces, catalog, sc)
    assert res["1"].tobytes() == res["0"].tobytes()
    assert res["2"].tobytes() == res["0"].tobytes()
    _check(ref, catalog, traces, sc, res["1"], "speculative select")


def test_run_metrics_errors_match_reference(ref):
    """compute_run_metrics' SimErrors (metrics.cpp:37-58): empty report, no
    completion outcomes, no reasoning outcomes."""
    catalog = synth.eight_model_catalog()
    comp = [m for m in range(len(catalog)) if catalog.models[m].task_class == api.TaskClass.COMPLETION]
    reas = [m for m in range(len(catalog)) if catalog.models[m].task_class == api.TaskClass.REASONING]
    t_comp = api.Trace(np.arange(5, dtype=float), np.array(comp[:1] * 5), np.full(5, 100), np.full(5, 10))
    t_reas = api.Trace(np.arange(5, dtype=float), np.array(reas[:1] * 5), np.full(5, 100), np.full(5, 10))
    t_empty = api.Trace(np.zeros(0), np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32))
    traces = [t_comp, t_reas, t_empty]
    sc = api.make_scenarios([(t, PolicyConfig(), ClusterConfig()) for t in range(3)])
    got = P.run_metrics(traces, catalog, sc, raise_on_error=False)
    assert list(got["status"]) == [N.CACE_E_METRICS_NO_E2E, N.CACE_E_METRICS_NO_TTFT, N.CACE_E_METRICS_EMPTY]
    rcat = ref_catalog(ref, catalog)
    msgs = []
    for k in range(3):
        with pytest.raises(Exception) as ei:
            ref.run_metrics(rcat, ref_trace(traces[k]), ref_scenario(ref, sc[k]))
        msgs.append(str(ei.value))
    for k in range(3):
        with pytest.raises(api.SimError) as ei:
            P.run_metrics([traces[k]], catalog, api.make_scenarios([(0, PolicyConfig(), ClusterConfig())]))
        assert str(ei.value) == msgs[k], (str(ei.value), msgs[k])


def test_average_metrics_matches_reference_formula():
    """average_metrics (metrics.cpp:89-104): elementwise mean in run order."""
    runs = np.zeros(3, N.METRICS_DTYPE)
    for i in range(3):
        runs[i]["cache_hit_rate"] = 0.1 * (i + 1)
        runs[i]["evictions"] = 10 * i
        runs[i]["ttft_completion"]["count"] = 5
        runs[i]["ttft_completion"]["p99_s"] = 1.0 + i
    avg = P.average_metrics(runs)
    assert avg["cache_hit_rate"] == ((0.1 + 0.2) + 0.30000000000000004) / 3.0
    assert avg["evictions"] == 10.0 and avg["ttft_completion"]["count"] == 15
    assert avg["ttft_completion"]["p99_s"] == 2.0


def _nearest_rank_stats(a):
    """summarize's order statistics (metrics.cpp:14-33) on the sorted samples."""
    if len(a) == 0:
        return np.zeros(4)
    s = np.sort(np.asarray(a, np.float64))
    n = len(s)
    out = []
    for q in (0.50, 0.95, 0.99):
        r = int(np.ceil(q * float(n)))
        r = min(max(r, 1), n)
        out.append(s[r - 1])
    out.append(s[-1])
    return np.array(out)


@pytest.mark.parametrize("spec", [0, 1, 2])
def test_metrics_select_kernel_edges(spec):
    """The select kernel alone against np.sort + nearest rank, bit-exact:
    lengths around the shared-list (5120), in-place (2 x 5120) and
    speculation (16384) thresholds, heavy duplicates, constants, values
    straddling the top-byte boundary at 2.0, zeros and subnormals."""
    rng = np.random.default_rng(42 + spec)
    lens = [1, 2, 3, 31, 5119, 5120, 5121, 10239, 10240, 10241, 16383, 16384, 16385, 70000]
    segs = []
    for k, n in enumerate(lens):
        kind = k % 5
        if kind == 0:
            a = rng.exponential(3.0, n)
        elif kind == 1:
            a = np.round(rng.exponential(2.0, n), 2)  # heavy duplicates
        elif kind == 2:
            a = np.full(n, 1.25)
        elif kind == 3:
            a = rng.uniform(1.9, 2.1, n)  # top byte changes at 2.0
        else:
            a = np.concatenate([np.zeros(n // 2), rng.uniform(0, 1e-310, n - n // 2)])
        b = rng.permutation(a)[: max(1, n // 3)] * 1.5
        segs.append((a, b))
    segs.append((np.zeros(0), rng.uniform(0, 5, 20000)))  # empty class -> zeros
    got = P.metrics_select(segs, spec=spec)
    for i, (a, b) in enumerate(segs):
        for c, x in enumerate((a, b)):
            want = _nearest_rank_stats(x)
            assert np.array_equal(bits(got[i, c]), bits(want)), (i, c, len(x), got[i, c], want)


@pytest.mark.gpu
def test_metrics_select_rejects_overlapping_segments():
    """The select compacts each segment in place, so the C ABI rejects
    overlapping sample ranges instead of racing (advisor round 1)."""
    import ctypes as C

    from paper_2506_18796_b200 import _native as N

    flat = np.arange(10, dtype=np.float64)
    off = np.array([0, 4], np.int64)
    ncomp = np.array([3, 3], np.uint32)
    stat = np.zeros(16)
    msg = C.create_string_buffer(256)
    opts = N.OptsABI(0, 0, -1, 0, None)
    for nreq, want in ((np.array([4, 6], np.uint32), N.CACE_OK), (np.array([5, 6], np.uint32), N.CACE_E_INVALID)):
        rc = N.lib.cace_metrics_select(N.ptr(flat), N.ptr(off), N.ptr(ncomp), N.ptr(nreq), 2, N.ptr(stat), 1,
                                       C.byref(opts), msg, len(msg))
        assert rc == want, (rc, msg.value)
    assert b"overlapping" in msg.value
