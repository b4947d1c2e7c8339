"""Shared test helpers: convert between the product's scenario rows and the
reference oracle's, and compare reports bit for bit."""
import numpy as np

from __graft_entry__ import _catalog_json  # noqa: F401  (re-exported)


def ref_catalog(ref, catalog):
    return ref.Catalog.from_json(_catalog_json(catalog))


def ref_trace(t):
    return dict(arrival=t.arrival_time_s, model=t.model, prompt=t.prompt_tokens, output=t.output_tokens)


def ref_scenario(ref, s):
    return ref.scenario(variant=int(s["variant"]), p1_mode=int(s["p1_mode"]),
                        window_length=int(s["window_length"]),
                        output_token_normalizer=int(s["output_token_normalizer"]),
                        num_accelerators=int(s["num_accelerators"]),
                        models_per_accelerator=int(s["models_per_accelerator"]),
                        w1=float(s["w1"]), unload_time_s=float(s["unload_time_s"]), trace=int(s["trace"]))


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def assert_report_equal(got, want, ctx=""):
    """Bit-exact comparison of a GPU SimulationReport with a reference RefReport."""
    assert (got.counters.hits, got.counters.misses, got.counters.evictions, got.loads, got.max_resident) == (
        want.hits, want.misses, want.evictions, want.loads, want.max_resident), ctx
    assert bits([got.counters.load_overhead_s])[0] == bits([want.load_overhead_s])[0], ctx
    assert np.array_equal(got.cold_start, want.cold), ctx
    for name, a, b in (("ttft", got.ttft_s, want.ttft), ("e2e", got.e2e_s, want.e2e),
                       ("queue_wait", got.queue_wait_s, want.queue_wait), ("load_wait", got.load_wait_s, want.load_wait),
                       ("prefill", got.prefill_s, want.prefill), ("decode", got.decode_s, want.decode)):
        bad = np.nonzero(bits(a) != bits(b))[0]
        assert len(bad) == 0, f"{ctx} {name} differs at {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}"
    assert np.array_equal(got.evicted_model, want.evict_model), f"{ctx} eviction sequence"
    assert np.array_equal(bits(got.eviction_clock), bits(want.evict_clock)), f"{ctx} eviction clocks"


SUMMARY_KEYS = ("hits", "misses", "evictions", "loads", "max_resident", "status", "n_completion", "n_reasoning",
                "eviction_hash", "outcome_hash")
SUMMARY_FLOAT_KEYS = ("load_overhead_s", "sum_ttft_completion", "sum_e2e_reasoning", "max_ttft_completion",
                      "max_e2e_reasoning")


def assert_summaries_equal(got, want, ctx=""):
    for k in SUMMARY_KEYS:
        bad = np.nonzero(got[k] != want[k])[0]
        assert len(bad) == 0, f"{ctx} summary {k} differs at scenarios {bad[:8]}"
    for k in SUMMARY_FLOAT_KEYS:
        bad = np.nonzero(bits(got[k]) != bits(want[k]))[0]
        assert len(bad) == 0, f"{ctx} summary {k} differs at scenarios {bad[:8]}"
