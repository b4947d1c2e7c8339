"""CPU: the replay kernel's device code (host-emulated, tests/emul) vs the reference.

The same request-synchronous algorithm that runs on the B200 is compiled as
host C++ and checked bit-exact against the compiled reference simulator on
many random scenarios.  This lets kernel-algorithm changes be validated on the
CPU box before a GPU run; the GPU tests (test_gpu_parity.py) then check the
actual sm_100a build the same way.
"""
import numpy as np
import pytest

from tests.helpers import assert_summaries_equal, bits, ref_catalog, ref_scenario, ref_trace


@pytest.fixture(scope="module")
def emul():
    from tests import emul as E

    E.build()
    return E


def _logv():
    from paper_2506_18796_b200 import api

    return api.probe_log_variant()


def _check_full(ref, emul, catalog, traces, sc, rolled_exact=True):
    got, d = emul.replay_batch(traces, catalog, sc, _logv(), dump=True, rolled_exact=rolled_exact)
    rcat = ref_catalog(ref, catalog)
    for k in range(len(sc)):
        want = ref.run(rcat, ref_trace(traces[int(sc[k]["trace"])]), ref_scenario(ref, sc[k]))
        g = got[k]
        ctx = f"scenario {k} {sc[k]}"
        assert g["status"] == 0, ctx
        assert (g["hits"], g["misses"], g["evictions"], g["loads"], g["max_resident"]) == (
            want.hits, want.misses, want.evictions, want.loads, want.max_resident), ctx
        assert bits([g["load_overhead_s"]])[0] == bits([want.load_overhead_s])[0], ctx
        o, n = int(d["off"][k]), int(d["sizes"][k])
        for name, arr, ref_arr in (("ttft", d["ttft"], want.ttft), ("e2e", d["e2e"], want.e2e),
                                   ("queue_wait", d["qw"], want.queue_wait), ("load_wait", d["lw"], want.load_wait)):
            bad = np.nonzero(bits(arr[o:o + n]) != bits(ref_arr))[0]
            assert len(bad) == 0, f"{ctx} {name} differs at {bad[:5]}"
        assert np.array_equal(d["cold"][o:o + n].astype(bool), want.cold), ctx
        ne = int(d["ne"][k])
        cap = d["cap"]
        assert ne == want.evictions, ctx
        assert np.array_equal(d["em"][k * cap:k * cap + ne], want.evict_model), f"{ctx} eviction sequence"
        assert np.array_equal(bits(d["ec"][k * cap:k * cap + ne]), bits(want.evict_clock)), f"{ctx} clocks"


@pytest.mark.parametrize("rolled", [True, False], ids=["rolled_exact", "unrolled_exact"])
@pytest.mark.parametrize("seed", range(8))
def test_emulated_kernel_random_scenarios(ref, emul, seed, rolled):
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    rng = np.random.default_rng(300 + seed)
    catalog = synth.eight_model_catalog() if seed % 2 == 0 else api.ModelCatalog.build_default()
    traces = [synth.mixed_trace(catalog, int(rng.integers(50, 2500)), seed=7000 * seed + k,
                                rate=float(rng.choice([0.2, 1.0, 3.0, 10.0, 40.0])), bursty=bool(k % 2))
              for k in range(3)]
    rows = []
    for _ in range(30):
        pol = PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.choice([0.0, 0.25, 0.5, 1.0, 1.7])),
                           window_length=int(rng.choice([1, 2, 3, 5, 10, 16, 50, 200])),
                           output_token_normalizer=int(rng.choice([600, 300, 50])), p1_mode=int(rng.integers(0, 2)))
        cl = ClusterConfig(num_accelerators=int(rng.integers(1, 11)),
                           unload_time_s=float(rng.choice([0.0, 0.0, 0.5, 2.0])))
        rows.append((int(rng.integers(0, 3)), pol, cl))
    _check_full(ref, emul, catalog, traces, api.make_scenarios(rows), rolled_exact=rolled)


def test_emulated_kernel_ties_and_unsorted(ref, emul):
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    catalog = synth.eight_model_catalog()
    rng = np.random.default_rng(5)
    n = 600
    t1 = api.Trace(np.round(rng.uniform(0, 60, n), 1), rng.integers(0, 8, n), np.full(n, 256), np.full(n, 50))
    arr = np.repeat(np.arange(n // 3, dtype=np.float64) * 0.5, 3)
    t2 = api.Trace(arr, np.tile(np.array([0, 2, 4, 6, 1, 3], np.int32), n // 6), np.full(n, 256), np.full(n, 64))
    rows = [(t, PolicyConfig(variant=v, window_length=w), ClusterConfig(num_accelerators=c))
            for t in (0, 1) for v in range(6) for w in (1, 3) for c in (1, 2, 3, 4, 6)]
    _check_full(ref, emul, catalog, [t1, t2], api.make_scenarios(rows))


def test_emulated_kernel_reference_build_trace(ref, emul):
    from paper_2506_18796_b200 import api
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    rcat = ref.Catalog.default()
    catalog = api.ModelCatalog.build_default()
    traces = []
    for pat, rate, seed in ((0, 15.0, 1), (1, 15.0, 2), (2, 4.0, 3)):
        t = ref.build_trace(rcat, pat, rate, 30.0, seed)
        traces.append(api.Trace(t["arrival"], t["model"], t["prompt"], t["output"]))
    rows = [(ti, PolicyConfig(variant=v, w1=w1, window_length=w), ClusterConfig(num_accelerators=c))
            for ti in range(3) for v in range(6) for (w1, w, c) in ((0.5, 10, 4), (1.0, 2, 3))]
    _check_full(ref, emul, catalog, traces, api.make_scenarios(rows))


def test_emulated_kernel_summaries_cfg_grid(ref, emul):
    """Summary hashes over a slice of the config-3/4 grid, 10k requests."""
    from paper_2506_18796_b200 import synth

    catalog = synth.eight_model_catalog()
    traces = [synth.mixed_trace(catalog, 10_000, seed=s) for s in (1, 2)]
    sc = synth.scenario_grid(synth.weight_vectors_cfg3()[::64], [3, 5, 7], 2, 600)
    got, _ = emul.replay_batch(traces, catalog, sc, _logv())
    want, _ = ref.run_batch(ref_catalog(ref, catalog), [ref_trace(t) for t in traces],
                            [ref_scenario(ref, s) for s in sc])
    assert_summaries_equal(got, want, "emulated grid")


@pytest.mark.parametrize("seed", range(3))
def test_emulated_wide_path_small_pools(ref, emul, seed):
    """The wide-pool code path (runtime capacity, fp32 p2 + p4 formed on the
    fly, exact p4 recomputed) forced on reference-expressible scenarios: full
    per-request reports bit-exact against the reference."""
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    rng = np.random.default_rng(4000 + seed)
    catalog = synth.eight_model_catalog() if seed % 2 == 0 else api.ModelCatalog.build_default()
    traces = [synth.mixed_trace(catalog, int(rng.integers(500, 3000)), seed=40 * seed + k,
                                rate=float(rng.choice([1.0, 10.0, 40.0])), bursty=bool(k % 2)) for k in range(2)]
    rows = []
    for _ in range(30):
        pol = PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.choice([0.0, 0.5, 1.0, 1.7])),
                           window_length=int(rng.choice([1, 3, 10, 50])), p1_mode=int(rng.integers(0, 2)),
                           output_token_normalizer=int(rng.choice([600, 50])))
        rows.append((int(rng.integers(0, 2)), pol,
                     ClusterConfig(num_accelerators=int(rng.integers(1, 16)),
                                   unload_time_s=float(rng.choice([0.0, 0.5])))))
    sc = api.make_scenarios(rows)
    got, d = emul.replay_batch(traces, catalog, sc, _logv(), dump=True, wide=True)
    rcat = ref_catalog(ref, catalog)
    want, _ = ref.run_batch(rcat, [ref_trace(t) for t in traces], [ref_scenario(ref, s) for s in sc])
    assert_summaries_equal(got, want, "wide path")


@pytest.mark.parametrize("rolled", [True, False])
def test_emulated_mixed_capacity_path(ref, emul, rolled):
    """The runtime-capacity one-lane path of the mixed-capacity launch
    (shallow sweeps: one kernel for every capacity <= 8) on the config-4 grid
    shape and random scenarios, both exact-fallback variants, bit-exact
    against the reference."""
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    catalog = synth.eight_model_catalog()
    traces = [synth.mixed_trace(catalog, 6000, seed=s) for s in (3, 4)]
    sc = synth.scenario_grid(synth.weight_vectors_cfg3()[::128], range(1, 9), 2, 600)
    rng = np.random.default_rng(77)
    rows = [(int(rng.integers(0, 2)),
             PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.choice([0.0, 0.7, 1.7])),
                          window_length=int(rng.choice([1, 4, 40])), p1_mode=int(rng.integers(0, 2))),
             ClusterConfig(num_accelerators=int(rng.integers(1, 5)), models_per_accelerator=int(rng.integers(1, 3)),
                           unload_time_s=float(rng.choice([0.0, 0.5]))))
            for _ in range(24)]
    sc = np.concatenate([sc, api.make_scenarios(rows)])
    got, _ = emul.replay_batch(traces, catalog, sc, _logv(), rolled_exact=rolled, mixed=True)
    want, _ = ref.run_batch(ref_catalog(ref, catalog), [ref_trace(t) for t in traces],
                            [ref_scenario(ref, s) for s in sc])
    assert_summaries_equal(got, want, "mixed-capacity path")
