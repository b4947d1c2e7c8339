"""CPU: pin the plain-C port oracle against the reference, then use it for
model pools the reference cannot key (> 16 models) against the host-emulated
kernel.  (The GPU build is checked against the port in test_gpu_pools.py.)"""
import numpy as np
import pytest

from tests.helpers import assert_summaries_equal, bits, ref_catalog, ref_scenario, ref_trace


@pytest.fixture(scope="module")
def port():
    from oracle import port as PO

    if not PO.available():
        pytest.skip("port oracle not built (make -C oracle port)")
    return PO


def _random_rows(rng, n_traces, count, cmax=8):
    from paper_2506_18796_b200 import api
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    rows = []
    for _ in range(count):
        pol = PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.choice([0.0, 0.5, 1.0, 1.7])),
                           window_length=int(rng.choice([1, 2, 5, 10, 40])), p1_mode=int(rng.integers(0, 2)),
                           output_token_normalizer=int(rng.choice([600, 60])))
        cl = ClusterConfig(num_accelerators=int(rng.integers(1, cmax + 1)),
                           unload_time_s=float(rng.choice([0.0, 1.0])))
        rows.append((int(rng.integers(0, n_traces)), pol, cl))
    return api.make_scenarios(rows)


@pytest.mark.parametrize("seed", range(4))
def test_port_matches_reference(ref, port, seed):
    from paper_2506_18796_b200 import api, synth

    rng = np.random.default_rng(900 + seed)
    catalog = synth.eight_model_catalog() if seed % 2 else api.ModelCatalog.build_default()
    traces = [synth.mixed_trace(catalog, int(rng.integers(100, 2000)), seed=50 * seed + k,
                                rate=float(rng.choice([0.5, 5.0, 30.0])), bursty=bool(k % 2)) for k in range(2)]
    sc = _random_rows(rng, 2, 24)
    pc = port.Catalog(catalog)
    rcat = ref_catalog(ref, catalog)
    for row in sc:
        got = port.run(pc, traces[int(row["trace"])], row)
        want = ref.run(rcat, ref_trace(traces[int(row["trace"])]), ref_scenario(ref, row))
        s = got.summary
        assert (s["hits"], s["misses"], s["evictions"], s["loads"], s["max_resident"]) == (
            want.hits, want.misses, want.evictions, want.loads, want.max_resident)
        assert np.array_equal(bits(got.ttft), bits(want.ttft)) and np.array_equal(bits(got.e2e), bits(want.e2e))
        assert np.array_equal(got.cold, want.cold)
        assert np.array_equal(got.evict_model, want.evict_model)
        assert np.array_equal(bits(got.evict_clock), bits(want.evict_clock))
    # summaries (hash spec) agree too
    ps, _ = port.run_batch(pc, traces, sc)
    rs, _ = ref.run_batch(rcat, [ref_trace(t) for t in traces], [ref_scenario(ref, r) for r in sc])
    assert_summaries_equal(ps, rs, "port vs ref summaries")


@pytest.mark.parametrize("n_models", [20, 40, 64])
def test_emulated_kernel_large_pool_vs_port(port, n_models):
    """Pools beyond the reference's 16 (language x task) keys: kernel
    algorithm (host emulation) vs the port oracle."""
    from paper_2506_18796_b200 import api, synth
    from tests import emul

    rng = np.random.default_rng(n_models)
    catalog = api.ModelCatalog.synthetic_pool(n_models, seed=n_models)
    traces = [synth.mixed_trace(catalog, 3000, seed=k, rate=8.0, bursty=bool(k)) for k in range(2)]
    sc = _random_rows(rng, 2, 40, cmax=16)
    got, _ = emul.replay_batch(traces, catalog, sc, api.probe_log_variant())
    want, _ = port.run_batch(port.Catalog(catalog), traces, sc)
    assert_summaries_equal(got, want, f"pool {n_models}")


@pytest.mark.parametrize("n_models,cmax,window", [(100, 32, 40), (256, 32, 1024), (40, 24, 300)])
def test_emulated_wide_pool_vs_port(port, n_models, cmax, window):
    """The wide-pool lane path (pools up to 256 models, capacities up to 32;
    BASELINE config 5 shape): host emulation vs the port oracle."""
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig
    from tests import emul

    rng = np.random.default_rng(n_models + cmax)
    catalog = api.ModelCatalog.synthetic_pool(n_models, seed=n_models)
    traces = [synth.mixed_trace(catalog, 4000, seed=k, rate=40.0, bursty=True) for k in range(2)]
    rows = []
    for _ in range(24):
        pol = PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.choice([0.0, 0.5, 1.0, 1.7])),
                           window_length=int(rng.choice([1, 10, window])), p1_mode=int(rng.integers(0, 2)),
                           output_token_normalizer=catalog.max_expected_output_tokens())
        rows.append((int(rng.integers(0, 2)), pol,
                     ClusterConfig(num_accelerators=int(rng.integers(max(2, cmax // 2), cmax + 1)),
                                   unload_time_s=float(rng.choice([0.0, 0.25])))))
    sc = api.make_scenarios(rows)
    got, _ = emul.replay_batch(traces, catalog, sc, api.probe_log_variant())
    want, _ = port.run_batch(port.Catalog(catalog), traces, sc)
    assert_summaries_equal(got, want, f"wide pool {n_models}")
