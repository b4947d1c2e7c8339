"""GPU: model pools beyond the reference's 16 keys (up to the lane kernel's
64) and capacities up to 16, checked against the port oracle (itself pinned
bit-exact to the reference in test_cpu_port.py)."""
import numpy as np
import pytest

from tests.helpers import assert_summaries_equal, bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_models", [24, 48, 64])
def test_large_pool_summaries_vs_port(n_models):
    import paper_2506_18796_b200 as P
    from oracle import port
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    rng = np.random.default_rng(77 + n_models)
    catalog = api.ModelCatalog.synthetic_pool(n_models, seed=n_models)
    traces = [synth.mixed_trace(catalog, 20_000, seed=k, rate=8.0, bursty=bool(k)) for k in range(2)]
    rows = []
    for _ in range(96):
        pol = PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.uniform(0, 2)),
                           window_length=int(rng.choice([1, 4, 16, 64, 256])), p1_mode=int(rng.integers(0, 2)))
        rows.append((int(rng.integers(0, 2)), pol, ClusterConfig(num_accelerators=int(rng.integers(1, 17)))))
    sc = api.make_scenarios(rows)
    got = P.run_batch(traces, catalog, sc)
    want, _ = port.run_batch(port.Catalog(catalog), traces, sc)
    assert_summaries_equal(got, want, f"pool {n_models}")


def test_large_pool_full_report_vs_port():
    import paper_2506_18796_b200 as P
    from oracle import port
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    catalog = api.ModelCatalog.synthetic_pool(40, seed=3)
    t = synth.mixed_trace(catalog, 4000, seed=9, rate=6.0)
    for c, w, v in ((12, 32, 1), (16, 200, 2), (7, 5, 0)):
        pol = PolicyConfig(variant=v, window_length=w, w1=0.7)
        rep = P.run(t, catalog, ClusterConfig(num_accelerators=c), pol)
        row = api.make_scenarios([(0, pol, ClusterConfig(num_accelerators=c))])[0]
        want = port.run(port.Catalog(catalog), t, row)
        assert np.array_equal(bits(rep.ttft_s), bits(want.ttft)) and np.array_equal(bits(rep.e2e_s), bits(want.e2e))
        assert np.array_equal(rep.evicted_model, want.evict_model)


def test_capacity_beyond_the_pool_is_accepted(ref):
    """The reference accepts any num_accelerators x models_per_accelerator
    (engine.cpp:83-84); with capacity >= the pool nothing is ever evicted, so
    the engine clamps it to the pool size: capacities up to 3000 replay
    bit-exact against the reference (16 models) and the port (48 models,
    clamped to 48 slots: the warp kernel).  Pools of more than 64 models with a
    capacity above 64 are rejected (CACE_E_INVALID)."""
    import paper_2506_18796_b200 as P
    from oracle import port
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig
    from tests.helpers import ref_catalog, ref_scenario, ref_trace

    cat16 = api.ModelCatalog.build_default()
    traces = [synth.mixed_trace(cat16, 3000, seed=41)]
    rows = [(0, PolicyConfig(variant=v, window_length=8), ClusterConfig(num_accelerators=a, models_per_accelerator=mpa))
            for v in (0, 1) for a, mpa in ((16, 1), (17, 1), (65, 1), (100, 3), (1000, 3))]
    sc = api.make_scenarios(rows)
    got = P.run_batch(traces, cat16, sc)
    assert (got["evictions"] == 0).all()
    want, _ = ref.run_batch(ref_catalog(ref, cat16), [ref_trace(t) for t in traces], [ref_scenario(ref, r) for r in sc])
    assert_summaries_equal(got, want, "capacity >= pool (16 models)")
    cat48 = api.ModelCatalog.synthetic_pool(48, seed=8)
    t48 = [synth.mixed_trace(cat48, 3000, seed=42, rate=5.0)]
    rows = [(0, PolicyConfig(variant=1, window_length=64), ClusterConfig(num_accelerators=a)) for a in (48, 49, 200, 3000)]
    sc = api.make_scenarios(rows)
    got = P.run_batch(t48, cat48, sc)
    want, _ = port.run_batch(port.Catalog(cat48), t48, sc)
    assert_summaries_equal(got, want, "capacity >= pool (48 models)")
    cat80 = api.ModelCatalog.synthetic_pool(80, seed=8)
    t80 = [synth.mixed_trace(cat80, 500, seed=43)]
    with pytest.raises(P.SimError):
        P.run_batch(t80, cat80, api.make_scenarios([(0, PolicyConfig(), ClusterConfig(num_accelerators=80))]))
