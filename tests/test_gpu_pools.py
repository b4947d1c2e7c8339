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
