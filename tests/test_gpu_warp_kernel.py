"""GPU: the warp-per-scenario kernel (large pools / capacities, BASELINE
config 5 regime) — forced on reference-expressible scenarios it must equal
the reference bit for bit; on 256-model pools with capacity 32-48 and a
1024-request window it must equal the port oracle."""
import numpy as np
import pytest

from tests.helpers import assert_report_equal, assert_summaries_equal, bits, ref_catalog, ref_scenario, ref_trace

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(4))
def test_forced_warp_kernel_vs_reference(ref, seed):
    import paper_2506_18796_b200 as P
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    rng = np.random.default_rng(500 + seed)
    catalog = synth.eight_model_catalog() if seed % 2 == 0 else api.ModelCatalog.build_default()
    traces = [synth.mixed_trace(catalog, int(rng.integers(50, 2500)), seed=300 * seed + k,
                                rate=float(rng.choice([0.3, 3.0, 20.0])), bursty=bool(k % 2)) for k in range(2)]
    rows = []
    for _ in range(30):
        pol = PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.choice([0.0, 0.5, 1.0, 1.7])),
                           window_length=int(rng.choice([1, 2, 5, 10, 50])), p1_mode=int(rng.integers(0, 2)),
                           output_token_normalizer=int(rng.choice([600, 50])))
        cl = ClusterConfig(num_accelerators=int(rng.integers(1, 12)), unload_time_s=float(rng.choice([0.0, 1.5])))
        rows.append((int(rng.integers(0, 2)), pol, cl))
    sc = api.make_scenarios(rows)
    summ, reps = P.run_batch(traces, catalog, sc, dump_scenarios=list(range(len(sc))), kernel=api.KERNEL_WARP)
    rcat = ref_catalog(ref, catalog)
    for k in range(len(sc)):
        want = ref.run(rcat, ref_trace(traces[int(sc[k]["trace"])]), ref_scenario(ref, sc[k]))
        assert_report_equal(reps[k], want, f"warp kernel scenario {k}")
    # the two kernels produce identical summaries
    lane = P.run_batch(traces, catalog, sc, kernel=api.KERNEL_LANE)
    assert_summaries_equal(summ, lane, "warp vs lane")


@pytest.mark.parametrize("cap,windows", [(32, (16, 256, 1024)), (48, (16, 256, 1024)),
                                         (32, (1000, 1024, 1025, 3000)), (40, (1, 1023, 2048))])
def test_config5_shape_vs_port(cap, windows):
    """256 CodeLLMs, bursty trace, capacity 32/48 (SPL 1/2); windows up to
    1024 use the first-occurrence bitmap, longer ones explicit ranks."""
    import paper_2506_18796_b200 as P
    from oracle import port
    from paper_2506_18796_b200 import api, synth
    from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig

    catalog = api.ModelCatalog.synthetic_pool(256, seed=5)
    traces = [synth.mixed_trace(catalog, 20_000, seed=k, rate=20.0, bursty=True) for k in range(2)]
    rng = np.random.default_rng(cap)
    rows = []
    for i in range(24):
        pol = PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.uniform(0, 2)),
                           window_length=int(rng.choice(windows)), p1_mode=int(rng.integers(0, 2)))
        rows.append((i % 2, pol, ClusterConfig(num_accelerators=cap)))
    sc = api.make_scenarios(rows)
    got = P.run_batch(traces, catalog, sc)
    want, _ = port.run_batch(port.Catalog(catalog), traces, sc)
    assert_summaries_equal(got, want, f"config-5 shape C={cap}")


def test_lane_and_warp_kernels_agree_at_scale():
    """Both kernels on 4096 config-4-grid scenarios x 20k requests: identical summaries."""
    import paper_2506_18796_b200 as P
    from paper_2506_18796_b200 import api, synth

    catalog = synth.eight_model_catalog()
    traces = [synth.mixed_trace(catalog, 20_000, seed=s) for s in (21, 22)]
    sc = synth.scenario_grid(synth.weight_vectors_cfg3()[::16], range(1, 9), 2, 600)
    a = P.run_batch(traces, catalog, sc, kernel=api.KERNEL_LANE)
    b = P.run_batch(traces, catalog, sc, kernel=api.KERNEL_WARP)
    assert_summaries_equal(a, b, "lane vs warp at scale")
