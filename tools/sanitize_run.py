"""Small replay through both kernels (lane and warp, summary and dump modes),
the metrics select kernel and the policy-level kernels, for compute-sanitizer
runs (tools/gpu_sanitize.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_18796_b200 as P  # noqa: E402
from paper_2506_18796_b200 import api, synth  # noqa: E402
from paper_2506_18796_b200.api import ClusterConfig, PolicyConfig  # noqa: E402

rng = np.random.default_rng(1)
for catalog in (synth.eight_model_catalog(), api.ModelCatalog.synthetic_pool(80, seed=2)):
    traces = [synth.mixed_trace(catalog, 600, seed=k, rate=5.0, bursty=bool(k)) for k in range(2)]
    rows = []
    for _ in range(70):
        rows.append((int(rng.integers(0, 2)),
                     PolicyConfig(variant=int(rng.integers(0, 6)), w1=float(rng.uniform(0, 2)),
                                  window_length=int(rng.choice([1, 3, 10, 100, 2000])), p1_mode=int(rng.integers(0, 2))),
                     ClusterConfig(num_accelerators=int(rng.integers(1, 17)), unload_time_s=float(rng.choice([0, 1.0])))))
    sc = api.make_scenarios(rows)
    for kern in (api.KERNEL_AUTO, api.KERNEL_WARP):
        a = P.run_batch(traces, catalog, sc, kernel=kern)
        b, _ = P.run_batch(traces, catalog, sc, kernel=kern, dump_scenarios=[0, 5, 9])
        assert (a["outcome_hash"] == b["outcome_hash"]).all()
    m = P.run_metrics(traces, catalog, sc, raise_on_error=False)
    assert (m["status"] == 0).all()
# RunMetrics on a trace long enough for the select's speculative digit and
# in-place compaction (> 16384 completion samples), chunked over the ring
# buffers, with the speculation both taken and forced to miss
catalog = synth.eight_model_catalog()
traces = [synth.mixed_trace(catalog, 25_000, seed=5)]
rows = [(0, PolicyConfig(variant=v, window_length=10), ClusterConfig(num_accelerators=c))
        for v in (0, 1) for c in (1, 3, 8)]
sc = api.make_scenarios(rows)
os.environ["CACE_METRICS_BUDGET_MB"] = "1"
ref_m = None
for mode in ("1", "2"):
    os.environ["CACE_METRICS_SPEC"] = mode
    m = P.run_metrics(traces, catalog, sc)
    ref_m = m if ref_m is None else ref_m
    assert m.tobytes() == ref_m.tobytes()
print("sanitize run ok")
