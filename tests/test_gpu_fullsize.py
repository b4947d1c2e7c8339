"""GPU, BASELINE config 4 at full size (1,048,576 scenarios x 100k requests):
size-independent invariants on every summary, plus a sample checked
bit-exact against the reference run() (oracle/_ref, all host threads): a
1024-scenario sample stratified over capacity x variant x P1 mode x window."""
import numpy as np
import pytest

from tests.helpers import SUMMARY_FLOAT_KEYS, SUMMARY_KEYS

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2506_18796_b200")
from paper_2506_18796_b200 import synth  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if P.device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU tests must run on a B200 (no CPU fallback)")


def test_config4_full_size_invariants_and_sample(ref):
    catalog, traces, sc = synth.config4()
    summ = P.run_batch(traces, catalog, sc)
    n = len(traces[0])
    assert (summ["status"] == 0).all()
    # conservation (test_engine.cpp:154-183, acceptance criterion 6)
    assert (summ["hits"] + summ["misses"] == n).all()
    assert (summ["loads"] == summ["misses"]).all()
    cap = sc["num_accelerators"] * sc["models_per_accelerator"]
    distinct = np.array([len(np.unique(t.model)) for t in traces])[sc["trace"]]
    assert (summ["max_resident"] == np.minimum(cap, distinct)).all()
    assert (summ["evictions"] == summ["loads"] - summ["max_resident"]).all()
    ncomp = np.array([(np.array([catalog.models[m].task_class for m in t.model]) == 0).sum() for t in traces])
    assert (summ["n_completion"] == ncomp[sc["trace"]]).all()
    assert (summ["n_completion"] + summ["n_reasoning"] == n).all()
    # capacity >= pool never evicts (test_engine.cpp:102-121)
    assert (summ["evictions"][cap >= len(catalog)] == 0).all()
    # a stratified 1024-scenario sample (every capacity x variant x P1 mode x
    # window stratum) bit-exact against the reference simulator, full length
    import os

    from bench import cpu_run, stratified_sample

    idx = stratified_sample(sc, 1024, 2026)
    want, _, kind = cpu_run(catalog, traces, sc, idx, os.cpu_count() or 1)
    assert kind == "reference"
    got = summ[idx]
    for k in SUMMARY_KEYS:
        assert (got[k] == want[k]).all(), k
    for k in SUMMARY_FLOAT_KEYS:
        assert (got[k].view(np.uint64) == want[k].view(np.uint64)).all(), k
