"""Multi-GPU paths on the engine (not the oracle).

* cace_replay_batch_multi (one process, a host thread + stream per device,
  summaries gathered to devices[0]): the same sweep on [0] and on [0, 0]
  (a repeated device takes the peer-copy gather; the NCCL gather needs
  distinct devices) equals the single-device replay bit for bit.
* one process per rank (the bench / torchrun layout): two gloo ranks sharing
  GPU 0 each replay their shard with the engine; the all-gathered sweep
  equals one single-rank replay.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.helpers import assert_summaries_equal, ref_catalog, ref_scenario, ref_trace

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2506_18796_b200")
from paper_2506_18796_b200 import synth  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if P.device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU tests must run on a B200 (no CPU fallback)")


def _sweep():
    catalog = synth.eight_model_catalog()
    traces = [synth.mixed_trace(catalog, 5000, seed=s) for s in (21, 22, 23)]
    sc = synth.scenario_grid(synth.weight_vectors_cfg3()[::16], range(1, 9), 3, 600)
    return catalog, traces, sc


def test_multi_device_entry_matches_single_device(ref):
    catalog, traces, sc = _sweep()
    one = P.run_batch(traces, catalog, sc)
    got1, k1 = P.run_batch(traces, catalog, sc, devices=[0], return_gather_kind=True)
    got2, k2 = P.run_batch(traces, catalog, sc, devices=[0, 0], return_gather_kind=True)
    assert (k1, k2) == (0, 2)
    assert got1.tobytes() == one.tobytes()
    assert got2.tobytes() == one.tobytes()
    # and the sweep is the reference's (a sample: the full sweep is 6144 scenarios)
    idx = np.arange(0, len(sc), 97)
    want, _ = ref.run_batch(ref_catalog(ref, catalog), [ref_trace(t) for t in traces],
                            [ref_scenario(ref, s) for s in sc[idx]])
    assert_summaries_equal(got2[idx], want, "multi-device")


def test_multi_device_errors_surface(ref):
    catalog, traces, sc = _sweep()
    bad = sc[:64].copy()
    bad["window_length"][40] = 0  # run: window_length must be >= 1 (engine.cpp:79)
    with pytest.raises(P.SimError, match="window_length must be >= 1"):
        P.run_batch(traces, catalog, bad, devices=[0, 0])
    with pytest.raises(P.SimError):
        P.run_batch(traces, catalog, sc[:64], devices=[0, 99])


@pytest.mark.parametrize("devices", [None, [0, 0]])
def test_first_failing_scenario_in_caller_order_is_reported(devices):
    """With several invalid scenarios the error is the first one in the
    caller's order (the reference's run_grid loop raises at the first), on the
    single- and the multi-device entry."""
    catalog, traces, sc = _sweep()
    kw = {} if devices is None else {"devices": devices}
    for first, second, msg in (("unload_time_s", "window_length", "unload_time_s must be in"),
                               ("window_length", "unload_time_s", "window_length must be >= 1")):
        bad = sc[:256].copy()
        bad[first][37] = -1.0 if first == "unload_time_s" else 0
        bad[second][200] = -1.0 if second == "unload_time_s" else 0
        with pytest.raises(P.SimError, match=msg):
            P.run_batch(traces, catalog, bad, **kw)


_RANK_WORKER = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
import paper_2506_18796_b200 as P
from paper_2506_18796_b200 import shard, synth
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
cat = synth.eight_model_catalog()
traces = [synth.mixed_trace(cat, 4000, seed=s) for s in (31, 32)]
sc = synth.scenario_grid(synth.weight_vectors_cfg3()[::8], range(1, 9), 2, 600)
parts = shard.shard_indices(sc, len(cat), world)
mine = P.run_batch(traces, cat, sc[parts[rank]], device=0)
full = shard.gather_summaries(torch.from_numpy(mine.view(np.uint8).copy()), parts)
if rank == 0:
    whole = P.run_batch(traces, cat, sc, device=0)
    assert full.tobytes() == whole.tobytes(), "gathered sweep differs from the single-rank replay"
    print("RANKS_OK", len(full), [len(p) for p in parts])
dist.destroy_process_group()
"""


def test_two_ranks_replay_shards_on_the_engine(tmp_path):
    script = tmp_path / "ranks.py"
    script.write_text(_RANK_WORKER)
    env = dict(os.environ, ROOT=ROOT, PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29541", str(script)]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "RANKS_OK" in out.stdout
