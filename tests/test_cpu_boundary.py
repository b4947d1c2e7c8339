"""CPU: the C-ABI library, the host-side glibc-log restatement, workload builders
and the multi-process shard/gather path (gloo, world_size 2)."""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cace_gpu.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(cace_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2506_18796_b200 import _native as N

    decl = _declared_functions()
    assert len(decl) >= 17, decl
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cace_[a-z_0-9]+)", out))
    missing = [f for f in decl if f not in exported]
    assert not missing, missing
    assert set(N.EXPORTED) <= exported


def test_library_is_sm100a():
    from paper_2506_18796_b200 import _native as N

    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    """No CUDA device here: replay must refuse (there is no CPU fallback)."""
    import paper_2506_18796_b200 as P
    from paper_2506_18796_b200 import synth

    if P.device_count() > 0:
        pytest.skip("a GPU is visible")
    cat, traces, sc = synth.config2(n_requests=100)
    with pytest.raises(P.SimError, match="no CUDA device"):
        P.run_batch(traces, cat, sc)


def test_host_log_restatement_matches_this_libm(ref):
    from paper_2506_18796_b200 import api

    rng = np.random.default_rng(3)
    x = np.concatenate([np.exp(rng.uniform(0, 25, 1_000_000)), 1 + rng.uniform(0, 0.0647, 300_000),
                        np.arange(1, 100_001, dtype=np.float64)])
    v = api.probe_log_variant()
    assert v in (0, 1)
    got = api.host_log(x, v)
    assert np.array_equal(got.view(np.uint64), ref.libm_log(x).view(np.uint64))


def test_host_log_sse2_variant_under_non_fma_libm(ref):
    """With glibc's FMA ifunc disabled, libm selects the SSE2 log; the probe and
    the SSE2 restatement must follow it (policy.cpp:51 bit hazard)."""
    code = ("import numpy as np; from paper_2506_18796_b200 import api; from oracle import ref;"
            "x=np.exp(np.random.default_rng(1).uniform(0,20,400000));"
            "print(api.probe_log_variant(), int((api.host_log(x,1).view(np.uint64)!=ref.libm_log(x).view(np.uint64)).sum()))")
    env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA", PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split() == ["1", "0"]


def test_default_catalog_matches_reference(ref):
    """build_default restated (catalog.cpp:76-99) equals the reference's catalog."""
    import json

    from __graft_entry__ import _catalog_json
    from paper_2506_18796_b200 import api

    mine = json.loads(_catalog_json(api.ModelCatalog.build_default()))["models"]
    theirs = ref.Catalog.default().models()
    assert mine == theirs


def test_workload_shapes():
    from paper_2506_18796_b200 import synth

    assert len(synth.weight_vectors_cfg3()) == 4096
    cat = synth.eight_model_catalog()
    assert [m.model_id for m in cat.models][:2] == ["java-completion", "java-reasoning"]
    t = synth.mixed_trace(cat, 10_000, seed=1)
    assert np.all(np.diff(t.arrival_time_s) >= 0)
    reasoning = np.array([cat.models[m].task_class for m in t.model])
    assert (reasoning == 0).sum() == 7000
    sc = synth.scenario_grid(synth.weight_vectors_cfg3(), range(1, 9), 2, 600)
    assert len(sc) == 4096 * 8 * 2
    assert set(np.unique(sc["num_accelerators"])) == set(range(1, 9))


def test_shards_cover_and_balance():
    """cace_shard_scenarios: every scenario in exactly one shard, every
    (capacity, trace) group split evenly in whole warps."""
    from paper_2506_18796_b200 import shard, synth

    sc = synth.scenario_grid(synth.weight_vectors_cfg3(), range(1, 9), 4, 600)
    for world in (1, 2, 4, 8):
        parts = shard.shard_indices(sc, 8, world)
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(len(sc)))
        for c in range(1, 9):
            for t in range(4):
                g = [int(((sc["num_accelerators"][p] == c) & (sc["trace"][p] == t)).sum()) for p in parts]
                assert max(g) - min(g) <= 32 and sum(g) == 4096, (world, c, t, g)
    # small groups rotate over the shards
    small = synth.scenario_grid(synth.weight_vectors_cfg3()[:40], range(1, 9), 4, 600)
    parts = shard.shard_indices(small, 8, 8)
    sizes = [len(p) for p in parts]
    assert sum(sizes) == len(small) and max(sizes) - min(sizes) <= 64, sizes


_GLOO_WORKER = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
from paper_2506_18796_b200 import shard, synth
from paper_2506_18796_b200._native import SUMMARY_DTYPE
from oracle import ref
from tests.helpers import ref_catalog, ref_scenario, ref_trace
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
cat = synth.eight_model_catalog()
traces = [synth.mixed_trace(cat, 1500, seed=s) for s in (1, 2)]
pols = synth.weight_vectors_cfg3()[::256]
sc = synth.scenario_grid(pols, [2, 3], 2, 600)
parts = shard.shard_indices(sc, len(cat), world)
mine = sc[parts[rank]]
rcat = ref_catalog(ref, cat)
summ, _ = ref.run_batch(rcat, [ref_trace(t) for t in traces], [ref_scenario(ref, s) for s in mine], threads=1)
full = shard.gather_summaries(torch.from_numpy(summ.view(np.uint8).copy()), parts)
if rank == 0:
    want, _ = ref.run_batch(rcat, [ref_trace(t) for t in traces], [ref_scenario(ref, s) for s in sc], threads=2)
    assert full.tobytes() == want.tobytes(), "gathered summaries differ"
    print("GATHER_OK", len(full))
dist.destroy_process_group()
"""


def test_multiprocess_shard_gather_gloo(ref, tmp_path):
    """world_size-2 gloo run of the N>1 path: shard, replay per rank, all-gather
    summaries; rank 0's gathered sweep equals the single-process sweep."""
    script = tmp_path / "worker.py"
    script.write_text(_GLOO_WORKER)
    env = dict(os.environ, ROOT=ROOT, PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", str(script)]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "GATHER_OK" in out.stdout


def test_cli_backend_swap_patch_type_checks():
    """integration/cacesim_main_gpu.patch (the simulate / compare / ablate
    backend swap, cacesim_main.cpp:194,330) applies to the reference CLI and
    type-checks against cacesim_gpu.hpp (needs /root/reference: skipped
    elsewhere)."""
    import os
    import subprocess

    if not os.path.isdir("/root/reference/proj/tools"):
        pytest.skip("reference sources not present")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(["make", "-s", "-C", os.path.join(root, "integration"), "cli-check"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
