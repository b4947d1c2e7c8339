"""Synthetic workloads of the shapes BASELINE.json names.

* traces: Poisson arrivals (rate λ, reference default 10 req/s,
  experiment.hpp:22), completion/reasoning mix 70/30 (IdeHeavy,
  workload.cpp:22-25) with exact quotas and a seeded shuffle (the
  assign_labels scheme, workload.cpp:85-111), languages uniform over the
  catalog, fixed token lengths 256/50 and 512/600 (TokenParams,
  workload.hpp:34-38); optionally bursty (two-state MMPP) for config 5.
* scenario grids: config 3's 4096 reference-expressible weight vectors and
  config 4's 1,048,576 = 4096 x capacities 1..8 x 32 seeds.

The reference's own build_trace needs the full 16-model catalog
(workload.cpp:132-142); these generators are the "builder extension" the
survey calls for and use numpy's PCG64, not the reference's splitmix64.
Host-side input generation only — not part of the replay path.
"""
from __future__ import annotations

import numpy as np

from .api import ClusterConfig, ModelCatalog, P1Mode, PolicyConfig, Trace, Variant, make_scenarios
from ._native import SCENARIO_DTYPE

# The 8-CodeLLM pool of configs 1-4: {java, python, cpp, javascript} x {completion, reasoning}.
EIGHT_LANGS = [0, 1, 2, 7]


def eight_model_catalog() -> ModelCatalog:
    return ModelCatalog.build_default(languages=EIGHT_LANGS)


def mixed_trace(catalog: ModelCatalog, n: int, seed: int, rate: float = 10.0,
                completion_frac: float = 0.7, bursty: bool = False) -> Trace:
    rng = np.random.default_rng(np.random.PCG64(seed))
    if bursty:
        # two-state MMPP: high state 8x the rate, mean sojourn 50 requests
        state = np.cumsum(rng.random(n) < 1.0 / 50.0) % 2
        lam = np.where(state == 1, rate * 8.0, rate * 0.5)
        gaps = rng.exponential(1.0, n) / lam
    else:
        gaps = rng.exponential(1.0 / rate, n)
    arrival = np.cumsum(gaps)
    n_c = int(round(n * completion_frac))
    tasks = np.concatenate([np.zeros(n_c, np.int32), np.ones(n - n_c, np.int32)])
    rng.shuffle(tasks)
    # models of each class in catalog order
    by_class = [np.array([i for i, m in enumerate(catalog.models) if m.task_class == c], np.int32) for c in (0, 1)]
    model = np.empty(n, np.int32)
    for c in (0, 1):
        idx = np.nonzero(tasks == c)[0]
        pool = by_class[c]
        model[idx] = pool[rng.integers(0, len(pool), len(idx))]
    prompt = np.where(tasks == 0, 256, 512).astype(np.int32)
    output = np.where(tasks == 0, 50, 600).astype(np.int32)
    return Trace(arrival, model, prompt, output, seed=seed)


def weight_vectors_cfg3():
    """4096 = w1 in linspace(0,2,64) x w in {1,2,4,...,128} x variant in
    {cace, -p1, -p2, -p3} x P1 mode in {prose, verbatim}."""
    out = []
    for variant in (Variant.CACE_FULL, Variant.CACE_MINUS_P1, Variant.CACE_MINUS_P2, Variant.CACE_MINUS_P3):
        for p1 in (P1Mode.PROSE_CONSISTENT, P1Mode.VERBATIM):
            for w in (1, 2, 4, 8, 16, 32, 64, 128):
                for w1 in np.linspace(0.0, 2.0, 64):
                    out.append(PolicyConfig(variant=variant, w1=float(w1), window_length=w,
                                            output_token_normalizer=600, p1_mode=p1))
    return out


def scenario_grid(policies, capacities, n_traces: int, normalizer: int | None = None) -> np.ndarray:
    """Cartesian product (trace, capacity, policy) as a SCENARIO_DTYPE array,
    built vectorised (1M rows)."""
    P = len(policies)
    pol = make_scenarios([(0, p, ClusterConfig()) for p in policies])
    caps = np.asarray(capacities, np.int32)
    n = n_traces * len(caps) * P
    a = np.empty(n, SCENARIO_DTYPE)
    base = np.tile(pol, n_traces * len(caps))
    a[:] = base
    a["trace"] = np.repeat(np.arange(n_traces, dtype=np.int32), len(caps) * P)
    a["num_accelerators"] = np.tile(np.repeat(caps, P), n_traces)
    a["models_per_accelerator"] = 1
    if normalizer is not None:
        a["output_token_normalizer"] = normalizer
    return a


def config4(n_requests: int = 100_000, n_seeds: int = 32, catalog: ModelCatalog | None = None, rate: float = 10.0):
    """BASELINE config 4: cfg3 vectors x C in 1..8 x seeds -> (catalog, traces, scenarios)."""
    catalog = catalog or eight_model_catalog()
    traces = [mixed_trace(catalog, n_requests, seed=1 + s, rate=rate) for s in range(n_seeds)]
    sc = scenario_grid(weight_vectors_cfg3(), range(1, 9), n_seeds, catalog.max_expected_output_tokens())
    return catalog, traces, sc


def config3(n_requests: int = 100_000, capacity: int = 3, seed: int = 1):
    catalog = eight_model_catalog()
    traces = [mixed_trace(catalog, n_requests, seed=seed)]
    sc = scenario_grid(weight_vectors_cfg3(), [capacity], 1, catalog.max_expected_output_tokens())
    return catalog, traces, sc


def config2(n_requests: int = 10_000, seed: int = 1, capacity: int = 3):
    """Config 1/2: one 10k mixed trace, 8 CodeLLMs, budget fits 3; CACE and LRU."""
    catalog = eight_model_catalog()
    traces = [mixed_trace(catalog, n_requests, seed=seed)]
    rows = [(0, PolicyConfig(variant=v, output_token_normalizer=catalog.max_expected_output_tokens()),
             ClusterConfig(num_accelerators=capacity)) for v in (Variant.CACE_FULL, Variant.LRU)]
    return catalog, traces, make_scenarios(rows)


def config5(n_requests: int = 10_000_000, n_scenarios: int = 8192, capacity: int = 32, window: int = 1024,
            trace_seed: int = 1):
    """BASELINE config 5: 256 CodeLLMs, one bursty (MMPP) trace, long window,
    capacity 32; scenarios = w1 x {cace, -p1, -p2, -p4} x P1 mode x unload
    delay (n_scenarios of that grid).  Runs on the wide-pool lane kernel (8 lanes
    per scenario)."""
    catalog = ModelCatalog.synthetic_pool(256, seed=5)
    traces = [mixed_trace(catalog, n_requests, seed=trace_seed, rate=40.0, bursty=True)]
    rows = []
    variants = (Variant.CACE_FULL, Variant.CACE_MINUS_P1, Variant.CACE_MINUS_P2, Variant.CACE_MINUS_P4)
    per = max(1, n_scenarios // (len(variants) * 2 * 16))
    for variant in variants:
        for p1 in (P1Mode.PROSE_CONSISTENT, P1Mode.VERBATIM):
            for u in range(16):
                for w1 in np.linspace(0.0, 2.0, per):
                    rows.append((0, PolicyConfig(variant=variant, w1=float(w1), window_length=window,
                                                 output_token_normalizer=catalog.max_expected_output_tokens(),
                                                 p1_mode=p1),
                                 ClusterConfig(num_accelerators=capacity, unload_time_s=0.25 * u)))
    return catalog, traces, make_scenarios(rows[:n_scenarios])
