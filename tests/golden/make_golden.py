#!/usr/bin/env python3
"""Generate tests/golden/*.npz by running the REFERENCE simulator (oracle/_ref).

The reference ships no golden per-request vectors, so these
fixtures are produced by the reference itself, compiled out of tree from
/root/reference/proj/src (oracle/Makefile), on:
  * traces from the reference's own generator build_trace (workload.cpp:127-179)
    over its 16-model default catalog, all three patterns, several seeds;
  * the hand-built traces of test_engine.cpp (cold start, warm hit, capacity-
    sufficient, LRU thrash, unload delay);
  * a synthetic 8-CodeLLM mixed trace (BASELINE config 1/2 shape, 2,000 req).
For each (trace, scenario): counters, per-request cold/queue_wait/load_wait/
prefill/decode/ttft/e2e (request order) and the eviction sequence.

Run in the source container (needs oracle/_ref):  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def scen_rows():
    rows = []
    for v in range(6):
        rows.append(dict(variant=v, p1_mode=0, window_length=10, output_token_normalizer=600,
                         num_accelerators=4, models_per_accelerator=1, w1=1.0, unload_time_s=0.0))
        rows.append(dict(variant=v, p1_mode=1, window_length=2, output_token_normalizer=600,
                         num_accelerators=3, models_per_accelerator=1, w1=0.5, unload_time_s=0.0))
        rows.append(dict(variant=v, p1_mode=0, window_length=5, output_token_normalizer=600,
                         num_accelerators=2, models_per_accelerator=1, w1=1.5, unload_time_s=1.25))
    return rows


def hand_traces(cat_models):
    idx = {m["model_id"]: i for i, m in enumerate(cat_models)}
    j, p, g, r = idx["java-completion"], idx["python-completion"], idx["go-completion"], idx["rust-completion"]
    out = {}
    out["cold_start"] = ([1.0], [j])
    out["warm_hit"] = ([0.0, 20.0], [j, j])
    out["capacity_sufficient"] = ([i * 3.0 for i in range(40)], [[j, p, g, r][i % 4] for i in range(40)])
    out["lru_thrash"] = ([i * 0.01 for i in range(40)], [[j, p, g, r][i % 4] for i in range(40)])
    out["unload_delay"] = ([0.0, 0.1], [j, p])
    return out


def main():
    cat = ref.Catalog.default()
    models = cat.models()
    traces = {}
    for pat in range(3):
        for seed in (1, 2):
            t = ref.build_trace(cat, pat, 10.0 if pat != 2 else 4.0, 20.0, seed)
            traces[f"build_trace_p{pat}_s{seed}"] = t
    for name, (arr, mdl) in hand_traces(models).items():
        n = len(arr)
        traces[name] = dict(arrival=np.array(arr, np.float64), model=np.array(mdl, np.int32),
                            prompt=np.full(n, 256, np.int32), output=np.full(n, 50, np.int32))
    rows = scen_rows()
    payload = {"scenario_fields": np.array(list(rows[0].keys())),
               "scenarios": np.array([[r[k] for k in rows[0]] for r in rows], np.float64)}
    for tname, t in traces.items():
        for k in ("arrival", "model", "prompt", "output"):
            payload[f"{tname}/trace/{k}"] = t[k]
        for si, r in enumerate(rows):
            rep = ref.run(cat, t, ref.scenario(**r))
            key = f"{tname}/s{si}"
            payload[key + "/counters"] = np.array([rep.hits, rep.misses, rep.evictions, rep.loads, rep.max_resident],
                                                  np.int64)
            payload[key + "/load_overhead_s"] = np.array([rep.load_overhead_s])
            payload[key + "/cold"] = rep.cold.astype(np.uint8)
            for f in ("queue_wait", "load_wait", "prefill", "decode", "ttft", "e2e"):
                payload[key + "/" + f] = getattr(rep, f)
            payload[key + "/evict_model"] = rep.evict_model
            payload[key + "/evict_clock"] = rep.evict_clock
    payload["catalog_json"] = np.array(cat.to_json())
    np.savez_compressed(os.path.join(OUT, "reference_runs.npz"), **payload)
    print("wrote", os.path.join(OUT, "reference_runs.npz"), len(traces), "traces x", len(rows), "scenarios")


if __name__ == "__main__":
    main()
