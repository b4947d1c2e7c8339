"""Time cace_run_metrics_batch (on-device RunMetrics) on BASELINE config 4."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_18796_b200 as P  # noqa: E402
from paper_2506_18796_b200 import synth  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cat, tr, sc = synth.config4(n_seeds=seeds)
for k in range(2):
    t0 = time.perf_counter()
    m = P.run_metrics(tr, cat, sc)
    dt = time.perf_counter() - t0
    print(f"run_metrics: {len(sc)} scenarios x {len(tr[0])} requests in {dt:.3f} s "
          f"({len(sc) * len(tr[0]) / dt:.3e} scenario-requests/s)", flush=True)
print("example", m[0])
