"""Device cost of the DUMP replay instantiation vs the summary one on config 4
(run_batch with one dumped scenario runs every segment through DUMP)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_18796_b200 as P  # noqa: E402
from paper_2506_18796_b200 import synth  # noqa: E402

cat, tr, sc = synth.config4(n_seeds=int(sys.argv[1]) if len(sys.argv) > 1 else 32)
for name, kw in (("summary", {}), ("dump1", {"dump_scenarios": [0]}), ("summary", {}), ("dump1", {"dump_scenarios": [0]})):
    t0 = time.perf_counter()
    P.run_batch(tr, cat, sc, **kw)
    print(f"{name}: {time.perf_counter() - t0:.3f} s", flush=True)
