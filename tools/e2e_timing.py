import os, time, sys
sys.path.insert(0, os.getcwd())
os.environ["CACE_TIMING"] = "1"
import paper_2506_18796_b200 as P
from paper_2506_18796_b200 import synth
cat, tr, sc = synth.config4()
for k in range(3):
    t0 = time.perf_counter(); P.run_batch(tr, cat, sc); print("run_batch total ms", 1e3*(time.perf_counter()-t0), file=sys.stderr)
