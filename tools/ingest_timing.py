"""Time JSONL trace ingestion: native parse (cace_trace_parse_jsonl, all host
threads) vs the reference's parse_trace (oracle/_ref), same text."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref  # noqa: E402
from paper_2506_18796_b200 import api  # noqa: E402

rate, dur = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0, float(sys.argv[2]) if len(sys.argv) > 2 else 10000.0
text = ref.serialize_built_trace(1, rate, dur, 7, 1)
cat = api.ModelCatalog.build_default()
t0 = time.perf_counter()
tr, hdr, _ = api.parse_trace(text, cat)
t1 = time.perf_counter()
want = ref.parse_trace(text)
t2 = time.perf_counter()
ok = (tr.arrival_time_s == want["arrival"]).all()
print(f"{len(tr)} requests, {len(text) / 1e6:.0f} MB: native {t1 - t0:.3f} s ({len(tr) / (t1 - t0):.3e} req/s, "
      f"{os.cpu_count()} threads), reference parse_trace {t2 - t1:.3f} s ({len(tr) / (t2 - t1):.3e} req/s); "
      f"identical={bool(ok)}")
