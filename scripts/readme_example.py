"""The README usage example end to end on a synthetic JSONL trace (checks the docs run)."""
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_02007_b200 as es  # noqa: E402
from paper_2506_02007_b200 import events  # noqa: E402

rng = np.random.default_rng(0)
d = tempfile.mkdtemp()
path = os.path.join(d, "trace.jsonl")
labels = []
with open(path, "w") as fh:
    for i in range(20000):
        slow = rng.random() < 1 / 6
        dur = int(rng.lognormal(12 if not slow else 15, 0.3))
        fh.write(json.dumps({"layer": "Nccl", "kind": "ncclAllReduce", "ts_start": 1000 + i * 100, "duration_ns": dur,
                             "pid": 1, "tid": 1, "attrs": {"message_bytes": int(rng.choice([4096, 65536, 1 << 20]))}})
                 + "\n")
        labels.append(1 if slow else 0)
labels = np.array(labels, np.uint8)

cols = events.read_trace_jsonl(path)
events.write_columnar(cols, os.path.join(d, "trace.escol"))
ds, idx = es.extract_features(events.read_columnar(os.path.join(d, "trace.escol")), "Nccl")
r = es.run_pipeline(ds, K=4, quantile_q=0.01)
m = es.metrics(es.confusion(labels, r.report.flags))
kb = es.kmeans_baseline(ds, 4, q=0.01)
mk = es.metrics(es.confusion(labels, kb.flags))
print(f"rows {ds.n_local}, GMM flagged {r.report.n_flagged}: precision {m.precision:.3f} recall {m.recall:.3f} "
      f"f1 {m.f1:.3f}; KMeans flagged {kb.n_flagged}: f1 {mk.f1:.3f}")
