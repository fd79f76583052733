"""Where a small-batch call's time goes: device spans from the call's own
events (qvg_stats: encode, search, device, total incl. copies) next to the
host wall time of the call and a CUDA-event bracket like bench.py's.  TOOL.
    python tools/call_breakdown.py [CONFIG] [BATCH] [CALLS]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_02171_b200 as Q  # noqa: E402
from workloads import datasets, graphs  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 100
cfg = datasets.CONFIGS[cfgn]
base, queries = datasets.config_data(cfg, nq=B * calls)
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
del qn, codes
stream = torch.cuda.current_stream()
ix.set_stream(stream)
qd = torch.from_numpy(queries).cuda()
out = (torch.empty((B, 10), dtype=torch.int32, device="cuda"),
       torch.empty((B, 10), dtype=torch.float32, device="cuda"),
       torch.empty(B, dtype=torch.int32, device="cuda"))
rows = []
for c in range(calls):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    t0 = time.perf_counter()
    _, _, _, st = ix.search(qd[c * B:(c + 1) * B], k=10, ef=64, out=out, stats=True)
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    rows.append((e0.elapsed_time(e1), (t1 - t0) * 1e3, st["encode_ms"], st["search_ms"],
                 st["device_ms"], st["total_ms"]))
r = np.median(np.array(rows[5:]), axis=0)
print(f"cfg{cfgn} batch {B}: p50 over {calls - 5} calls (ms)")
for n_, v in zip(["bench-style event bracket", "host wall time of the call", "encode kernel",
                  "search kernel", "encode..search (device)", "call total (first..last event)"], r):
    print(f"  {n_:32s} {v:.4f}")
