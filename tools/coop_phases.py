"""Per-step timeline of the latency kernel (search_coop.cu) for batch-1 calls
on a config graph: the instrumented build records SM-clock timestamps of the
leader's and helper 0's phase boundaries for every expansion of query 0.
    python paper_2605_02171_b200/build.py --variant cphases -DQVG_COOP_PHASES
    QVG_LIB=build/cphases/libqvg.so python tools/coop_phases.py [CONFIG] [EF] [CALLS]
TOOL, not product."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_02171_b200 as Q  # noqa: E402
from paper_2605_02171_b200 import _native as N  # noqa: E402
from workloads import datasets, graphs  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 64
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 50
cfg = datasets.CONFIGS[cfgn]
base, queries = datasets.config_data(cfg, nq=calls)
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
del qn, codes
L = N.lib()
L.qvg_debug_coop_trace.argtypes = [C.c_void_p, C.c_int]
seg = {"helper: gather round trip": (8, 9), "helper: score": (9, 10),
       "helper: wait for pool (bar 1)": (10, 11), "helper: contender test": (11, 12),
       "leader: merge + scan (C)": (0, 1), "leader: wait S1": (1, 2),
       "leader: combine": (2, 3), "leader: adjacency row": (3, 4), "leader: filter": (4, 5)}
acc = {k: [] for k in seg}
steps_t, ms = [], []
for i in range(calls):
    r = ix.search_ex(queries[i:i + 1], k=10, ef=ef, pools=False)
    ms.append(r["stats"]["search_ms"])
    nexp = int(r["counters"][0][0])
    tr = np.zeros((1024, 16), np.uint64)
    L.qvg_debug_coop_trace(tr.ctypes.data, 1024)
    tr = tr[: nexp].astype(np.int64)
    for k, (a, b) in seg.items():
        d = tr[:, b] - tr[:, a]
        acc[k].append(d[(d > 0) & (d < 10**7)].mean())
    st = np.diff(tr[:, 0])
    steps_t.append(st[(st > 0) & (st < 10**7)].mean())
clk = 1.965e3
print(f"cfg{cfgn} ef={ef}: {calls} batch-1 calls, search kernel p50 {np.median(ms) * 1e3:.1f} us, "
      f"mean step {np.mean(steps_t) / clk:.2f} us")
for k in seg:
    print(f"  {k:32s} {np.mean(acc[k]) / clk:6.3f} us per step")
