import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2605_02171_b200 as Q
from workloads import datasets, graphs
cfg = datasets.CONFIGS[2]
base, queries = datasets.config_data(cfg, nq=1000)
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
for nq in (1, 16, 128):
    ks, ds, ts, ws = [], [], [], []
    for i in range(50):
        q = queries[i * nq % 800: i * nq % 800 + nq]
        t0 = time.perf_counter()
        ids, sc, cnt, st = ix.search(q, k=10, ef=64, stats=True)
        ws.append((time.perf_counter() - t0) * 1e3)
        ks.append(st["search_ms"]); ds.append(st["device_ms"]); ts.append(st["total_ms"])
    print(f"nq {nq}: kernel {np.median(ks):.3f} ms  device {np.median(ds):.3f}  total(events) {np.median(ts):.3f}  wall {np.median(ws):.3f}")
