import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_02171_b200 as Q
from workloads import datasets, graphs
cfg = datasets.CONFIGS[2]
base, queries = datasets.config_data(cfg, nq=10000)
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
pin = torch.from_numpy(queries).pin_memory()
for name, q in (("pageable", queries), ("pinned", pin)):
    for _ in range(3): ix.search(q, k=10, ef=64)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20): ix.search(q, k=10, ef=64)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
    print(name, f"{dt*1e3:.3f} ms per 10k batch -> {1e4/dt/1e6:.3f} M QPS (host wall clock)")
