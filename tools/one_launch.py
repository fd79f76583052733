"""One warm-up + one measured search launch on a config graph (for ncu).

    ncu -k regex:search_kernel -s 1 -c 1 ... python tools/one_launch.py CONFIG [NQ] [EF] [dev]

`dev`: queries already in HBM (the bench's `value` path: separate encode
kernel); default: host queries (pipelined upload + fused encode prologue).
A 6th argument picks the generator's sigma mode (literal | norm).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_02171_b200 as Q  # noqa: E402
from workloads import datasets, graphs  # noqa: E402

cfg = datasets.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
ef = int(sys.argv[3]) if len(sys.argv) > 3 else 64
mode = sys.argv[5] if len(sys.argv) > 5 else "literal"
base, queries = datasets.config_data(cfg, nq=nq, sigma_mode=mode)
g = graphs.load_graph(cfg, mode, base.shape[0], base)
if g is None:
    g = graphs.load_graph(cfg, mode, base.shape[0], base, builder="gpu")
if g is None:
    bi = Q.GpuIndex.build(base, Q.BuildParams(m=cfg.m, ef_c=cfg.ef_c, alpha=cfg.alpha))
    _, adj, _ = bi.export()
    g = dict(adj=adj, entry=bi.entry_point)
    bi.close()
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
del qn, codes
if len(sys.argv) > 4 and sys.argv[4] == "dev":
    import torch
    queries = torch.from_numpy(queries).cuda()
for _ in range(2):
    r = ix.search_ex(queries, k=10, ef=ef, pools=False, counters=False)
print("search_ms", r["stats"]["search_ms"])
