"""Full-size parity at every ef of a config's sweep: all queries, GPU results
(device-resident and host/pipelined) vs the reference's own run_query_batch on
the same graph (ids identical, score bit patterns identical).

    python tools/parity_sweep.py [CONFIG] [SIGMA_MODE] [EFS]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2605_02171_b200 as Q  # noqa: E402
from oracle.oracle import RefIndex  # noqa: E402
from workloads import datasets, graphs  # noqa: E402

cfg = datasets.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
mode = sys.argv[2] if len(sys.argv) > 2 else "literal"
base, queries = datasets.config_data(cfg, nq=10000, sigma_mode=mode)
g = graphs.load_graph(cfg, mode, base.shape[0], base)
if g is None:
    g = graphs.load_graph(cfg, mode, base.shape[0], base, builder="gpu")
efs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else list(cfg.efs)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
del qn, codes
ref = RefIndex.from_graph(base, g["adj"], cfg.m, int(g["entry"]), cfg.alpha, threads=os.cpu_count())
qd = torch.from_numpy(queries).cuda()
rows = []
for ef in efs:
    t0 = time.time()
    rid, rsc, rcnt = ref.run_query_batch(queries, ef, 10, threads=os.cpu_count())
    tr = time.time() - t0
    d_ids, d_sc, d_cnt = ix.search(qd, k=10, ef=ef)
    h_ids, h_sc, h_cnt = ix.search(queries, k=10, ef=ef)
    row = dict(config=cfg.name, ef=ef, queries=len(queries),
               device_ids_identical=float((d_ids == rid).all(axis=1).mean()),
               device_scores_bit_identical=float((d_sc.view(np.uint32) == rsc.view(np.uint32)).all(axis=1).mean()),
               host_ids_identical=float((h_ids == rid).all(axis=1).mean()),
               host_scores_bit_identical=float((h_sc.view(np.uint32) == rsc.view(np.uint32)).all(axis=1).mean()),
               counts_identical=bool((d_cnt == rcnt).all()), reference_seconds=tr)
    rows.append(row)
    print(json.dumps(row), flush=True)
