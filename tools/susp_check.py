"""Tail-balancing (suspended queries) check on the headline geometry: results,
pools and counters for several batch sizes / ef against the exact-visited
(non-headline kernel, whole queries) path and the reference.  TOOL."""
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

cfg = datasets.CONFIGS[2]
base, queries = datasets.config_data(cfg, nq=30000)
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
del qn, codes
ref = RefIndex.from_graph(base, g["adj"], cfg.m, int(g["entry"]), cfg.alpha, threads=os.cpu_count())
ok = True
for ef in (16, 64, 200):
    rid, rsc, rcnt = ref.run_query_batch(queries, ef, 10, threads=os.cpu_count())
    for nq in (2369, 2400, 4736, 5000, 10000, 30000):
        q = queries[:nq]
        qd = torch.from_numpy(q).cuda()
        t0 = time.time()
        r = ix.search_ex(qd, k=10, ef=ef)                 # headline kernel, device queries
        t1 = time.time()
        h_ids, h_sc, h_cnt = ix.search(q, k=10, ef=ef)   # pipelined host path (fused prologue)
        x = ix.search_ex(q, k=10, ef=ef, exact_visited=True)
        same = (np.array_equal(r["ids"], rid[:nq]) and np.array_equal(r["scores"].view(np.uint32), rsc[:nq].view(np.uint32))
                and np.array_equal(r["count"], rcnt[:nq]) and np.array_equal(h_ids, rid[:nq])
                and np.array_equal(h_sc.view(np.uint32), rsc[:nq].view(np.uint32))
                and np.array_equal(r["pool_ids"], x["pool_ids"]) and np.array_equal(r["pool_dists"], x["pool_dists"])
                and np.array_equal(r["counters"][:, 0], x["counters"][:, 0])      # expansions
                and np.array_equal(r["counters"][:, 1], x["counters"][:, 1])      # tie expansions
                and (r["status"] == 0).all())
        ok &= same
        print(f"ef {ef} nq {nq}: identical {same}  search_ms {r['stats']['search_ms']:.3f}  "
              f"evals lossy {r['stats']['dist_evals'] / nq:.1f} exact {x['stats']['dist_evals'] / nq:.1f}", flush=True)
print("ALL OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
