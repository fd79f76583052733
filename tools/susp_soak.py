"""Soak test of tail balancing: random batch sizes / ef on the headline index,
device and host paths alternating, every result compared with the reference.  TOOL."""
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

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 150
cfg = datasets.CONFIGS[2]
base, queries = datasets.config_data(cfg, nq=20000)
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
del qn, codes
ref = RefIndex.from_graph(base, g["adj"], cfg.m, int(g["entry"]), cfg.alpha, threads=os.cpu_count())
efs = (48, 64, 100, 128, 200)
want = {ef: ref.run_query_batch(queries, ef, 10, threads=os.cpu_count()) for ef in efs}
qd = torch.from_numpy(queries).cuda()
qp = torch.from_numpy(queries).pin_memory()
rng = np.random.default_rng(7)
bad = 0
t0 = time.time()
for it in range(iters):
    ef = int(rng.choice(efs))
    nq = int(rng.integers(2369, 20001))
    off = int(rng.integers(0, 20000 - nq + 1))
    src = (qd, qp, queries)[it % 3][off:off + nq]
    ids, sc, cnt = ix.search(src, k=10, ef=ef)
    rid, rsc, rcnt = want[ef]
    ok = (np.array_equal(ids, rid[off:off + nq]) and
          np.array_equal(sc.view(np.uint32), rsc[off:off + nq].view(np.uint32)) and
          np.array_equal(cnt, rcnt[off:off + nq]))
    bad += not ok
    if not ok or it % 25 == 0:
        print(f"iter {it}: ef {ef} nq {nq} off {off} path {('device', 'pinned', 'pageable')[it % 3]} ok {ok}", flush=True)
print(f"{iters} iterations in {time.time() - t0:.1f}s, mismatches {bad}")
sys.exit(1 if bad else 0)
