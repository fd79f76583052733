"""Config-5 build quality sweep on the GPU: Recall@10 at ef=64 of GPU-built
graphs (variants of passes / batch / ef_c) next to the reference-built graph's
(tests/golden/cfg5_norm_ref_ids_ef64.npz).  TOOL.
    python tools/build_sweep.py "2,65536,128" "2,16384,128" ..."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_02171_b200 as Q  # noqa: E402
from workloads import datasets  # noqa: E402

fx = dict(np.load(os.path.join(ROOT, "tests", "golden", "cfg5_norm_ref_ids_ef64.npz")))
cfg = datasets.CONFIGS[2]
base, q = datasets.config_data(cfg, sigma_mode="norm")
qn, _, _ = Q.encode_queries(q)
bn, _, _ = Q.encode_queries(base)
gt = Q.brute_force_topk(torch.from_numpy(bn).cuda(), torch.from_numpy(qn).cuda(), 10)


def recall(ids):
    return np.mean([len(set(a.tolist()) & set(b.tolist())) for a, b in zip(ids, gt)]) / 10


print(f"reference graph: R@10 {recall(fx['ids']):.4f}", flush=True)
for spec in sys.argv[1:]:
    passes, batch, efc, vm = (int(x) for x in (spec + ",0").split(",")[:4])
    t0 = time.time()
    st = {}
    ix = Q.GpuIndex.build(base, Q.BuildParams(m=32, ef_c=efc, alpha=1.2, passes=passes,
                                              batch=batch, prune_candidates=vm), stats=st)
    dt = time.time() - t0
    ids, _, _ = ix.search(q, 10, 64)
    print(f"passes {passes} batch {batch} ef_c {efc} V-mode {vm}: R@10 {recall(ids):.4f}  build {dt:.1f}s "
          f"deg {st['mean_degree']:.2f} reprunes {st['reprunes']}", flush=True)
    ix.close()
