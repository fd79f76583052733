"""Warp occupancy over time of one search launch (QVG_TAIL build).

    python paper_2605_02171_b200/build.py --variant tail -DQVG_TAIL
    QVG_LIB=build/tail/libqvg.so python tools/tail_profile.py [CONFIG] [EF]

Each query records its wall-clock span (%globaltimer) and warp slot; prints the
launch span, the mean busy fraction of the warp slots, and how much of the
span passes with fewer than 90 / 50 % of the slots busy (the tail of a
persistent warp-per-query launch).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_02171_b200 as Q  # noqa: E402
from workloads import datasets, graphs  # noqa: E402

cfg = datasets.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 64
base, queries = datasets.config_data(cfg, nq=10000)
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
if g is None:
    g = graphs.load_graph(cfg, "literal", base.shape[0], base, builder="gpu")
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
del qn, codes
import torch  # noqa: E402
qd = torch.from_numpy(queries).cuda()
for _ in range(3):
    r = ix.search_ex(qd, k=10, ef=ef, pools=False)
c = r["counters"].astype(np.int64)
t0 = c[:, 0].min()
start = (c[:, 0] - t0) & 0xFFFFFFFF
end = (c[:, 1] - t0) & 0xFFFFFFFF
warp = c[:, 2]
span = end.max()
slots = len(np.unique(warp))
busy = (end - start).sum() / (span * slots)
ts = np.linspace(0, span, 2001)
active = np.array([((start <= t) & (end > t)).sum() for t in ts])
nwarps = r["stats"].get("resident_warps_per_sm", 0)
print(f"cfg{cfg.name} ef={ef}: span {span / 1e3:.1f} us, kernel {r['stats']['search_ms'] * 1e3:.1f} us, "
      f"{slots} warp slots used, busy fraction {busy:.3f}")
print(f"  query time us: mean {(end - start).mean() / 1e3:.1f} p50 {np.median(end - start) / 1e3:.1f} "
      f"p99 {np.percentile(end - start, 99) / 1e3:.1f} max {(end - start).max() / 1e3:.1f}")
for frac in (0.9, 0.5, 0.1):
    below = (active < frac * slots).mean()
    print(f"  span fraction with < {int(frac * 100)}% of warp slots busy: {below:.3f}")
np.savez(os.path.join(ROOT, "gpurun_out", f"tail_cfg{cfg.name}_ef{ef}.npz"), start=start, end=end,
         warp=warp, counters_exp=ix.search_ex(qd, k=10, ef=ef, pools=False)["counters"][:, 0],
         pool0=ix.search_ex(qd, k=10, ef=ef)["pool_dists"][:, 0])
print(f"  contenders per query {c[:, 4].mean():.1f}")
print(f"  first time below 90 pct busy: {ts[np.argmax(active < 0.9 * slots)] / 1e3:.1f} us")
