"""TEST/BENCH INPUT PREPARATION — builds a config's graph with the REFERENCE
builder (qivr::build_index, builder.cpp:137-155) exactly as BASELINE.json
specifies ("graph built in BQ space by the reference"), and caches the
adjacency + entry point under data_cache/ (git-ignored, travels to the GPU box
with the snapshot).  The base vectors are NOT stored: every consumer regenerates
them with paper_2605_02171_b200.datasets (seeded) and checks `data_digest`.

    python oracle/make_ref_graph.py --config 2 [--sigma-mode literal] [--threads 8]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import RefIndex  # noqa: E402
from workloads.datasets import CONFIGS, config_data  # noqa: E402
from workloads.graphs import data_digest, graph_path  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--sigma-mode", default="literal")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--n", type=int, default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    t0 = time.time()
    base, _ = config_data(cfg, n=a.n, nq=0, sigma_mode=a.sigma_mode)
    dig = data_digest(base)
    print(f"generated {base.shape} in {time.time() - t0:.1f}s digest={dig}", flush=True)
    t0 = time.time()
    ref = RefIndex.build(base, m=cfg.m, ef_c=cfg.ef_c, alpha=cfg.alpha, threads=a.threads,
                         seed=42)
    secs = time.time() - t0
    print(f"reference build {secs:.1f}s threads={a.threads}", flush=True)
    adj = ref.adjacency()
    path = graph_path(cfg, a.sigma_mode, base.shape[0], builder="ref")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez(path, adj=adj, entry=np.uint32(ref.entry), m=np.uint32(cfg.m),
             ef_c=np.uint32(cfg.ef_c), alpha=np.float32(cfg.alpha), digest=dig,
             build_seconds=np.float64(secs), threads=np.uint32(a.threads))
    deg = adj[:, 0]
    print(f"saved {path}: degree mean {deg.mean():.2f} min {deg.min()} max {deg.max()}")


if __name__ == "__main__":
    main()
