"""BASELINE config 5 at full size: the GPU batched BQ-space Vamana build
(qvg_build: 2 passes, alpha 1.0 then 1.2, R=64, L=128, batches of 65,536) of
1M x 768 vectors, judged by the contract's bar — "Recall@10 at ef=64 of the
GPU-built graph within 0.5 points of the reference-built graph".

The reference graph's answers come from tests/golden/cfg5_norm_ref_ids_ef64.npz
(made by tests/golden/make_cfg5_fixture.py with qivr::build_index +
qivr::run_query_batch, builder.cpp:137-155 / eval.cpp:225-247; the reference
build takes ~7 min, too long for a test).  Ground truth is recomputed here on
the GPU (qvg_brute_force_topk, bit-identical to qivr::brute_force_topk,
tests/test_gpu_eval.py).  Data: config 2's generator with sigma/sqrt(D) per
coordinate (the clustered variant: Recall@10 of order 90 %, where a 0.5-point
bar means something; the literal reading is near structureless, ~1.5 %)."""
import json
import os
import time

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import paper_2605_02171_b200 as Q  # noqa: E402
from workloads import datasets, graphs  # noqa: E402

FIXTURE = os.path.join(GOLDEN, "cfg5_norm_ref_ids_ef64.npz")


def recall(ids, gt, k=10):
    """eval.cpp:171-195 (mean |result ∩ truth| / k)"""
    hits = [len(set(a[:k].tolist()) & set(b[:k].tolist())) for a, b in zip(ids, gt)]
    return float(np.mean(hits)) / k


def test_cfg5_gpu_build_recall_within_half_point_of_reference_graph():
    fx = dict(np.load(FIXTURE))
    cfg = datasets.CONFIGS[2]
    base, q = datasets.config_data(cfg, sigma_mode="norm")
    assert str(fx["digest"]) == graphs.data_digest(base), "generator drifted from the fixture"
    assert str(fx["query_digest"]) == graphs.data_digest(q)
    import torch
    torch.cuda.synchronize()
    t0 = time.time()
    st = {}
    ix = Q.GpuIndex.build(base, Q.BuildParams(m=cfg.m, ef_c=cfg.ef_c, alpha=cfg.alpha,
                                              passes=2, batch=65536), stats=st)
    build_s = time.time() - t0
    assert st["max_degree"] <= 2 * cfg.m and st["mean_degree"] > 0.8 * 2 * cfg.m
    ids, _, cnt = ix.search(q, k=10, ef=64)
    assert (cnt == 10).all()
    # exact ground truth on the GPU over the index's own normalised rows
    _, _, cold = ix.export()
    qn, _, _ = Q.encode_queries(q)
    gt = Q.brute_force_topk(torch.from_numpy(cold).cuda(), torch.from_numpy(qn).cuda(), 10)
    rec_gpu = recall(ids, gt)
    rec_ref = recall(fx["ids"], gt)
    rec = {"config": "cfg5: N=1000000 D=768 (cfg2 generator, sigma/sqrt(D)) R=64 L=128 "
                     "2 passes alpha 1.0 -> 1.2, batch 65536",
           "gpu_build_seconds": build_s, "gpu_mean_degree": st["mean_degree"],
           "gpu_reprunes": st["reprunes"], "recall_at_10_gpu_graph": rec_gpu,
           "recall_at_10_reference_graph": rec_ref, "delta_pt": 100 * (rec_gpu - rec_ref),
           "reference_build_seconds": float(fx["ref_build_seconds"]),
           "reference_build_threads": int(fx["ref_build_threads"]),
           "reference_mean_degree": float(fx["ref_mean_degree"]), "queries": len(q)}
    print(json.dumps(rec))
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "cfg5_build_record.json"), "w") as f:
            f.write(json.dumps(rec) + "\n")
    assert rec_gpu >= rec_ref - 0.005, rec
