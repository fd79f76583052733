"""Generate the committed golden fixtures from the REFERENCE library itself.

Run here (needs /root/reference compiled by `make -C oracle`):
    python tests/golden/make_golden.py
Every expected value below is produced by the reference (oracle/_ref,
libqivr_ref.so = /root/reference/proj/core/src/*.cpp + forwarding shim):
qivr::build_index (threads=1, deterministic), run_query_batch, beam_search_words,
encode_sm2 / normalize_l2, brute_force_topk.  The fixtures travel with the repo;
the GPU tests compare against them without needing /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import (RefIndex, ref_brute_force_topk, ref_encode_query,  # noqa: E402
                           ref_encode_raw, ref_sm2, words_for_dim)
from workloads.datasets import mixture  # noqa: E402


def u64list(a):
    return [int(x) for x in np.asarray(a, np.uint64).reshape(-1)]


def known_answers():
    out = {}
    v = [0.5, -0.2, 0.9, -0.1]
    code, tau = ref_encode_raw(np.array(v, np.float32))
    out["encode_worked"] = dict(x=v, code=u64list(code), tau=float(tau))
    zero_code, zero_tau = ref_encode_raw(np.zeros(4, np.float32))
    out["encode_zero"] = dict(x=[0, 0, 0, 0], code=u64list(zero_code), tau=float(zero_tau))
    ones_code, ones_tau = ref_encode_raw(np.ones(4, np.float32))
    out["encode_ones"] = dict(x=[1, 1, 1, 1], code=u64list(ones_code), tau=float(ones_tau))
    pairs = [([0.5, -0.2, 0.9, -0.1], [-0.5, -0.2, 0.9, 0.1]),
             ([9, -9, 9, 0.1], [-9, 9, -9, 0.2])]
    out["sm2_pairs"] = []
    for a, b in pairs:
        ca, _ = ref_encode_raw(np.array(a, np.float32))
        cb, _ = ref_encode_raw(np.array(b, np.float32))
        out["sm2_pairs"].append(dict(a=a, b=b, dist=ref_sm2(ca, cb)))
    # constructed maximum penalty (test_encoding.cpp "sm2 maximum penalty 4D")
    a = np.array([0b1111, 0b1111], np.uint64)
    b = np.array([0b0000, 0b1111], np.uint64)
    out["sm2_constructed"] = dict(a=u64list(a), b=u64list(b), dist=ref_sm2(a, b))
    # query-path encodings (normalise then encode) at awkward dims
    rng = np.random.Generator(np.random.PCG64(5))
    qe = []
    for d in (1, 3, 4, 63, 64, 65, 99, 100, 384, 1023):
        x = rng.standard_normal(d).astype(np.float32)
        nrm, code, tau = ref_encode_query(x)
        qe.append(dict(dim=d, x=x.view(np.uint32).tolist(), norm=nrm.view(np.uint32).tolist(),
                       code=u64list(code), tau=float(tau)))
    out["query_encodings"] = qe
    return out


def save_index_npz(path, ref: RefIndex, queries, efs, k=10, extra=None, gt=True):
    d = dict(codes=ref.codes(), adj=ref.adjacency(), cold=ref.cold(),
             entry=np.uint32(ref.entry), m=np.uint32(ref.m), queries=queries,
             efs=np.array(efs, np.uint32), k=np.uint32(k))
    for ef in efs:
        ids, sc, cnt = ref.run_query_batch(queries, ef, k, threads=1)
        d[f"ids_{ef}"] = ids
        d[f"scores_{ef}"] = sc.view(np.uint32)  # bit patterns
        d[f"count_{ef}"] = cnt
        P = np.full((len(queries), ef), 0xFFFFFFFF, np.uint32)
        Pd = np.full((len(queries), ef), 0xFFFFFFFF, np.uint32)
        Pn = np.zeros(len(queries), np.uint32)
        for i, q in enumerate(queries):
            _, code, _ = ref_encode_query(q)
            pi, pd = ref.beam_search(code, ef)
            P[i, : len(pi)] = pi
            Pd[i, : len(pi)] = pd
            Pn[i] = len(pi)
        d[f"pool_ids_{ef}"] = P
        d[f"pool_dists_{ef}"] = Pd
        d[f"pool_n_{ef}"] = Pn
    if gt:
        d["gt10"] = ref_brute_force_topk(ref.cold(), queries, 10, threads=8)
    if extra:
        d.update(extra)
    np.savez_compressed(path, **d)


def main():
    ka = known_answers()
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(ka, f, indent=1)

    # g1: clustered mixture, D=64, single-threaded (deterministic) reference build
    base, q = mixture(1500, 64, 30, 0.35, seed=7, nq=200, sigma_mode="norm")
    q = np.concatenate([q, base[[0, 5, 77, 1499]]])  # self-queries
    ref = RefIndex.build(base, m=8, ef_c=48, alpha=1.2, threads=1, seed=42)
    save_index_npz(os.path.join(HERE, "g1.npz"), ref, q, efs=(10, 32, 100))

    # g2: D=99 (pad bits, float tail), R=10, includes ef >= N
    base, q = mixture(700, 99, 12, 0.35, seed=9, nq=60, sigma_mode="literal")
    ref = RefIndex.build(base, m=5, ef_c=20, alpha=1.2, threads=1, seed=3)
    save_index_npz(os.path.join(HERE, "g2.npz"), ref, q, efs=(10, 50, 700))

    # g3: hand-made pathological graph: duplicate ids in a row, self loops,
    # degree-0 entry neighbourhood, unreachable nodes, zero-id slots.
    rng = np.random.Generator(np.random.PCG64(11))
    n, dim, m = 120, 40, 4
    R = 2 * m
    raw = rng.standard_normal((n, dim)).astype(np.float32)
    cold = raw / np.linalg.norm(raw, axis=1, keepdims=True)
    W = words_for_dim(dim)
    codes = np.zeros((n, 2 * W), np.uint64)
    for i in range(n):
        c, _ = ref_encode_raw(cold[i])
        codes[i] = c
    adj = np.zeros((n, R + 1), np.uint32)
    for u in range(n):
        if u >= 110:
            continue  # unreachable tail / zero degree
        deg = int(rng.integers(0, R + 1))
        ids = rng.integers(0, 110, deg).astype(np.uint32)
        if deg >= 3:
            ids[2] = ids[0]      # duplicate
            ids[1] = u           # self loop
        adj[u, 0] = deg
        adj[u, 1:1 + deg] = ids
    adj[0, 1:4] = [0, 0, 7]  # zero ids (valid id 0) plus a real one
    adj[0, 0] = 3
    ref = RefIndex.from_parts(codes, adj, cold, dim, m, entry=3, alpha=1.2)
    q = rng.standard_normal((40, dim)).astype(np.float32)
    save_index_npz(os.path.join(HERE, "g3.npz"), ref, q, efs=(5, 10, 40, 120), k=5,
                   gt=False)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
