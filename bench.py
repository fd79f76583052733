#!/usr/bin/env python
"""Benchmark of the B200-native BQ query path (BASELINE.json metric):
"batched QPS @ Recall@10 vs ef on 1 B200; gathered-bytes GB/s vs HBM peak".

One step = one batch of `--nq` queries (default 10,000) through encode ->
exact BQ beam search -> float32 rerank, on the headline workload (config 2:
N=1e6, D=768, R=64, L=128, alpha=1.2, ef=64, k=10, literal sigma=0.3).
The graph is the reference-built one cached in data_cache/ (see
oracle/make_ref_graph.py); vectors and queries are regenerated (seeded).

  value : device-resident queries, CUDA events on the launching stream around
          each step, L2 flushed (256 MB write) between steps.
  e2e   : the same search through the public API with pinned HOST buffers:
          H2D of the queries and D2H of ids/scores/counts inside each step.
  --impl reference : the reference's own CPU run_query_batch (oracle/_ref) on
          the same graph/queries, all host threads.
Multi-GPU (torchrun): replicas only — every rank runs its own batch on its own
copy of the index; no collective on the data path; max-over-ranks timing.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched QPS @ Recall@10 vs ef on 1 B200; gathered-bytes GB/s vs HBM peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--ef", type=int, default=64)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--n", type=int, default=None, help="override corpus size (testing)")
    ap.add_argument("--sigma-mode", default="literal", choices=["literal", "norm"])
    ap.add_argument("--sweep", default="auto", help="extra ef values ('auto', 'none', list)")
    ap.add_argument("--sweep-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--recall-queries", type=int, default=1000)
    ap.add_argument("--visited-slots", type=int, default=0)
    ap.add_argument("--rerank-depths", default="auto",
                    help="GPU-only rerank-depth rows: 'auto' = config 4's ef x {ef, 2ef}, "
                         "'none', or 'ef:depth,...'")
    ap.add_argument("--batch-sizes", default="auto",
                    help="latency regime: batch sizes to time per call ('auto' = config 3's "
                         "{1,128,10000} when --config 3, 'none', or a list)")
    ap.add_argument("--relaxed", default="2",
                    help="relaxed-variant rows at the headline ef: expansions per step "
                         "list ('2', '2,4', 'none'); reported separately, never parity")
    ap.add_argument("--depth-parity-queries", type=int, default=500,
                    help="queries checked against orc_query_depth per rerank-depth row")
    ap.add_argument("--variant-rows", default="auto",
                    help="'auto': with the default headline run also report the clearly-labelled "
                         "sigma/sqrt(D) variant of the same config (SURVEY 8d), 'none': skip")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    return ap.parse_args()


# ----------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def log(*a):
    if int(os.environ.get("RANK", "0")) == 0:
        print(*a, file=sys.stderr, flush=True)


def load_workload(args, allow_gpu_build=True):
    """-> (cfg, base, queries, adjacency, entry, provenance).  The reference arm
    passes allow_gpu_build=False: it never imports the product package, and
    without a cached graph it builds one with the reference builder."""
    from workloads import datasets, graphs
    cfg = datasets.CONFIGS[args.config]
    t0 = time.time()
    base, queries = datasets.config_data(cfg, n=args.n, nq=args.nq, sigma_mode=args.sigma_mode)
    log(f"[bench] generated {base.shape} + {queries.shape} in {time.time() - t0:.1f}s")
    g = graphs.load_graph(cfg, args.sigma_mode, base.shape[0], base, builder="ref")
    provenance = "reference qivr::build_index (cached, data_cache/)"
    if g is None:
        g = graphs.load_graph(cfg, args.sigma_mode, base.shape[0], base, builder="gpu")
        provenance = "GPU builder qvg_build (cached, data_cache/)"
    if g is None and not allow_gpu_build:
        from oracle.oracle import RefIndex
        log("[bench] no cached graph: building with the reference builder")
        t0 = time.time()
        ref = RefIndex.build(base, m=cfg.m, ef_c=cfg.ef_c, alpha=cfg.alpha, seed=42)
        g = dict(adj=ref.adjacency(), entry=np.uint32(ref.entry))
        provenance = f"reference qivr::build_index (built in this run, {time.time() - t0:.0f}s)"
        ref.close()
    if g is None:
        import paper_2605_02171_b200 as Q
        log("[bench] no cached graph: building on the GPU (qvg_build)")
        t0 = time.time()
        st = {}
        ix = Q.GpuIndex.build(base, Q.BuildParams(m=cfg.m, ef_c=cfg.ef_c, alpha=cfg.alpha),
                              stats=st)
        _, adj, _ = ix.export()
        g = dict(adj=adj, entry=np.uint32(ix.entry_point), build_seconds=time.time() - t0)
        path = graphs.graph_path(cfg, args.sigma_mode, base.shape[0], builder="gpu")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        np.savez(path, adj=adj, entry=np.uint32(ix.entry_point), m=np.uint32(cfg.m),
                 ef_c=np.uint32(cfg.ef_c), alpha=np.float32(cfg.alpha),
                 digest=graphs.data_digest(base), build_seconds=np.float64(g["build_seconds"]))
        provenance = "GPU builder qvg_build (built in this run)"
        ix.close()
    return cfg, base, queries, g["adj"], int(g["entry"]), provenance


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload_key):
    """dram bytes per launch of the search kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    e = d.get(workload_key)
    if not e:
        return None, None
    return e.get("dram_bytes_per_launch"), e.get("source")


def algorithmic_bytes(st, W, D, k, nq):
    """sum_exp(4+4 deg) + evals*16W + |pool|*4D + 4D + 8k per query."""
    return (st["adjacency_bytes"] + st["dist_evals"] * 16 * W + st["cold_accesses"] * 4 * D +
            nq * (4 * D + 8 * k))


def recall_at_k(res, gt, k):
    """eval.cpp:171-195"""
    tot = 0.0
    if gt is None or len(res) == 0:
        return None
    for r, g in zip(res, gt):
        gs = set(int(x) for x in g[:k])
        tot += sum(1 for x in r[:k] if int(x) in gs) / k
    return tot / len(res)


# ----------------------------------------------------------------------------
L2_NOTE = ("GPU arm: L2 flushed between steps (256 MB write); "
           "reference arm: CPU, host caches not flushed")


def bench_config(args, cfg, n, D, nq, provenance):
    """The `config` object — byte-identical in both arms (same workload, same graph)."""
    return {"workload": f"cfg{args.config}: N={n} D={D} R={2 * cfg.m} L={cfg.ef_c} "
                        f"alpha={cfg.alpha} nq={nq} ef={args.ef} k={args.k} "
                        f"sigma={cfg.sigma} ({args.sigma_mode})",
            "graph": provenance, "l2": L2_NOTE}


def cpu_info():
    """Host CPU of the baseline: model, physical cores, logical CPUs, SMT, and the
    threads this process may run on (the count the baseline uses)."""
    model, phys, cores, logical = None, None, set(), 0
    try:
        for ln in open("/proc/cpuinfo"):
            key, _, v = ln.partition(":")
            key, v = key.strip(), v.strip()
            if key == "processor":
                logical += 1
            elif key == "model name" and model is None:
                model = v
            elif key == "physical id":
                phys = v
            elif key == "core id":
                cores.add((phys, v))
    except Exception:
        pass
    usable = (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
              else os.cpu_count() or 1)
    physical = len(cores) or None
    return {"model": model, "logical_cpus": logical or os.cpu_count(),
            "physical_cores": physical,
            "smt": None if physical is None else bool(logical > physical),
            "threads_used": usable}


class RefRunner:
    """The reference's own CPU path — qivr::run_query_batch from oracle/_ref (the
    unmodified reference compiled from its sources) — on the same graph and
    queries.  Results are cached per ef: they are the parity oracle of every
    timed GPU row."""

    def __init__(self, cfg, base, adj, entry, threads):
        from oracle.oracle import RefIndex
        t0 = time.time()
        self.ref = RefIndex.from_graph(base, adj, cfg.m, entry, cfg.alpha, threads=threads)
        log(f"[bench] reference index (stage0 + cached graph) in {time.time() - t0:.1f}s")
        self.threads = threads
        self.cache = {}

    def results(self, queries, ef, k):
        if ef not in self.cache:
            self.cache[ef] = self.ref.run_query_batch(queries, ef, k, threads=self.threads)
        return self.cache[ef]

    def timed(self, queries, ef, k, threads=None):
        t0 = time.time()
        r = self.ref.run_query_batch(queries, ef, k, threads=threads or self.threads)
        return r, time.time() - t0

    def oracle_view(self):
        """Plain-C restatement over the reference's own stores (for the GPU-only
        rerank-depth rows, which have no reference counterpart)."""
        from oracle.oracle import OracleIndex
        return OracleIndex.from_ref(self.ref)


def parity(got, want, rows=None):
    """ids / score bit patterns / counts of one timed output vs the reference,
    compared over each query's first count[i] (= reference count) entries."""
    ids, sc, cnt = (np.asarray(x) for x in got)
    rids, rsc, rcnt = want
    if rows is not None:
        rids, rsc, rcnt = rids[rows], rsc[rows], rcnt[rows]
    ids = ids.view(np.uint32).reshape(rids.shape)
    sc = sc.view(np.uint32).reshape(rsc.shape)
    cnt = cnt.view(np.uint32).reshape(rcnt.shape)
    mask = np.arange(rids.shape[1])[None, :] < rcnt[:, None]
    ok_ids = np.where(mask, ids == rids, True).all(axis=1) & (cnt == rcnt)
    ok_sc = np.where(mask, sc == rsc.view(np.uint32), True).all(axis=1) & (cnt == rcnt)
    return {"queries": int(rids.shape[0]), "ids_identical": float(ok_ids.mean()),
            "scores_bit_identical": float(ok_sc.mean()),
            "counts_identical": float((cnt == rcnt).mean())}


def clustered_variant(args, local, k, threads):
    """the literal generator's per-coordinate sigma gives a nearly
    structureless mixture (Recall@10 of a few %), so the headline config is also
    reported on its clearly-labelled sigma / sqrt(D) variant, where "QPS @
    Recall@10 vs ef" is meaningful: device-resident QPS, Recall@10 against exact
    ground truth and parity against the reference on the same graph, per ef.
    The graph is the cached reference-built one when present, else built here by
    qvg_build (and then handed to the reference for the parity run)."""
    import ctypes as C

    import torch

    import paper_2605_02171_b200 as Q
    from paper_2605_02171_b200 import _native as N
    va = argparse.Namespace(**vars(args))
    va.sigma_mode = "norm"
    cfg, base, queries, adj, entry, provenance = load_workload(va)
    nq, D = queries.shape
    qn, codes, _ = Q.encode_queries(base, device=local)
    ix = Q.GpuIndex.from_arrays(codes, adj, qn, entry, device=local)
    del codes
    stream = torch.cuda.current_stream()
    ix.set_stream(stream)
    rq = min(max(args.recall_queries, 1000), nq)
    base_dev = torch.from_numpy(qn).cuda()
    qnq, _, _ = Q.encode_queries(queries[:rq], device=local)
    gt = Q.brute_force_topk(base_dev, torch.from_numpy(qnq).cuda(), k, device=local)
    del base_dev, qn
    rr = RefRunner(cfg, base, adj, entry, threads)
    q_dev = torch.from_numpy(queries).cuda()
    ids_d = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    sc_d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cnt_d = torch.empty(nq, dtype=torch.int32, device="cuda")
    st_d = torch.empty(nq, dtype=torch.int32, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    opts = N.qvg_search_opts(entry_point=N.SENTINEL, timing_only=1)
    rows = []
    for e in (64, 128, 256):
        def step():
            st = N.qvg_stats()
            if N.lib().qvg_search_ex(ix._h, q_dev.data_ptr(), nq, k, e, C.byref(opts),
                                     ids_d.data_ptr(), sc_d.data_ptr(), cnt_d.data_ptr(),
                                     st_d.data_ptr(), None, None, None, None, C.byref(st)):
                raise RuntimeError(N.last_error())
            return st
        for _ in range(3):
            step()
        ev, kern = [], []
        torch.cuda.synchronize()
        for _ in range(args.sweep_steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            kern.append(step().search_ms)
            e1.record(stream)
            ev.append((e0, e1))
        torch.cuda.synchronize()
        t_ms = sum(a.elapsed_time(b) for a, b in ev)
        got = (ids_d.cpu().numpy().view(np.uint32).copy(), sc_d.cpu().numpy().copy(),
               cnt_d.cpu().numpy().view(np.uint32).copy())
        want, dt = rr.timed(queries, e, k)
        rows.append(dict(ef=e, qps=nq * args.sweep_steps / (t_ms / 1e3),
                         kernel_ms=float(np.mean(kern)),
                         recall_at_10=recall_at_k(got[0][:rq], gt, k),
                         reference_cpu_qps=nq / dt, parity=parity(got, want)))
    ix.close()
    return {"workload": f"cfg{args.config} with sigma / sqrt(D): N={base.shape[0]} D={D} nq={nq} k={k}",
            "graph": provenance, "recall_gt": f"exact brute force, first {rq} queries",
            "timing": f"device-resident queries, {args.sweep_steps} steps per row, L2 flushed",
            "rows": rows}


def ours(args):
    import ctypes as C

    import torch

    import paper_2605_02171_b200 as Q
    from paper_2605_02171_b200 import _native as N

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, base, queries, adj, entry, provenance = load_workload(args)
    n, D = base.shape
    k, ef = args.k, args.ef

    t0 = time.time()
    qn, codes, _ = Q.encode_queries(base, device=local)  # stage0: normalize + encode
    ix = Q.GpuIndex.from_arrays(codes, adj, qn, entry, device=local)
    del codes
    log(f"[bench] index in HBM in {time.time() - t0:.1f}s (n={n}, D={D}, R={ix.max_degree})")
    stream = torch.cuda.current_stream()
    ix.set_stream(stream)
    nq = queries.shape[0]
    W = ix.W

    # ---- untimed stats passes: exact visited (algorithmic counts) and default
    ex = ix.search_ex(queries, k=k, ef=ef, exact_visited=True, pools=False)
    lo = ix.search_ex(queries, k=k, ef=ef, visited_slots=args.visited_slots, pools=False)
    assert np.array_equal(ex["ids"], lo["ids"]), "lossy-visited result differs from exact"
    alg_bytes = algorithmic_bytes(ex["stats"], W, D, k, nq)

    q_host = torch.from_numpy(queries).pin_memory()
    q_dev = q_host.cuda()
    ids_d = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    sc_d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cnt_d = torch.empty(nq, dtype=torch.int32, device="cuda")
    st_d = torch.empty(nq, dtype=torch.int32, device="cuda")
    ids_h = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    sc_h = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    cnt_h = torch.empty(nq, dtype=torch.int32).pin_memory()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    opts = N.qvg_search_opts(visited_slots=args.visited_slots, entry_point=N.SENTINEL,
                             timing_only=1)

    def dev_out():
        """the last timed device launch's outputs (host copies)"""
        torch.cuda.synchronize()
        return (ids_d.cpu().numpy().view(np.uint32).copy(), sc_d.cpu().numpy().copy(),
                cnt_d.cpu().numpy().view(np.uint32).copy())

    def step_dev(efv=ef, o=opts, q_ptr=None, nqv=None):
        st = N.qvg_stats()
        rc = N.lib().qvg_search_ex(ix._h, q_ptr or q_dev.data_ptr(), nqv or nq, k, efv,
                                   C.byref(o), ids_d.data_ptr(), sc_d.data_ptr(),
                                   cnt_d.data_ptr(), st_d.data_ptr(), None, None, None, None,
                                   C.byref(st))
        if rc:
            raise RuntimeError(N.last_error())
        return st

    def step_e2e():
        # the public drop-in call (qvg_search = run_query_batch) on pinned host buffers
        rc = N.lib().qvg_search(ix._h, q_host.data_ptr(), nq, k, ef, ids_h.data_ptr(),
                                sc_h.data_ptr(), cnt_h.data_ptr(), None, None)
        if rc:
            raise RuntimeError(N.last_error())

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, sampler=None):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        kern = []
        barrier()
        if sampler:
            sampler.start()
        for i in range(steps):
            flush.zero_()
            ev[i][0].record(stream)
            r = fn()
            ev[i][1].record(stream)
            if r is not None:
                kern.append(r.search_ms)
        barrier()
        clocks = sampler.stop() if sampler else None
        ms = [a.elapsed_time(b) for a, b in ev]
        tot = sum(ms)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([tot], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = float(t.item())
        return tot, ms, kern, clocks

    for _ in range(max(args.warmup, 3)):
        step_dev()
        step_e2e()
    sampler = ClockSampler(local)
    tot_ms, ms, kern_ms, clocks = timed(step_dev, args.steps, sampler)
    out_dev = dev_out()
    e2e_ms, _, _, _ = timed(step_e2e, args.steps)
    out_e2e = (ids_h.numpy().view(np.uint32).copy(), sc_h.numpy().copy(),
               cnt_h.numpy().view(np.uint32).copy())
    assert np.array_equal(out_dev[0], ex["ids"]), "timed results differ from the stats pass"

    value = world * nq * args.steps / (tot_ms / 1e3)
    e2e = world * nq * args.steps / (e2e_ms / 1e3)
    kern_avg = float(np.mean(kern_ms))
    peak, peak_src = measured_peaks()
    achieved = alg_bytes / (kern_avg / 1e3) / 1e9
    key = f"cfg{args.config}_{args.sigma_mode}_ef{ef}_nq{nq}"
    traffic, traffic_src = ncu_traffic(key)

    # ---- recall (GPU exact brute force on a sample) ---------------------------
    rq = min(args.recall_queries, nq)
    gt = None
    if rq > 0:
        base_dev = torch.from_numpy(qn).cuda()
        qnq, _, _ = Q.encode_queries(queries[:rq], device=local)  # normalised like query()
        # exact ground truth on the GPU: qivr::brute_force_topk(float_cosine)
        # semantics (4-chain double dot, ties by id) via qvg_brute_force_topk
        gt = Q.brute_force_topk(base_dev, torch.from_numpy(qnq).cuda(), k, device=local)
        del base_dev
    recall = recall_at_k(ex["ids"][:rq], gt, k)

    # ---- ef sweep (each row's timed outputs are kept for parity) --------------
    sweep, sweep_out = [], []
    efs = [] if args.sweep == "none" else (
        [e for e in cfg.efs if e != ef] if args.sweep == "auto" else
        [int(x) for x in args.sweep.split(",") if x])
    for e in efs:
        if e < k:
            continue
        s_ex = ix.search_ex(queries, k=k, ef=e, exact_visited=True, pools=False)
        for _ in range(3):
            step_dev(e)
        t_ms, _, km, _ = timed(lambda: step_dev(e), args.sweep_steps)
        sweep_out.append(dev_out())
        b = algorithmic_bytes(s_ex["stats"], W, D, k, nq)
        ka = float(np.mean(km))
        sweep.append(dict(ef=e, qps=world * nq * args.sweep_steps / (t_ms / 1e3),
                          recall_at_10=recall_at_k(s_ex["ids"][:rq], gt, k),
                          kernel_ms=ka, gbs=b / (ka / 1e3) / 1e9,
                          frac=b / (ka / 1e3) / 1e9 / peak,
                          bytes_per_query=b / nq,
                          expansions_per_query=s_ex["stats"]["expansions"] / nq,
                          evals_per_query=s_ex["stats"]["dist_evals"] / nq))

    # ---- rerank depth (config 4): share of the rerank in time and bytes ---------
    depth_rows, depth_out = [], []
    if args.rerank_depths == "auto":
        pairs = [(e, d) for e in cfg.efs for d in (e, 2 * e)] if args.config == 4 else []
    elif args.rerank_depths == "none":
        pairs = []
    else:  # "ef:depth,ef:depth"
        pairs = [tuple(int(v) for v in p.split(":")) for p in args.rerank_depths.split(",") if p]
    for e, d in pairs:
        o_d = N.qvg_search_opts(visited_slots=args.visited_slots, entry_point=N.SENTINEL,
                                timing_only=1, rerank_depth=d)
        o_nr = N.qvg_search_opts(visited_slots=args.visited_slots, entry_point=N.SENTINEL,
                                 timing_only=1, no_rerank=1)
        s_ex = ix.search_ex(queries, k=k, ef=e, exact_visited=True, pools=False, rerank_depth=d)
        for _ in range(3):
            step_dev(e, o_d)
            step_dev(e, o_nr)
        t_ms, _, km, _ = timed(lambda: step_dev(e, o_d), args.sweep_steps)
        depth_out.append(dev_out())
        _, _, km_nr, _ = timed(lambda: step_dev(e, o_nr), args.sweep_steps)
        b = algorithmic_bytes(s_ex["stats"], W, D, k, nq)
        ka, kn = float(np.mean(km)), float(np.mean(km_nr))
        depth_rows.append(dict(
            ef=e, depth=d, qps=world * nq * args.sweep_steps / (t_ms / 1e3), kernel_ms=ka,
            kernel_ms_no_rerank=kn, rerank_time_share=1.0 - kn / ka,
            rerank_rows_per_query=s_ex["stats"]["cold_accesses"] / nq,
            rerank_byte_share=s_ex["stats"]["cold_accesses"] * 4 * D / b,
            gbs=b / (ka / 1e3) / 1e9, recall_at_10=recall_at_k(s_ex["ids"][:rq], gt, k)))

    # ---- relaxed variant: reported separately, never the
    # parity path; Recall@10 against the same ground truth as the exact rows ----
    rel_rows = []
    rels = [] if args.relaxed == "none" else [int(x) for x in args.relaxed.split(",") if x]
    for rx in rels:
        if rx * ((ix.max_degree + 31) // 32) > 4:
            continue
        o_r = N.qvg_search_opts(visited_slots=args.visited_slots, entry_point=N.SENTINEL,
                                timing_only=1, relaxed_expansions=rx)
        s_r = ix.search_ex(queries, k=k, ef=ef, pools=False, relaxed=rx)
        for _ in range(3):
            step_dev(ef, o_r)
        t_ms, _, km, _ = timed(lambda: step_dev(ef, o_r), args.sweep_steps)
        ka = float(np.mean(km))
        r_rec = recall_at_k(s_r["ids"][:rq], gt, k)
        rel_rows.append(dict(
            ef=ef, expansions_per_step=rx, qps=world * nq * args.sweep_steps / (t_ms / 1e3),
            kernel_ms=ka, recall_at_10=r_rec, exact_recall_at_10=recall,
            recall_delta_pt=(None if r_rec is None or recall is None else 100 * (r_rec - recall)),
            expansions_per_query=s_r["stats"]["expansions"] / nq,
            evals_per_query=s_r["stats"]["dist_evals"] / nq,
            ids_identical_to_exact=float((s_r["ids"] == ex["ids"]).all(axis=1).mean())))

    # ---- latency regime: per-call latency at small batch sizes (config 3) -------
    # every timed call's outputs are kept (copied after its closing event) for parity
    lat, lat_out = [], []
    bss = ([1, 128, 10000] if args.config == 3 else []) if args.batch_sizes == "auto" else (
        [] if args.batch_sizes == "none" else [int(x) for x in args.batch_sizes.split(",") if x])
    for B in bss:
        B = min(B, nq)
        calls = max(20, min(200, 20000 // B))
        times, outs = [], []
        for c in range(calls + 3):
            off = (c * B) % max(1, nq - B + 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step_dev(ef, opts, q_dev.data_ptr() + off * D * 4, B)
            e1.record(stream)
            torch.cuda.synchronize()
            if c >= 3:
                times.append(e0.elapsed_time(e1))
                outs.append((off, ids_d[:B].cpu().numpy().view(np.uint32).copy(),
                             sc_d[:B].cpu().numpy().copy(),
                             cnt_d[:B].cpu().numpy().view(np.uint32).copy()))
        lat_out.append(outs)
        st = sorted(times)
        lat.append(dict(batch=B, calls=calls, p50_ms=st[len(st) // 2],
                        p99_ms=st[min(len(st) - 1, int(0.99 * len(st)))],
                        qps=B * len(st) / (sum(st) / 1e3)))

    # ---- CPU baseline + parity of every timed output (rank 0, N=1) -------------
    cpu, par = None, None
    if rank == 0 and world == 1:
        try:
            from oracle.oracle import ref_available
            if not ref_available():
                raise RuntimeError("oracle/_ref/libqivr_ref.so missing (run make -C oracle ref)")
            ci = cpu_info()
            threads = ci["threads_used"]
            rr = RefRunner(cfg, base, adj, entry, threads)
            if not args.no_cpu_baseline:
                runs = []
                for _ in range(3):
                    r, dt = rr.timed(queries, ef, k)
                    runs.append(nq / dt)
                rr.cache[ef] = r
                n1 = 300
                _, dt1 = rr.timed(queries[:n1], ef, k, threads=1)
                cpu = {"value": float(np.mean(runs)), "unit": "queries/s", "cores": threads,
                       "kind": "reference",
                       "sample": f"the full {nq}-query cfg{args.config} batch x 3 runs, ef={ef}, "
                                 f"k={k}: qivr::run_query_batch with {threads} threads "
                                 "(oracle/_ref, -O3 -march=sapphirerapids)",
                       "qps_1thread": n1 / dt1, "cpu": ci}
            want = rr.results(queries, ef, k)
            par = {"vs": "reference qivr::run_query_batch on the same graph and queries",
                   "timed_device": parity(out_dev, want),
                   "timed_e2e": parity(out_e2e, want),
                   "stats_pass": parity((ex["ids"], ex["scores"], ex["count"]), want)}
            for row, o in zip(sweep, sweep_out):
                row["parity"] = parity(o, rr.results(queries, row["ef"], k))
            for row, outs in zip(lat, lat_out):
                agg = {"queries": 0, "ids_identical": 0.0, "scores_bit_identical": 0.0,
                       "counts_identical": 0.0}
                for off, i_, s_, c_ in outs:
                    p = parity((i_, s_, c_), want, rows=slice(off, off + row["batch"]))
                    for f in ("ids_identical", "scores_bit_identical", "counts_identical"):
                        agg[f] += p[f] * p["queries"]
                    agg["queries"] += p["queries"]
                for f in ("ids_identical", "scores_bit_identical", "counts_identical"):
                    agg[f] /= max(agg["queries"], 1)
                agg["vs"] = "reference, every timed call"
                row["parity"] = agg
            orc = None
            for row, o in zip(depth_rows, depth_out):
                if row["depth"] == row["ef"]:
                    row["parity"] = parity(o, rr.results(queries, row["ef"], k))
                    row["parity"]["vs"] = "reference run_query_batch"
                else:  # GPU-only knob: the C restatement's orc_query_depth
                    orc = orc or rr.oracle_view()
                    sq = min(nq, args.depth_parity_queries)
                    od = orc.query_depth(queries[:sq], row["ef"], k, row["depth"])
                    row["parity"] = parity(tuple(x[:sq] for x in o),
                                           (od["ids"], od["scores"], od["count"]))
                    row["parity"]["vs"] = f"oracle orc_query_depth, first {sq} queries"
        except Exception as exc:  # report, never fake
            log(f"[bench] reference leg failed: {exc!r}")
            if cpu is None and not args.no_cpu_baseline:
                cpu = {"value": None, "error": str(exc)[:200]}
            par = par or {"error": str(exc)[:200]}

    if rank != 0:
        return
    variant = None
    if (world == 1 and args.variant_rows == "auto" and args.config == 2 and
            args.sigma_mode == "literal" and args.n is None):
        try:
            ix.close()
            del base, flush
            torch.cuda.empty_cache()
            variant = clustered_variant(args, local, k, cpu_info()["threads_used"])
        except Exception as exc:  # report, never fake
            log(f"[bench] sigma/sqrt(D) variant failed: {exc!r}")
            variant = {"error": str(exc)[:200]}
    out = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded clustered mixture)",
        "config": bench_config(args, cfg, n, D, nq, provenance),
        "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
        "recall_at_10": recall,
        "recall_gt": f"exact brute force (qvg_brute_force_topk), first {rq} queries",
        "e2e": {"value": e2e, "unit": "queries/s", "h2d_bytes_per_step": nq * D * 4,
                "d2h_bytes_per_step": nq * (8 * k + 4) + 4,
                "api": "qvg_search (C-ABI drop-in for run_query_batch), pinned host buffers"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "search_kernel (fused BQ beam search + rerank)",
                     "kernel_ms": kern_avg, "kernel_share": sum(kern_ms) / tot_ms,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_per_query": alg_bytes / nq, "peak_source": peak_src,
                     "traffic_source": traffic_src,
                     # the contract's nominal peak next to the measured one,
                     # and the code gathers the lossy visited table repeats (overhead,
                     # never counted as algorithmic bytes)
                     "frac_of_nominal_8tbs": achieved / 8000.0,
                     "lossy_regather_bytes_per_launch":
                         (lo["stats"]["dist_evals"] - ex["stats"]["dist_evals"]) * 16
                         * ((D + 63) // 64)},
        "counters": {"expansions_per_query": ex["stats"]["expansions"] / nq,
                     "tie_expansions_per_query": ex["stats"]["tie_expansions"] / nq,
                     "evals_per_query_exact": ex["stats"]["dist_evals"] / nq,
                     "evals_per_query_lossy": lo["stats"]["dist_evals"] / nq,
                     "tie_overflows": ex["stats"]["tie_overflows"]},
        "cpu_baseline": cpu, "parity": par, "ef_sweep": sweep, "batch_latency": lat,
        "rerank_depth": depth_rows, "relaxed": rel_rows,
        "sigma_over_sqrt_d_variant": variant,
        "gpu_launches": 2 * args.steps, "clocks": clocks,
    }
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


def reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (qivr::run_query_batch from oracle/_ref) with every host thread, on the same
    workload, graph and config as our arm; each step is the FULL query batch.
    This process never imports the product package (libqvg.so is not loaded)."""
    rank, world, local = dist_env()
    if rank != 0:
        return  # the reference arm runs on rank 0 only
    cfg, base, queries, adj, entry, provenance = load_workload(args, allow_gpu_build=False)
    k, ef = args.k, args.ef
    n, D = base.shape
    nq = queries.shape[0]
    ci = cpu_info()
    threads = ci["threads_used"]
    rr = RefRunner(cfg, base, adj, entry, threads)
    for _ in range(args.warmup):
        rr.timed(queries, ef, k)
    t = 0.0
    for _ in range(args.steps):
        _, dt = rr.timed(queries, ef, k)
        t += dt
    value = nq * args.steps / t
    out = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
           "data": "synthetic (seeded clustered mixture)", "impl": "reference",
           "config": bench_config(args, cfg, n, D, nq, provenance),
           "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads,
                            "kind": "reference",
                            "sample": f"the full {nq}-query batch per step (no subsampling), "
                                      f"qivr::run_query_batch with {threads} threads "
                                      "(oracle/_ref: the unmodified reference sources, "
                                      "-O3 -march=sapphirerapids)",
                            "cpu": ci},
           "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(json.dumps(out) + "\n")


def main():
    args = parse()
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
